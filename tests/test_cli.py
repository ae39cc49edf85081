"""The vcsolve CLI (paper_2204_10402_b200/cli/vcsolve.cpp) against the reference CLI's own
end-to-end checks (proj/tests/python/test_cli.py): same options, report formats, exit codes and
sweep matrix, plus `--strategy gpu`. The "oracle" strategy is host-only, so the sweep logic and
the report writers are covered on CPU; every run that searches is marked gpu."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2204_10402_b200", "bin", "vcsolve")
DATA = os.path.join(ROOT, "tests", "data")

pytestmark = pytest.mark.skipif(not os.path.exists(BIN), reason="vcsolve not built (make)")


def run_cli(*args, expect=0):
    proc = subprocess.run([BIN, *args], capture_output=True, text=True, timeout=300)
    assert proc.returncode == expect, proc.stderr
    return proc


def data(name):
    return os.path.join(DATA, name)


# ------------------------------------------------------------------ host-only (CPU)

def test_oracle_strategy_and_its_limit():  # test_cli.py:68-71
    proc = run_cli("--input", data("petersen.el"), "--strategy", "oracle")
    rep = json.loads(proc.stdout)
    assert rep["size"] == 6 and rep["status"] == "complete" and rep["worker_nodes"] == [1024]
    assert len(rep["cover"]) == 6
    run_cli("--input", data("big_path.el"), "--strategy", "oracle", expect=1)


def test_oracle_cover_matches_reference_brute_force(reference):
    rep = json.loads(run_cli("--input", data("petersen.el"), "--strategy", "oracle").stdout)
    size, cover = reference.brute_force(reference.parse(open(data("petersen.el")).read()))
    assert rep["size"] == size and rep["cover"] == list(cover)


def test_missing_k_is_a_usage_error():  # test_cli.py:59-60
    run_cli("--input", data("p3.el"), "--mode", "pvc", expect=1)
    run_cli("--input", data("p3.el"), "--mode", "pvc", "--k", "0", expect=1)


def test_usage_errors():
    run_cli("--input", data("p3.el"), "--strategy", "fast", expect=1)
    run_cli("--input", data("p3.el"), "--depth", "31", expect=1)
    run_cli("--input", data("p3.el"), "--output", "xml", expect=1)
    run_cli("--mode", "mvc", expect=1)  # --input is required
    run_cli("--input", data("p3.el"), "--bogus", expect=1)
    run_cli("--input", "/nonexistent/graph.el", "--strategy", "oracle", expect=1)


def test_parse_error_exit_code(tmp_path):
    bad = tmp_path / "bad.el"
    bad.write_text("0 1\n1 x\n")
    proc = run_cli("--input", str(bad), "--strategy", "oracle", expect=1)
    assert "parse error" in proc.stderr and "line 2" in proc.stderr


def test_oracle_pvc_and_dimacs_complement():  # test_cli.py:47-54 on the host-only strategy
    rep = json.loads(run_cli("--input", data("triangle_plus.clq"), "--format", "dimacs",
                             "--complement", "--strategy", "oracle").stdout)
    assert rep["complemented"] is True and rep["n"] == 5 and rep["m"] == 6
    yes = json.loads(run_cli("--input", data("petersen.el"), "--mode", "pvc", "--k", "6",
                             "--strategy", "oracle").stdout)
    assert yes["feasible"] is True and yes["size"] == 6 and yes["k"] == 6
    no = json.loads(run_cli("--input", data("petersen.el"), "--mode", "pvc", "--k", "5",
                            "--strategy", "oracle").stdout)
    assert no["feasible"] is False and no["size"] is None and no["cover"] == []


def test_csv_text_and_report_file(tmp_path):  # test_cli.py:79-90
    out = tmp_path / "report.csv"
    run_cli("--input", data("p3.el"), "--strategy", "oracle", "--output", "csv",
            "--report", str(out))
    lines = out.read_text().strip().splitlines()
    assert len(lines) == 2
    header, row = lines[0].split(","), lines[1].split(",")
    assert len(header) == len(row) and "cover" not in header
    assert row[header.index("size")] == "1"
    assert header == ("file,complemented,n,m,mode,k,strategy,workers,capacity,"
                      "threshold_fraction,depth,size,feasible,wall_ms,status,worker_nodes,"
                      "load_ratios,phase_shares").split(",")
    text = run_cli("--input", data("p3.el"), "--strategy", "oracle", "--output", "text").stdout
    assert "result:    size=1" in text and "cover:     1" in text


def test_sweep_matrix_host_only(tmp_path):  # test_cli.py:93-113 with the oracle strategy
    out = tmp_path / "sweep.json"
    run_cli("sweep", "--input", data("petersen.el"), "--strategies", "oracle",
            "--instances", "pvc-1,pvc,pvc+1,mvc", "--out", str(out))
    rows = json.loads(out.read_text())
    assert [r["instance"] for r in rows] == ["mvc", "pvc-1", "pvc", "pvc+1"]
    assert all(r["best"] for r in rows)
    assert rows[0]["size"] == 6
    assert rows[1]["feasible"] is False and rows[1]["k"] == 5
    assert rows[2]["feasible"] is True and rows[3]["k"] == 7
    csv = tmp_path / "sweep.csv"
    run_cli("--input", data("c5.el"), "--output", "csv", "sweep", "--strategies", "oracle",
            "--instances", "mvc", "--out", str(csv))
    lines = csv.read_text().strip().splitlines()
    assert lines[0].startswith("instance,best,file,") and len(lines) == 2
    assert lines[1].split(",")[lines[0].split(",").index("size")] == "3"


# ------------------------------------------------------------------ device runs

@pytest.mark.gpu
def test_solve_p3_seq_json():  # test_cli.py:25-30
    rep = json.loads(run_cli("--input", data("p3.el"), "--mode", "mvc", "--strategy",
                             "seq").stdout)
    assert rep["size"] == 1 and rep["cover"] == [1] and rep["status"] == "complete"
    assert rep["workers"] == 1 and rep["engine"]["kernel_launches"] >= 1


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["hybrid", "gpu", "stackonly"])
def test_solve_petersen_pvc(strategy):  # test_cli.py:33-44
    rep = json.loads(run_cli("--input", data("petersen.el"), "--mode", "pvc", "--k", "6",
                             "--strategy", strategy, "--workers", "8").stdout)
    assert rep["feasible"] is True and rep["size"] <= 6
    rep = json.loads(run_cli("--input", data("petersen.el"), "--mode", "pvc", "--k", "5",
                             "--strategy", strategy, "--workers", "4").stdout)
    assert rep["feasible"] is False and rep["size"] is None


@pytest.mark.gpu
def test_dimacs_complement_report():  # test_cli.py:47-54
    rep = json.loads(run_cli("--input", data("triangle_plus.clq"), "--format", "dimacs",
                             "--complement", "--strategy", "seq").stdout)
    assert rep["complemented"] is True and rep["n"] == 5 and rep["m"] == 6


@pytest.mark.gpu
def test_depth_with_hybrid_warns_but_runs():  # test_cli.py:63-65
    proc = run_cli("--input", data("p3.el"), "--strategy", "hybrid", "--depth", "4")
    assert "ignored" in proc.stderr
    assert json.loads(proc.stdout)["size"] == 1


@pytest.mark.gpu
def test_budget_exit_code():  # test_cli.py:74-76
    run_cli("--input", data("petersen.el"), "--strategy", "seq", "--node-budget", "2", expect=2)


@pytest.mark.gpu
def test_stackonly_csv_report_file(tmp_path):  # test_cli.py:79-90
    out = tmp_path / "report.csv"
    run_cli("--input", data("p3.el"), "--strategy", "stackonly", "--depth", "2", "--workers", "2",
            "--output", "csv", "--report", str(out))
    lines = out.read_text().strip().splitlines()
    header, row = lines[0].split(","), lines[1].split(",")
    assert len(lines) == 2 and len(header) == len(row) and row[header.index("size")] == "1"


@pytest.mark.gpu
def test_sweep_matrix(tmp_path):  # test_cli.py:93-113, with gpu added to the strategies
    out = tmp_path / "sweep.json"
    run_cli("sweep", "--input", data("petersen.el"),
            "--strategies", "seq,stackonly,hybrid,gpu", "--workers", "2", "--depths", "4",
            "--capacities", "64", "--fractions", "0.5", "--instances", "mvc,pvc-1,pvc,pvc+1",
            "--out", str(out))
    rows = json.loads(out.read_text())
    mvc_rows = [r for r in rows if r["instance"] == "mvc"]
    assert len(mvc_rows) == 4 and all(r["size"] == 6 for r in mvc_rows)
    for strategy in ("seq", "stackonly", "hybrid", "gpu"):
        group = [r for r in mvc_rows if r["strategy"] == strategy]
        assert sum(1 for r in group if r["best"]) == 1
    pvc_minus = [r for r in rows if r["instance"] == "pvc-1"]
    assert pvc_minus and all(r["feasible"] is False for r in pvc_minus)
    for inst in ("pvc", "pvc+1"):
        rows_inst = [r for r in rows if r["instance"] == inst]
        assert rows_inst and all(r["feasible"] is True for r in rows_inst)


@pytest.mark.gpu
def test_sweep_thresholds_same_size(tmp_path):  # test_cli.py:116-128
    out = tmp_path / "sweep.csv"
    run_cli("sweep", "--input", data("c5.el"), "--strategies", "hybrid", "--workers", "2",
            "--capacities", "16", "--fractions", "0.25,0.5,0.75,1.0", "--instances", "mvc",
            "--output", "csv", "--out", str(out))
    lines = out.read_text().strip().splitlines()
    assert len(lines) == 5
    header = lines[0].split(",")
    assert {ln.split(",")[header.index("size")] for ln in lines[1:]} == {"3"}


@pytest.mark.gpu
def test_gpu_strategy_on_config_c1_matches_golden(config_golden):
    path = os.path.join(ROOT, "data", "configs", "c1.clq.gz")
    if not os.path.exists(path):
        pytest.skip("config graphs not present")
    import gzip
    import tempfile
    with tempfile.NamedTemporaryFile("wb", suffix=".clq", delete=False) as f:
        f.write(gzip.decompress(open(path, "rb").read()))
    try:
        rep = json.loads(run_cli("--input", f.name, "--strategy", "gpu").stdout)
    finally:
        os.unlink(f.name)
    assert rep["size"] == config_golden["c1"]["mvc"] and rep["status"] == "complete"
