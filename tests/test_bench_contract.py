"""bench.py's reference arm runs on the host CPU: check its JSON line against the driver
contract (keys, types, impl tag, cpu_baseline / e2e blocks)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line(reference):
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
         "--warmup", "1", "--ref-sample-s", "0.5"],
        capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["unit"] == "nodes/s" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["warmup"] == 1
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_reference_arm_other_ranks_exit_silently():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_workloads_and_shared_config():
    """N=1 defaults to C5 (the headline), N>1 to C5-scale; both arms build the config dict with
    the same function, so the driver sees identical configs."""
    sys.path.insert(0, ROOT)
    import bench
    ns = type("A", (), {"workload": None})()
    assert bench.workload_of(ns, 1) == "c5" and bench.workload_of(ns, 8) == "c5s"
    a = bench.bench_config("c5s", 500, 31127, 4)
    assert a == bench.bench_config("c5s", 500, 31127, 4)
    assert a["k"] == 448 and a["nodes_per_step"] == 5969685861 and "C5-scale" in a["workload"]
    assert bench.WORKLOADS["c5"]["nodes"] == 21461369


def test_reference_arm_at_n2_times_c5_scale(reference):
    """Under torchrun (N>1) rank 0 runs the reference on the N>1 workload (C5-scale), with the
    same config dict as the GPU arm."""
    env = dict(os.environ, RANK="0", WORLD_SIZE="2", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--steps", "1", "--warmup", "0", "--ref-sample-s", "0.5"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["config"]["name"] == "c5s" and d["config"]["k"] == 448 and d["value"] > 0
