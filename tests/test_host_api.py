"""The drop-in surface on the host (CPU only): libvcgpu.so loads and exports every symbol
include/vcgpu.h declares; the graph loader, make_graph/complement, greedy seed, brute force and
error mapping behave like the reference's Python module (proj/tests/python/test_smoke.py,
proj/tests/test_graph.cpp). No solve runs here (no GPU in this container)."""
import os
import re

import numpy as np
import pytest

import paper_2204_10402_b200 as vc
from paper_2204_10402_b200 import _native
from paper_2204_10402_b200.configs import load_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def petersen():
    return vc.make_graph(10, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0), (0, 5), (1, 6), (2, 7),
                              (3, 8), (4, 9), (5, 7), (7, 9), (9, 6), (6, 8), (8, 5)])


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "vcgpu.h")).read()
    declared = set(re.findall(r"VCG_API\s+[\w\s\*]+?\b(vcg_\w+)\s*\(", header))
    assert len(declared) >= 25
    assert declared == set(_native.EXPORTS), declared ^ set(_native.EXPORTS)
    for name in declared:
        assert hasattr(_native.lib, name), name
    assert b"sm_100a" in _native.lib.vcg_version()


# ---- proj/tests/python/test_smoke.py --------------------------------------------------------

def test_parse_edge_list():
    g = vc.parse_edge_list("0 1\n1 2\n")
    assert g.num_vertices == 3 and g.num_edges == 2
    assert g.degree(1) == 2 and g.neighbors(1) == [0, 2]


def test_parse_dimacs_and_complement():
    g = vc.parse_dimacs("p edge 3 2\ne 1 2\ne 2 3\n")
    assert g.num_vertices == 3 and g.num_edges == 2
    gc = vc.complement(g)
    assert gc.num_edges == 1 and gc.has_edge(0, 2)


def test_parse_error_carries_line_info():
    with pytest.raises(ValueError, match="line 2"):
        vc.parse_edge_list("0 1\nbogus 2\n")
    with pytest.raises(vc.ParseError):
        vc.parse_edge_list("0 1\nbogus 2\n")


def test_greedy_is_a_valid_upper_bound():
    g = petersen()
    size, cover = vc.greedy_approx(g)
    assert size >= 6 and len(cover) == size
    assert vc.verify_cover(g, cover, original_ids=False)


def test_load_graph_roundtrip(tmp_path):
    p = tmp_path / "p3.el"
    p.write_text("0 1\n1 2\n")
    g = vc.load_graph(p)
    assert g.num_vertices == 3
    assert vc.write_edge_list(g) == "0 1\n1 2\n"


def test_oracle_size_limit():
    g = vc.make_graph(25, [(i, i + 1) for i in range(24)])
    with pytest.raises(Exception):
        vc.brute_force_mvc(g)


# ---- parser semantics (graph.cpp:81-159, test_graph.cpp) -----------------------------------

@pytest.mark.parametrize("text,n,m,base", [
    ("1 2\n2 3\n", 3, 2, 1),                        # 1-based autodetect
    ("# c\n% c\n\n0 1\n", 2, 1, 0),                 # comments and blanks
    ("0 1\n1 0\n0 0\n", 2, 1, 0),                   # duplicates and self-loops dropped
    ("0 5\n", 6, 1, 0),                             # isolated vertices up to the max id kept
    ("", 0, 0, 0),
    ("3 4\r\n4 5\r\n", 5, 2, 1),                    # CR is whitespace; 1-based, n = max id
])
def test_edge_list_semantics(text, n, m, base):
    g = vc.parse_edge_list(text)
    assert (g.num_vertices, g.num_edges, g.id_base) == (n, m, base if n else 0)


@pytest.mark.parametrize("text,msg", [
    ("0\n", "line 1: expected 'u v' pair"),
    ("0 1 2\n", "line 1: trailing token '2'"),
    ("0 1\n0 -1\n", "line 2: malformed vertex id '-1'"),
    ("0 4294967295\n", "line 1: vertex id out of range '4294967295'"),
])
def test_edge_list_errors(text, msg):
    with pytest.raises(ValueError) as e:
        vc.parse_edge_list(text)
    assert str(e.value) == msg


@pytest.mark.parametrize("text,msg", [
    ("e 1 2\n", "line 1: 'e' line before 'p' line"),
    ("p edge 3 1\np edge 3 1\n", "line 2: duplicate 'p' line"),
    ("p foo 3 1\n", "line 1: unsupported format 'foo'"),
    ("p edge x 1\n", "line 1: malformed 'p' line"),
    ("p edge 3 1\ne 1 4\n", "line 2: edge endpoint outside 1..3"),
    ("p edge 3 1\nx 1 2\n", "line 2: unrecognized line type 'x'"),
    ("c only\n", "line 1: missing 'p edge N M' line"),
    ("", "line 1: missing 'p edge N M' line"),
])
def test_dimacs_errors(text, msg):
    with pytest.raises(ValueError) as e:
        vc.parse_dimacs(text)
    assert str(e.value) == msg


def test_dimacs_triangle_plus_complement():  # tests/data/triangle_plus.clq, test_cli.py:47-54
    g = vc.parse_dimacs("c triangle with two pendants\np edge 5 4\ne 1 2\ne 2 3\ne 1 3\ne 4 5\n")
    assert (g.num_vertices, g.num_edges, g.id_base) == (5, 4, 1)
    assert vc.complement(g).num_edges == 6


def test_parsers_match_the_reference(reference):
    texts = ["0 1\n1 2\n", "5 6\n6 7\n7 5\n", "# x\n3 1\n1 3\n2 2\n9 4\n", "3 4\r\n4 5\r\n"]
    for t in texts:
        a = vc.parse_edge_list(t)
        b = reference.parse(t)
        off, nbr = a.csr()
        assert a.num_vertices == b.n and a.id_base == b.id_base
        assert (off == b.offsets).all() and (nbr == b.neighbors).all()
    for bad in ["0 1 2\n", "a b\n", "1\n"]:
        with pytest.raises(ValueError) as e:
            vc.parse_edge_list(bad)
        with pytest.raises(ValueError) as f:
            reference.parse(bad)
        assert str(e.value) == str(f.value)


def test_make_graph_and_complement_match_oracle(oracle, corpus):
    for it in corpus[::7]:
        g = vc.make_graph(it["n"], [tuple(e) for e in it["edges"]])
        o = oracle.make_graph(it["n"], it["edges"])
        off, nbr = g.csr()
        assert (off == o.offsets).all() and (nbr == o.neighbors).all()
        gc = vc.complement(g)
        oc = oracle.complement(o)
        off, nbr = gc.csr()
        assert (off == oc.offsets).all() and (nbr == oc.neighbors).all()


def test_graph_equality_and_invariants():
    a = petersen()
    b = petersen()
    assert a == b and not (a == vc.complement(a))
    off, nbr = a.csr()
    c = vc.from_csr(a.num_vertices, a.num_edges, off, nbr)
    assert c == a
    bad = nbr.copy()
    bad[0], bad[1] = bad[1], bad[0]  # unsorted slice
    with pytest.raises(ValueError):
        vc.from_csr(a.num_vertices, a.num_edges, off, bad)
    # asymmetric: vertex 0 lists 1, 4, 5; retarget its last slot to 6 (sorted, but 6 does not
    # list 0 and 5 now has one entry too many)
    asym = nbr.copy()
    assert list(asym[off[0]:off[1]]) == [1, 4, 5]
    asym[off[1] - 1] = 6
    with pytest.raises(ValueError):
        vc.from_csr(a.num_vertices, a.num_edges, off, asym)
    # a self-loop / out-of-range id
    loop = nbr.copy()
    loop[off[1] - 1] = 0
    with pytest.raises(ValueError):
        vc.from_csr(a.num_vertices, a.num_edges, off, loop)


# ---- host seed and oracle functions vs the reference's golden answers ---------------------

def test_greedy_cover_equals_the_reference(corpus):
    for it in corpus:
        g = vc.make_graph(it["n"], [tuple(e) for e in it["edges"]])
        assert vc.greedy_approx(g) == (it["greedy_size"], it["greedy_cover"]), it["name"]


def test_greedy_on_configs_equals_the_reference(config_golden):
    for name in ("c1", "c2", "c3", "c4", "c5"):
        assert vc.greedy_approx(load_config(name))[0] == config_golden[name]["greedy"], name


def test_greedy_cover_c4_equals_reference_cover(reference):
    g = load_config("c4")
    off, nbr = g.csr()
    from oracle.oracle import CSR
    assert vc.greedy_approx(g) == reference.greedy(CSR(g.num_vertices, g.num_edges, off, nbr))


def test_brute_force_equals_the_reference(corpus):
    for it in corpus[::3]:
        g = vc.make_graph(it["n"], [tuple(e) for e in it["edges"]])
        size, cover = vc.brute_force_mvc(g)
        assert size == it["mvc"] and cover == it["brute_force_cover"]


def test_verify_cover():
    g = petersen()
    assert vc.verify_cover(g, [1, 3, 4, 5, 6, 7])
    assert not vc.verify_cover(g, [1, 3, 4, 5, 6])
    assert not vc.verify_cover(g, [99])


# ---- solve entry points: argument errors map like the reference; no CPU fallback -----------

def test_solve_argument_errors():
    g = petersen()
    with pytest.raises(ValueError, match="pvc requires k >= 1"):
        vc.solve_pvc(g, 0)
    with pytest.raises(ValueError, match="unknown strategy"):
        vc.solve_mvc(g, strategy="magic")
    with pytest.raises(ValueError, match="threshold_fraction"):
        vc.solve_mvc(g, threshold_fraction=0.0)
    with pytest.raises(ValueError, match="worklist_capacity"):
        vc.solve_mvc(g, capacity=0)
    with pytest.raises(ValueError, match="stackonly_depth"):
        vc.solve_mvc(g, depth=31)


@pytest.mark.skipif(vc.device_count() > 0, reason="a GPU is visible")
def test_solve_fails_loudly_without_a_gpu():
    with pytest.raises(RuntimeError, match="CUDA"):
        vc.solve_mvc(petersen())


def test_report_metrics_semantics():
    from paper_2204_10402_b200.report import collect_metrics
    ratios, shares = collect_metrics([10, 30], [0] * 10, 0)
    assert ratios == [0.5, 1.5] and shares["other"] == 1.0
    ratios, _ = collect_metrics([0, 0], [0] * 10, 0)
    assert ratios == [1.0, 1.0]  # metrics.cpp:32-36
    _, shares = collect_metrics([5], [10] + [0] * 9, 40)
    assert shares["worklist_remove"] == 0.25 and abs(shares["other"] - 0.75) < 1e-12


# ---- multi-shard session API: argument validation happens before any device work ----------

def test_session_open_validates_like_solve():
    import ctypes as C
    from paper_2204_10402_b200 import _native, _params
    g = petersen()
    h = C.c_void_p()
    p, _ = _params("pvc", 0, "gpu", 0, 4096, 0.5, 8, 50, None, None)
    with pytest.raises(ValueError, match="k >= 1"):
        _native.check(_native.lib.vcg_session_open(g._h, C.byref(p), 0, C.byref(h)))
    p, _ = _params("pvc", 3, "seq", 1, 4096, 0.5, 8, 50, None, None)
    with pytest.raises(ValueError, match="hybrid"):
        _native.check(_native.lib.vcg_session_open(g._h, C.byref(p), 0, C.byref(h)))
    p, _ = _params("mvc", 0, "gpu", 0, 4096, 1.5, 8, 50, None, None)
    with pytest.raises(ValueError, match="threshold_fraction"):
        _native.check(_native.lib.vcg_session_open(g._h, C.byref(p), 0, C.byref(h)))
    with pytest.raises(ValueError):
        _native.check(_native.lib.vcg_session_link_local(None, 2))
    assert _native.lib.vcg_session_handle_bytes() == 3 * 64  # three cudaIpcMemHandle_t


def test_shard_rejects_k_zero():
    from paper_2204_10402_b200.shards import Shard
    with pytest.raises(ValueError, match="k >= 1"):
        Shard(petersen(), "pvc", 0)


def test_shard_combine_rules():
    """shards.combine: PVC is feasible if any part found a cover; MVC keeps the smallest
    certificate among the frontier's and the parts' search covers; node counts add up."""
    from paper_2204_10402_b200.shards import combine
    fr = dict(nodes=7, levels=2, found=False, cover=[0, 1, 2, 3], greedy_size=4,
              kernel_launches=2, frontier_size=0)

    def part(**kw):
        d = dict(size=0, feasible=False, cover=[], cover_from_search=False, status="complete",
                 worker_nodes=[5], nodes_total=5, device_ms=1.0, donated=1, donated_peer=0,
                 kernel_launches=2, greedy_size=4)
        d.update(kw)
        return d
    r = combine(None, "pvc", fr, [part(), part(feasible=True, cover=[1, 2], size=2)], 1.0)
    assert r["feasible"] and r["cover"] == [1, 2] and r["size"] == 2
    assert r["nodes_total"] == 7 + 10 and r["rank_nodes"] == [5, 5]
    r = combine(None, "pvc", fr, [part(), part(status="timeout")], 1.0)
    assert not r["feasible"] and r["size"] is None and r["status"] == "timeout"
    r = combine(None, "mvc", fr, [part(size=3, cover=[0, 1, 2], cover_from_search=True, feasible=True),
                                 part(size=4, cover=[4, 5, 6, 7], feasible=True)], 1.0)
    assert r["size"] == 3 and r["cover"] == [0, 1, 2]
    r = combine(None, "mvc", fr, [part(size=4, feasible=True)], 1.0)
    assert r["size"] == 4 and r["cover"] == [0, 1, 2, 3]  # the frontier's (greedy) certificate


# ---- worker semantics of the drop-in strategies (bindings.cpp:174-202 defaults) ------------

def test_hybrid_defaults_fill_the_device_and_fold_the_report():
    """strategy="hybrid" keeps the reference's num_workers for the report (vcg_params.workers)
    but leaves the device worker count to the engine (device_workers = 0: fill the device) with
    the tuned donation policy; device_workers fixes a warp count and the reference's policy;
    "gpu" reports per warp (workers = 0)."""
    from paper_2204_10402_b200 import _params
    p, _ = _params("mvc", 0, "hybrid", None, 4096, 0.5, 8, 50, None, None)
    assert p.workers == 4 and p.device_workers == 0 and p.donate_oldest == 1
    p, _ = _params("mvc", 0, "hybrid", 4, 4096, 0.5, 8, 50, None, None, device_workers=64)
    assert p.workers == 4 and p.device_workers == 64 and p.donate_oldest == 0
    p, _ = _params("mvc", 0, "gpu", None, 4096, 0.5, 8, 50, None, None)
    assert p.workers == 0 and p.device_workers == 0 and p.donate_oldest == 1
    p, _ = _params("mvc", 0, "gpu", 512, 4096, 0.5, 8, 50, None, None)
    assert p.workers == 0 and p.device_workers == 512
    p, _ = _params("pvc", 3, "stackonly", 8, 4096, 0.5, 4, 50, None, None)
    assert p.workers == 8 and p.device_workers == 0
    with pytest.raises(ValueError):
        _params("mvc", 0, "hybrid", 4, 4096, 0.5, 8, 50, None, None, device_workers=0)
    q = _native.Params()
    _native.lib.vcg_params_init(q)
    assert q.donate_oldest == 1 and q.device_workers == 0 and q.capacity == 4096


def test_engine_names_cover_every_variant():
    from paper_2204_10402_b200 import _ENGINES
    assert set(_ENGINES) == {"auto", "dense", "sparse", "dense-wide", "dense-nomid",
                             "dense-mid8", "dense-mid4", "sparse-global"}
    with pytest.raises(ValueError):
        vc.solve_mvc(petersen(), engine="nope")


def test_c5_scale_config_loads():
    g = load_config("c5s")
    assert g.num_vertices == 500 and g.num_edges == 31127
