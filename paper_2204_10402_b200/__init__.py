"""B200-native exact Minimum / Parameterized Vertex Cover search (arXiv 2204.10402).

Drop-in for the reference's Python module ``vcsolve`` (proj/python/vcsolve/__init__.py,
proj/python/bindings.cpp): the same graph loader, the same ``solve_mvc`` / ``solve_pvc`` entry
points and report dict, the same exceptions. Every solve runs on the GPU through
``libvcgpu.so`` (include/vcgpu.h); strategies:

* ``"hybrid"`` (default) — the paper's hybrid traversal (per-worker stacks + a threshold-gated
  device worklist) with ``workers`` GPU workers (warps), like run_hybrid (scheduler.cpp:328-359);
* ``"gpu"``    — the same traversal sized to fill the device (``workers=None``);
* ``"seq"``    — one GPU worker, no donation: the reference's sequential order
  (solve_mvc_seq / solve_pvc_seq, solver_seq.cpp:56-159), node for node.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as _n
from ._native import ParseError
from .report import make_report

__all__ = [
    "BaseGraph", "ParseError", "brute_force_mvc", "complement", "greedy_approx", "load_graph",
    "make_graph", "parse_dimacs", "parse_edge_list", "solve_mvc", "solve_pvc",
    "write_edge_list", "verify_cover", "device_count",
]

_lib = _n.lib


class BaseGraph:
    """Immutable CSR graph (graph.hpp:34-53); wraps a library-owned ``vcg_graph``."""

    __slots__ = ("_h",)

    def __init__(self, handle):
        if not handle:
            raise ValueError("null graph handle")
        self._h = C.c_void_p(handle)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.vcg_graph_destroy(h)
            self._h = None

    @property
    def num_vertices(self) -> int:
        return int(_lib.vcg_graph_num_vertices(self._h))

    @property
    def num_edges(self) -> int:
        return int(_lib.vcg_graph_num_edges(self._h))

    @property
    def id_base(self) -> int:
        return int(_lib.vcg_graph_id_base(self._h))

    def csr(self):
        """(offsets u64[n+1], neighbors u32[2m]) — copies of the library's CSR."""
        n, m = self.num_vertices, self.num_edges
        off = np.ctypeslib.as_array(C.cast(_lib.vcg_graph_offsets(self._h),
                                           C.POINTER(C.c_uint64)), shape=(n + 1,)).copy()
        if m:
            nbr = np.ctypeslib.as_array(C.cast(_lib.vcg_graph_neighbors(self._h),
                                               C.POINTER(C.c_uint32)), shape=(2 * m,)).copy()
        else:
            nbr = np.zeros(0, np.uint32)
        return off, nbr

    def degree(self, v: int) -> int:
        off, _ = self.csr()
        return int(off[v + 1] - off[v])

    def has_edge(self, u: int, v: int) -> bool:
        return bool(_lib.vcg_has_edge(self._h, u, v))

    def neighbors(self, v: int):
        off, nbr = self.csr()
        return nbr[int(off[v]):int(off[v + 1])].tolist()

    def __eq__(self, other):
        return isinstance(other, BaseGraph) and bool(_lib.vcg_graph_equal(self._h, other._h))

    __hash__ = None

    def __repr__(self):
        return f"BaseGraph(n={self.num_vertices}, m={self.num_edges})"


def _graph_out(fn, *args) -> BaseGraph:
    h = C.c_void_p()
    _n.check(fn(*args, C.byref(h)))
    return BaseGraph(h.value)


def parse_edge_list(text: str) -> BaseGraph:
    """Parse a whitespace-separated edge list ('#'/'%' comments) (graph.cpp:81-114)."""
    b = text.encode()
    return _graph_out(_lib.vcg_parse_edge_list, b, len(b))


def parse_dimacs(text: str) -> BaseGraph:
    """Parse a DIMACS ascii clique file ('p edge N M') (graph.cpp:116-159)."""
    b = text.encode()
    return _graph_out(_lib.vcg_parse_dimacs, b, len(b))


def make_graph(num_vertices: int, edges) -> BaseGraph:
    """Build a graph from (u, v) pairs; duplicates and self-loops are dropped (graph.cpp:22-54)."""
    p = np.ascontiguousarray(np.asarray(list(edges) if not isinstance(edges, np.ndarray) else edges,
                                        dtype=np.int64).reshape(-1))
    if len(p) and (p.min() < 0 or p.max() > 0xFFFFFFFF):
        raise ValueError("vertex id out of range")
    p = p.astype(np.uint32)
    return _graph_out(_lib.vcg_make_graph, num_vertices, len(p) // 2,
                      p.ctypes.data if len(p) else None, 0)


def from_csr(n, m, offsets, neighbors, id_base=0) -> BaseGraph:
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    nbr = np.ascontiguousarray(neighbors, dtype=np.uint32)
    return _graph_out(_lib.vcg_graph_from_csr, n, m, off.ctypes.data,
                      nbr.ctypes.data if len(nbr) else None, id_base)


def complement(graph: BaseGraph) -> BaseGraph:
    """Edge complement (graph.cpp:161-185)."""
    return _graph_out(_lib.vcg_complement, graph._h)


def write_edge_list(graph: BaseGraph) -> str:
    """One "u v" line per edge, u < v, original ids (graph.cpp:187-193)."""
    p = C.c_void_p()
    ln = C.c_size_t()
    _n.check(_lib.vcg_write_edge_list(graph._h, C.byref(p), C.byref(ln)))
    try:
        return C.string_at(p, ln.value).decode()
    finally:
        _lib.vcg_free_buffer(p)


def greedy_approx(graph: BaseGraph):
    """Greedy upper bound: (size, cover in internal ids) (bounds.cpp:7-19)."""
    size = C.c_uint32()
    cov = np.zeros(max(graph.num_vertices, 1), np.uint32)
    _n.check(_lib.vcg_greedy(graph._h, C.byref(size), cov.ctypes.data))
    return int(size.value), cov[: size.value].tolist()


def brute_force_mvc(graph: BaseGraph):
    """Exhaustive oracle for graphs of at most 20 vertices (solver_seq.cpp:173-211)."""
    size = C.c_uint32()
    cov = np.zeros(max(graph.num_vertices, 1), np.uint32)
    _n.check(_lib.vcg_brute_force(graph._h, C.byref(size), cov.ctypes.data))
    return int(size.value), cov[: size.value].tolist()


def verify_cover(graph: BaseGraph, cover, original_ids=True) -> bool:
    """verify_cover (bounds.cpp:32-45); ``cover`` in original ids unless original_ids=False."""
    c = np.asarray(list(cover), dtype=np.int64)
    if original_ids:
        c = c - graph.id_base
    if len(c) and (c.min() < 0 or c.max() >= graph.num_vertices):
        return False
    c = np.ascontiguousarray(c.astype(np.uint32))
    ok = C.c_int()
    _n.check(_lib.vcg_verify_cover(graph._h, c.ctypes.data if len(c) else None, len(c), C.byref(ok)))
    return bool(ok.value)


def device_count() -> int:
    return int(_lib.vcg_device_count())


def load_graph(path, fmt=None, complement_input=False) -> BaseGraph:
    """Load a graph file (vcsolve/__init__.py:38-51): "edgelist" or "dimacs", sniffed from the
    extension (.clq/.col/.dimacs mean DIMACS); optionally solve on the edge complement."""
    if fmt is None:
        lower = str(path).lower()
        fmt = "dimacs" if lower.endswith((".clq", ".col", ".dimacs")) else "edgelist"
    with open(path, "r", encoding="utf-8") as handle:
        text = handle.read()
    graph = parse_dimacs(text) if fmt == "dimacs" else parse_edge_list(text)
    return complement(graph) if complement_input else graph


_STRATEGIES = {"hybrid": _n.VCG_HYBRID, "gpu": _n.VCG_HYBRID, "seq": _n.VCG_SEQ,
               "stackonly": _n.VCG_STACKONLY}
_RULES = {"reference": 0, "parallel": 1}
_ENGINES = {"auto": 0, "dense": 1, "sparse": 2, "dense-wide": 3, "dense-nomid": 4,
            "dense-mid8": 5, "dense-mid4": 6, "sparse-global": 7}


def _solve(graph, mode, k, strategy, workers, capacity, threshold_fraction, depth, backoff_us,
           timeout_s, node_budget, *, device=0, rules="reference", block_warps=0,
           instrument=False, initial_best=0, seeds=None, mailbox=None, raw=False,
           donate_oldest=None, stream=None, engine="auto", certify=False, debug_flags=0,
           device_workers=None):
    """The strategy dispatch of bindings.cpp:60-99, on the GPU through vcg_solve."""
    p, keep = _params(mode, k, strategy, workers, capacity, threshold_fraction, depth, backoff_us,
                      timeout_s, node_budget, device=device, rules=rules, block_warps=block_warps,
                      instrument=instrument, initial_best=initial_best, seeds=seeds,
                      mailbox=mailbox, donate_oldest=donate_oldest, stream=stream, engine=engine,
                      certify=certify, debug_flags=debug_flags, device_workers=device_workers)
    workers = p.workers
    r = _n.Result()
    _n.check(_lib.vcg_solve(graph._h, C.byref(p), C.byref(r)))
    try:
        out = _result_dict(r)
    finally:
        _lib.vcg_result_free(C.byref(r))
    del keep
    if raw:
        out.pop("_worker_nodes_np", None)
        return out
    return make_report(graph, mode, k, strategy, workers if workers else out["num_workers"],
                       capacity, threshold_fraction, depth, out)


def _params(mode, k, strategy, workers, capacity, threshold_fraction, depth, backoff_us,
            timeout_s, node_budget, *, device=0, rules="reference", block_warps=0,
            instrument=False, initial_best=0, seeds=None, mailbox=None, donate_oldest=None,
            stream=None, engine="auto", certify=False, debug_flags=0, device_workers=None):
    """vcg_params for one solve (validated like bindings.cpp:60-99) + the arrays it points to.

    Workers: "hybrid" keeps the reference's meaning of ``workers`` (its report has that many
    entries) but always fills the device — its device workers are folded into the report —
    unless ``device_workers`` fixes the warp / CTA count. "gpu": ``workers`` = device workers
    (0 = fill the device), one report entry each. "stackonly": ``workers`` device workers."""
    if strategy not in _STRATEGIES:
        raise ValueError(f"unknown strategy: {strategy}")  # bindings.cpp:92
    if engine not in _ENGINES:
        raise ValueError(f"unknown engine: {engine}")
    if workers is None:
        workers = {"hybrid": 4, "gpu": 0, "seq": 1, "stackonly": 4}[strategy]
    if workers < 0 or (strategy != "gpu" and workers < 1):
        raise ValueError("num_workers must be >= 1")  # scheduler.cpp:21
    p = _n.Params()
    _lib.vcg_params_init(C.byref(p))
    p.mode = _n.VCG_PVC if mode == "pvc" else _n.VCG_MVC
    p.k = k
    p.strategy = _STRATEGIES[strategy]
    if device_workers is not None and device_workers < 1:
        raise ValueError("device_workers must be >= 1")
    if strategy == "gpu":
        p.workers, p.device_workers = 0, workers
    else:
        p.workers, p.device_workers = workers, device_workers or 0
    p.capacity = capacity
    p.threshold_fraction = threshold_fraction
    p.depth = depth
    p.backoff_us = backoff_us
    p.timeout_s = -1.0 if timeout_s is None else float(timeout_s)
    p.node_budget = node_budget or 0
    p.device = device
    p.rules = _RULES[rules]
    p.block_warps = block_warps
    p.engine = _ENGINES[engine]
    p.instrument = int(bool(instrument))
    if donate_oldest is None:
        # the tuned policy on a filled device; the reference's (donate the new child) when
        # hybrid runs a fixed, small number of device workers
        donate_oldest = not (strategy == "hybrid" and device_workers)
    p.donate_oldest = int(bool(donate_oldest))
    p.initial_best = initial_best or 0
    p.debug_flags = int(debug_flags) | (_n.VCG_DEBUG_CERTIFY if certify else 0)
    keep = None
    if seeds is not None and len(seeds):
        keep = np.ascontiguousarray(seeds, dtype=np.uint32)
        p.num_seeds = keep.shape[0]
        p.seeds = keep.ctypes.data_as(C.POINTER(C.c_uint32))
    if mailbox is not None:
        p.mailbox = C.cast(mailbox, C.POINTER(C.c_uint32))
    if stream is not None:
        p.stream = C.c_void_p(int(stream))
    return p, keep


def _array(ptr, count):
    """A library-owned C array as a Python int list (one bulk copy, not per-element ctypes)."""
    if count == 0 or not ptr:
        return []
    return np.ctypeslib.as_array(ptr, shape=(count,)).tolist()


def _array_np(ptr, count):
    """A copy of a library-owned C array as a numpy array (valid after vcg_result_free)."""
    if count == 0 or not ptr:
        return np.zeros(0, dtype=np.uint64)
    return np.ctypeslib.as_array(ptr, shape=(count,)).copy()


def _result_dict(r):
    nw = r.num_workers
    return dict(
        status=_n.STATUS_NAMES[r.status], size=int(r.size), feasible=bool(r.feasible),
        greedy_size=int(r.greedy_size),
        cover=_array(r.cover, r.cover_len),
        cover_from_search=bool(r.cover_from_search), num_workers=nw,
        worker_nodes=_array(r.worker_nodes, nw),
        # (the same counts as an array: the report's load ratios without a list -> array pass
        # over thousands of device workers on the host's critical path between solves)
        _worker_nodes_np=_array_np(r.worker_nodes, nw),
        worker_stack_high_water=_array(r.worker_stack_high_water, nw),
        nodes_total=int(r.nodes_total),
        worklist=dict(added=int(r.wl_added), removed=int(r.wl_removed),
                      max_size=int(r.wl_max_size), current_size=int(r.wl_current_size)),
        wall_ms=float(r.wall_ms), device_ms=float(r.device_ms), greedy_ms=float(r.greedy_ms),
        h2d_ms=float(r.h2d_ms), h2d_bytes=int(r.h2d_bytes), d2h_bytes=int(r.d2h_bytes),
        rounds=int(r.rounds), maxdeg_passes=int(r.maxdeg_passes), children=int(r.children),
        removals=int(r.removals), donated=int(r.donated),
        removals_deg1=int(r.removals_deg1), removals_deg2=int(r.removals_deg2),
        removals_high=int(r.removals_high), doomed=int(r.doomed), degree_bytes=int(r.degree_bytes), n_padded=int(r.n_padded),
        engine=int(r.engine), grid_blocks=int(r.grid_blocks), block_threads=int(r.block_threads),
        kernel_launches=int(r.kernel_launches),
        phase_cycles=[int(x) for x in r.phase_cycles], active_cycles=int(r.active_cycles),
        donated_peer=int(r.donated_peer),
        certify_nodes=int(r.certify_nodes), certify_ms=float(r.certify_ms),
        timeline=dict(first_node_ms=[float(x) for x in r.t_first_ms],
                      exit_ms=[float(x) for x in r.t_end_ms],
                      idle_share=float(r.idle_share),
                      final_wait_ms=[float(x) for x in r.t_lastwait_ms]),
    )


def solve_mvc(graph, strategy="hybrid", workers=None, capacity=4096, threshold_fraction=0.5,
              depth=8, backoff_us=50, timeout_s=None, node_budget=None, **gpu):
    """Solve MVC; returns the run report as a dict (bindings.cpp:174-187).

    GPU keyword knobs: device, device_workers, engine ("auto" | "dense" | "sparse"), rules, block_warps,
    instrument, donate_oldest, initial_best, seeds, mailbox, stream, raw; certify=True re-proves
    the optimum by PVC(size - 1) (a debug cross-check, reported as certify_nodes / certify_ms)."""
    return _solve(graph, "mvc", 0, strategy, workers, capacity, threshold_fraction, depth,
                  backoff_us, timeout_s, node_budget, **gpu)


def solve_pvc(graph, k, strategy="hybrid", workers=None, capacity=4096, threshold_fraction=0.5,
              depth=8, backoff_us=50, timeout_s=None, node_budget=None, **gpu):
    """Solve PVC for a given k; returns the run report as a dict (bindings.cpp:188-202)."""
    if k < 1:
        raise ValueError("pvc requires k >= 1")  # bindings.cpp:194
    if "initial_best" in gpu:
        raise TypeError("initial_best applies to MVC only")
    return _solve(graph, "pvc", k, strategy, workers, capacity, threshold_fraction, depth,
                  backoff_us, timeout_s, node_budget, **gpu)
