"""ctypes access to the CHECKERS — TEST INFRASTRUCTURE ONLY.

* ``Oracle``    : liboracle.so, our plain-C restatement of the reference (oracle.c).
* ``Reference`` : _ref/libvcref.so, the unmodified reference sources + ref_shim.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / ``--impl reference``
arm may import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
U32P = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
U64P = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
REMOVED = 0xFFFFFFFF


class CSR:
    """A host CSR (n, m, offsets u64[n+1], neighbors u32[2m]) in the reference's layout."""

    def __init__(self, n, m, offsets, neighbors, id_base=0):
        self.n = int(n)
        self.m = int(m)
        self.offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        self.neighbors = np.ascontiguousarray(neighbors, dtype=np.uint32)
        self.id_base = int(id_base)

    @staticmethod
    def from_pairs(n, pairs):
        """graph.cpp:22-54 make_graph semantics, in numpy (clean, sort, dedupe, CSR)."""
        e = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
        e = e[e[:, 0] != e[:, 1]]
        e = np.sort(e, axis=1)
        e = np.unique(e, axis=0) if len(e) else e
        m = len(e)
        deg = np.bincount(e.ravel(), minlength=n) if m else np.zeros(n, np.int64)
        off = np.zeros(n + 1, np.uint64)
        off[1:] = np.cumsum(deg)
        both = np.concatenate([e, e[:, ::-1]]) if m else np.zeros((0, 2), np.int64)
        order = np.lexsort((both[:, 1], both[:, 0]))
        nbr = both[order, 1].astype(np.uint32)
        return CSR(n, m, off, nbr)

    def pairs(self):
        src = np.repeat(np.arange(self.n, dtype=np.uint32), np.diff(self.offsets).astype(np.int64))
        mask = src < self.neighbors
        return np.stack([src[mask], self.neighbors[mask]], axis=1)

    def degrees(self):
        return np.diff(self.offsets).astype(np.uint32)


class _Graph(C.Structure):
    _fields_ = [("n", C.c_uint32), ("m", C.c_uint64),
                ("off", C.POINTER(C.c_uint64)), ("nbr", C.POINTER(C.c_uint32))]


class _OrcResult(C.Structure):
    _fields_ = [("size", C.c_uint32), ("feasible", C.c_int32), ("status", C.c_int32),
                ("greedy_size", C.c_uint32), ("nodes", C.c_uint64),
                ("stack_high_water", C.c_uint64)]


class Oracle:
    """Our C restatement (oracle.c). Each method names the reference function it restates."""

    def __init__(self, path=None):
        self.lib = C.CDLL(path or os.path.join(HERE, "liboracle.so"))
        L = self.lib
        L.orc_reduce.argtypes = [C.POINTER(_Graph), U32P, C.POINTER(C.c_uint32),
                                 C.POINTER(C.c_uint64), C.c_int, C.c_uint32, C.c_uint32, C.c_int]
        L.orc_should_prune.argtypes = [C.c_uint32, C.c_uint64, C.c_int, C.c_uint32, C.c_uint32]
        L.orc_greedy.argtypes = [C.POINTER(_Graph), U32P]
        L.orc_greedy.restype = C.c_uint32
        L.orc_verify_cover.argtypes = [C.POINTER(_Graph), U32P, C.c_uint32]
        L.orc_brute_force.argtypes = [C.POINTER(_Graph), U32P]
        L.orc_brute_force.restype = C.c_uint32
        L.orc_fingerprint.argtypes = [U32P, C.c_uint32, C.c_uint32, C.c_uint64]
        L.orc_fingerprint.restype = C.c_uint64
        L.orc_solve_seq.argtypes = [C.POINTER(_Graph), C.c_int, C.c_uint32, C.c_uint64,
                                    C.POINTER(_OrcResult), U32P]
        L.orc_make_graph.argtypes = [C.c_uint32, C.c_uint64, U32P, C.POINTER(_Graph)]
        L.orc_complement.argtypes = [C.POINTER(_Graph), C.POINTER(_Graph)]
        L.orc_graph_free.argtypes = [C.POINTER(_Graph)]
        L.orc_has_edge.argtypes = [C.POINTER(_Graph), C.c_uint32, C.c_uint32]

    @staticmethod
    def _g(csr):
        g = _Graph(csr.n, csr.m, csr.offsets.ctypes.data_as(C.POINTER(C.c_uint64)),
                   csr.neighbors.ctypes.data_as(C.POINTER(C.c_uint32)))
        g._keep = csr  # keep arrays alive
        return g

    def make_graph(self, n, pairs):
        """graph.cpp:22-54"""
        p = np.ascontiguousarray(np.asarray(pairs, dtype=np.uint32).reshape(-1))
        g = _Graph()
        if self.lib.orc_make_graph(n, len(p) // 2, p if len(p) else np.zeros(2, np.uint32),
                                   C.byref(g)) != 0:
            raise ValueError("vertex id out of range")
        return self._take(g)

    def _take(self, g):
        off = np.ctypeslib.as_array(g.off, shape=(g.n + 1,)).copy()
        nbr = (np.ctypeslib.as_array(g.nbr, shape=(2 * g.m,)).copy() if g.m
               else np.zeros(0, np.uint32))
        self.lib.orc_graph_free(C.byref(g))
        return CSR(g.n, g.m, off, nbr)

    def complement(self, csr):
        """graph.cpp:161-185"""
        out = _Graph()
        self.lib.orc_complement(C.byref(self._g(csr)), C.byref(out))
        return self._take(out)

    def has_edge(self, csr, u, v):
        return bool(self.lib.orc_has_edge(C.byref(self._g(csr)), u, v))

    def reduce(self, csr, degrees, cover_count, edges, pvc=False, k=0, best_or_k=0, which=0):
        """reductions.cpp:7-114; returns (degrees, cc, edges, changed)"""
        d = np.ascontiguousarray(degrees, dtype=np.uint32).copy()
        cc = C.c_uint32(cover_count)
        e = C.c_uint64(edges)
        ch = self.lib.orc_reduce(C.byref(self._g(csr)), d, C.byref(cc), C.byref(e), int(pvc),
                                 k, best_or_k, which)
        return d, cc.value, e.value, ch

    def should_prune(self, cc, edges, pvc, k, best):
        return bool(self.lib.orc_should_prune(cc, edges, int(pvc), k, best))

    def greedy(self, csr):
        """bounds.cpp:7-19 → (size, cover internal ids)"""
        cov = np.zeros(max(csr.n, 1), np.uint32)
        s = self.lib.orc_greedy(C.byref(self._g(csr)), cov)
        return int(s), cov[:s].tolist()

    def verify_cover(self, csr, cover):
        c = np.ascontiguousarray(cover, dtype=np.uint32)
        if len(c) == 0:
            c = np.zeros(1, np.uint32)
            return bool(self.lib.orc_verify_cover(C.byref(self._g(csr)), c, 0))
        return bool(self.lib.orc_verify_cover(C.byref(self._g(csr)), c, len(cover)))

    def brute_force(self, csr):
        """solver_seq.cpp:173-211 → (size, cover internal ids); ValueError for n > 20"""
        cov = np.zeros(max(csr.n, 1), np.uint32)
        s = self.lib.orc_brute_force(C.byref(self._g(csr)), cov)
        if s == 0xFFFFFFFF:
            raise ValueError("brute force oracle is limited to 20 vertices")
        return int(s), cov[:s].tolist()

    def fingerprint(self, degrees, cc, edges):
        d = np.ascontiguousarray(degrees, dtype=np.uint32)
        return int(self.lib.orc_fingerprint(d, len(d), cc, edges))

    def solve_seq(self, csr, pvc=False, k=0, node_budget=0):
        """solver_seq.cpp:56-159 → dict(size, feasible, status, nodes, cover, ...)"""
        if pvc and k < 1:
            raise ValueError("pvc requires k >= 1")
        r = _OrcResult()
        cov = np.zeros(max(csr.n, 1), np.uint32)
        self.lib.orc_solve_seq(C.byref(self._g(csr)), int(pvc), k, node_budget, C.byref(r), cov)
        return dict(size=r.size, feasible=bool(r.feasible), status=("complete", "", "budget")[r.status],
                    nodes=r.nodes, greedy_size=r.greedy_size, stack_high_water=r.stack_high_water,
                    cover=cov[:r.size].tolist() if r.feasible else [])


class _RefResult(C.Structure):
    _fields_ = [("size", C.c_uint32), ("feasible", C.c_int32), ("status", C.c_int32),
                ("greedy_size", C.c_uint32), ("cover_len", C.c_uint32),
                ("num_workers", C.c_uint32), ("wall_ms", C.c_double),
                ("nodes_total", C.c_uint64), ("wl_added", C.c_uint64),
                ("wl_removed", C.c_uint64), ("wl_max_size", C.c_uint64),
                ("wl_current_size", C.c_uint64), ("stack_high_water", C.c_uint64)]


STRATEGIES = {"seq": 0, "hybrid": 1, "stackonly": 2}
STATUS = ("complete", "timeout", "budget")


class Reference:
    """The reference itself (oracle/_ref/libvcref.so). Raises OSError when it was not built."""

    def __init__(self, path=None):
        path = path or os.path.join(HERE, "_ref", "libvcref.so")
        self.lib = C.CDLL(path)
        L = self.lib
        vp = C.c_void_p
        L.vcref_last_error.restype = C.c_char_p
        L.vcref_graph_from_csr.restype = vp
        L.vcref_graph_from_csr.argtypes = [C.c_uint32, C.c_uint64, U64P, U32P, C.c_uint32]
        L.vcref_make_graph.restype = vp
        L.vcref_make_graph.argtypes = [C.c_uint32, C.c_uint64, U32P]
        L.vcref_parse.restype = vp
        L.vcref_parse.argtypes = [C.c_char_p, C.c_int]
        L.vcref_gen_gnp.restype = vp
        L.vcref_gen_gnp.argtypes = [C.c_uint32, C.c_double, C.c_uint64]
        L.vcref_gen_tree.restype = vp
        L.vcref_gen_tree.argtypes = [C.c_uint32, C.c_uint64]
        L.vcref_complement.restype = vp
        L.vcref_complement.argtypes = [vp]
        L.vcref_graph_free.argtypes = [vp]
        for f in ("vcref_n", "vcref_id_base"):
            getattr(L, f).restype = C.c_uint32
            getattr(L, f).argtypes = [vp]
        L.vcref_m.restype = C.c_uint64
        L.vcref_m.argtypes = [vp]
        L.vcref_csr.argtypes = [vp, U64P, U32P]
        L.vcref_greedy.restype = C.c_uint32
        L.vcref_greedy.argtypes = [vp, U32P]
        L.vcref_brute_force.restype = C.c_uint32
        L.vcref_brute_force.argtypes = [vp, U32P]
        L.vcref_reduce.argtypes = [vp, U32P, C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                                   C.c_int, C.c_uint32, C.c_uint32, C.c_int]
        L.vcref_should_prune.argtypes = [C.c_uint32, C.c_uint64, C.c_int, C.c_uint32, C.c_uint32]
        L.vcref_fingerprint.restype = C.c_uint64
        L.vcref_fingerprint.argtypes = [U32P, C.c_uint32, C.c_uint32, C.c_uint64]
        L.vcref_solve.argtypes = [vp, C.c_int, C.c_uint32, C.c_int, C.c_uint, C.c_uint64,
                                  C.c_double, C.c_uint, C.c_uint64, C.c_double, C.c_uint64,
                                  C.POINTER(_RefResult), U32P, U64P]

    # graph handles ---------------------------------------------------------------------
    def _csr_of(self, h):
        n, m = self.lib.vcref_n(h), self.lib.vcref_m(h)
        off = np.zeros(n + 1, np.uint64)
        nbr = np.zeros(max(2 * m, 1), np.uint32)
        self.lib.vcref_csr(h, off, nbr)
        ib = self.lib.vcref_id_base(h)
        self.lib.vcref_graph_free(h)
        return CSR(n, m, off, nbr[: 2 * m], ib)

    def _handle(self, csr):
        nbr = csr.neighbors if len(csr.neighbors) else np.zeros(1, np.uint32)
        return self.lib.vcref_graph_from_csr(csr.n, csr.m, csr.offsets, nbr, csr.id_base)

    def gnp(self, n, p, seed):
        """testutil.hpp:62-70"""
        return self._csr_of(self.lib.vcref_gen_gnp(n, p, seed))

    def random_tree(self, n, seed):
        """testutil.hpp:73-81"""
        return self._csr_of(self.lib.vcref_gen_tree(n, seed))

    def make_graph(self, n, pairs):
        p = np.ascontiguousarray(np.asarray(pairs, dtype=np.uint32).reshape(-1))
        if len(p) == 0:
            p = np.zeros(2, np.uint32)
            return self._csr_of(self.lib.vcref_make_graph(n, 0, p))
        return self._csr_of(self.lib.vcref_make_graph(n, len(p) // 2, p))

    def parse(self, text, dimacs=False):
        h = self.lib.vcref_parse(text.encode(), int(dimacs))
        if not h:
            raise ValueError(self.lib.vcref_last_error().decode())
        return self._csr_of(h)

    def complement(self, csr):
        h = self._handle(csr)
        out = self._csr_of(self.lib.vcref_complement(h))
        self.lib.vcref_graph_free(h)
        return out

    # algorithm ---------------------------------------------------------------------------
    def greedy(self, csr):
        h = self._handle(csr)
        cov = np.zeros(max(csr.n, 1), np.uint32)
        s = self.lib.vcref_greedy(h, cov)
        self.lib.vcref_graph_free(h)
        return int(s), cov[:s].tolist()

    def brute_force(self, csr):
        h = self._handle(csr)
        cov = np.zeros(max(csr.n, 1), np.uint32)
        s = self.lib.vcref_brute_force(h, cov)
        self.lib.vcref_graph_free(h)
        if s == 0xFFFFFFFF:
            raise ValueError(self.lib.vcref_last_error().decode())
        return int(s), cov[:s].tolist()

    def reduce(self, csr, degrees, cover_count, edges, pvc=False, k=0, best_or_k=0, which=0):
        h = self._handle(csr)
        d = np.ascontiguousarray(degrees, dtype=np.uint32).copy()
        cc = C.c_uint32(cover_count)
        e = C.c_uint64(edges)
        ch = self.lib.vcref_reduce(h, d, C.byref(cc), C.byref(e), int(pvc), k, best_or_k, which)
        self.lib.vcref_graph_free(h)
        return d, cc.value, e.value, ch

    def should_prune(self, cc, edges, pvc, k, best):
        return bool(self.lib.vcref_should_prune(cc, edges, int(pvc), k, best))

    def fingerprint(self, degrees, cc, edges):
        d = np.ascontiguousarray(degrees, dtype=np.uint32)
        return int(self.lib.vcref_fingerprint(d, len(d), cc, edges))

    def solve(self, csr, pvc=False, k=0, strategy="hybrid", workers=4, capacity=4096,
              threshold_fraction=0.5, depth=8, backoff_us=50, timeout_s=None, node_budget=None):
        """bindings.cpp:60-99 dispatch → dict"""
        h = self._handle(csr)
        r = _RefResult()
        cov = np.zeros(max(csr.n, 1), np.uint32)
        wn = np.zeros(max(workers, 1), np.uint64)
        rc = self.lib.vcref_solve(h, int(pvc), k, STRATEGIES[strategy], workers, capacity,
                                  threshold_fraction, depth, backoff_us,
                                  -1.0 if timeout_s is None else float(timeout_s),
                                  node_budget or 0, C.byref(r), cov, wn)
        self.lib.vcref_graph_free(h)
        if rc != 0:
            raise ValueError(self.lib.vcref_last_error().decode())
        return dict(size=r.size if r.feasible else None, feasible=bool(r.feasible),
                    status=STATUS[r.status], greedy_size=r.greedy_size, wall_ms=r.wall_ms,
                    nodes=r.nodes_total, worker_nodes=wn[: r.num_workers].tolist(),
                    cover=cov[: r.cover_len].tolist(),
                    worklist=dict(added=r.wl_added, removed=r.wl_removed,
                                  max_size=r.wl_max_size, current_size=r.wl_current_size),
                    stack_high_water=r.stack_high_water)
