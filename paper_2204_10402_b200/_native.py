"""ctypes binding of libvcgpu.so — the C-ABI declared in include/vcgpu.h.

The library is the product: there is no Python or CPU fallback. Importing this module fails
loudly (ImportError) when the shared library has not been built, and every solve fails loudly
(RuntimeError) when no CUDA device is visible.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VCGPU_LIB", os.path.join(_HERE, "libvcgpu.so"))

VCG_OK, VCG_EINVAL, VCG_EPARSE, VCG_ECUDA, VCG_ENOMEM, VCG_ERANGE, VCG_EVERIFY = range(7)
VCG_DEBUG_CERTIFY, VCG_DEBUG_CORRUPT_COVER, VCG_DEBUG_SMALL_STACK = 1, 2, 4
VCG_MVC, VCG_PVC = 0, 1
VCG_HYBRID, VCG_SEQ, VCG_STACKONLY = 0, 1, 2
STATUS_NAMES = ("complete", "timeout", "budget")  # run_status_name (solver_seq.cpp:15-22)


class Params(C.Structure):
    """vcg_params (include/vcgpu.h)."""

    _fields_ = [
        ("mode", C.c_int32), ("k", C.c_uint32), ("strategy", C.c_int32),
        ("workers", C.c_uint32), ("capacity", C.c_uint64), ("threshold_fraction", C.c_double),
        ("depth", C.c_uint32), ("backoff_us", C.c_uint64), ("timeout_s", C.c_double),
        ("node_budget", C.c_uint64), ("device", C.c_int32), ("rules", C.c_int32),
        ("block_warps", C.c_uint32), ("engine", C.c_int32), ("instrument", C.c_int32),
        ("donate_oldest", C.c_int32),
        ("initial_best", C.c_uint32), ("num_seeds", C.c_uint64),
        ("seeds", C.POINTER(C.c_uint32)), ("mailbox", C.POINTER(C.c_uint32)),
        ("stream", C.c_void_p), ("debug_flags", C.c_uint32),
        ("device_workers", C.c_uint32),
    ]


class Result(C.Structure):
    """vcg_result (include/vcgpu.h)."""

    _fields_ = [
        ("status", C.c_int32), ("size", C.c_uint32), ("feasible", C.c_int32),
        ("greedy_size", C.c_uint32), ("cover_len", C.c_uint32),
        ("cover", C.POINTER(C.c_uint32)), ("cover_from_search", C.c_int32),
        ("num_workers", C.c_uint32), ("worker_nodes", C.POINTER(C.c_uint64)),
        ("worker_stack_high_water", C.POINTER(C.c_uint64)), ("nodes_total", C.c_uint64),
        ("wl_added", C.c_uint64), ("wl_removed", C.c_uint64), ("wl_max_size", C.c_uint64),
        ("wl_current_size", C.c_uint64), ("wall_ms", C.c_double), ("device_ms", C.c_double),
        ("greedy_ms", C.c_double), ("h2d_ms", C.c_double), ("h2d_bytes", C.c_uint64),
        ("d2h_bytes", C.c_uint64), ("rounds", C.c_uint64), ("maxdeg_passes", C.c_uint64),
        ("children", C.c_uint64), ("removals", C.c_uint64), ("donated", C.c_uint64),
        ("removals_deg1", C.c_uint64), ("removals_deg2", C.c_uint64),
        ("removals_high", C.c_uint64), ("doomed", C.c_uint64),
        ("degree_bytes", C.c_uint32),
        ("n_padded", C.c_uint32), ("engine", C.c_int32), ("grid_blocks", C.c_uint32),
        ("block_threads", C.c_uint32), ("kernel_launches", C.c_uint32),
        ("phase_cycles", C.c_uint64 * 10),
        ("active_cycles", C.c_uint64), ("donated_peer", C.c_uint64),
        ("certify_nodes", C.c_uint64), ("certify_ms", C.c_double),
        ("certify_launches", C.c_uint32),
        ("t_first_ms", C.c_double * 4), ("t_end_ms", C.c_double * 4), ("idle_share", C.c_double),
        ("t_lastwait_ms", C.c_double * 4),
    ]


class Frontier(C.Structure):
    """vcg_frontier (include/vcgpu.h)."""

    _fields_ = [
        ("num_seeds", C.c_uint64), ("seeds", C.POINTER(C.c_uint32)),
        ("nodes_visited", C.c_uint64), ("levels", C.c_uint32), ("best", C.c_uint32),
        ("greedy_size", C.c_uint32), ("found", C.c_int32), ("cover_len", C.c_uint32),
        ("cover", C.POINTER(C.c_uint32)), ("kernel_launches", C.c_uint32),
    ]


# (name, restype, argtypes) for every symbol include/vcgpu.h declares
_VP = C.c_void_p
_SIGS = [
    ("vcg_graph_from_csr", C.c_int, [C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint32, C.POINTER(_VP)]),
    ("vcg_make_graph", C.c_int, [C.c_uint32, C.c_uint64, C.c_void_p, C.c_uint32, C.POINTER(_VP)]),
    ("vcg_parse_edge_list", C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(_VP)]),
    ("vcg_parse_dimacs", C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(_VP)]),
    ("vcg_complement", C.c_int, [_VP, C.POINTER(_VP)]),
    ("vcg_write_edge_list", C.c_int, [_VP, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]),
    ("vcg_free_buffer", None, [C.c_void_p]),
    ("vcg_graph_destroy", None, [_VP]),
    ("vcg_graph_num_vertices", C.c_uint32, [_VP]),
    ("vcg_graph_num_edges", C.c_uint64, [_VP]),
    ("vcg_graph_id_base", C.c_uint32, [_VP]),
    ("vcg_graph_offsets", C.c_void_p, [_VP]),
    ("vcg_graph_neighbors", C.c_void_p, [_VP]),
    ("vcg_has_edge", C.c_int, [_VP, C.c_uint32, C.c_uint32]),
    ("vcg_graph_equal", C.c_int, [_VP, _VP]),
    ("vcg_check_invariants", C.c_int, [_VP]),
    ("vcg_greedy", C.c_int, [_VP, C.POINTER(C.c_uint32), C.c_void_p]),
    ("vcg_brute_force", C.c_int, [_VP, C.POINTER(C.c_uint32), C.c_void_p]),
    ("vcg_verify_cover", C.c_int, [_VP, C.c_void_p, C.c_uint32, C.POINTER(C.c_int)]),
    ("vcg_params_init", None, [C.POINTER(Params)]),
    ("vcg_solve", C.c_int, [_VP, C.POINTER(Params), C.POINTER(Result)]),
    ("vcg_result_free", None, [C.POINTER(Result)]),
    ("vcg_expand_frontier", C.c_int, [_VP, C.POINTER(Params), C.c_uint64, C.POINTER(Frontier)]),
    ("vcg_frontier_free", None, [C.POINTER(Frontier)]),
    ("vcg_session_open", C.c_int, [_VP, C.POINTER(Params), C.c_int, C.POINTER(_VP)]),
    ("vcg_session_handle_bytes", C.c_size_t, []),
    ("vcg_session_export", C.c_int, [_VP, C.c_void_p]),
    ("vcg_session_link_ipc", C.c_int, [_VP, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]),
    ("vcg_session_link_local", C.c_int, [C.c_void_p, C.c_uint32]),
    ("vcg_session_launch", C.c_int, [_VP]),
    ("vcg_session_reset", C.c_int, [_VP]),
    ("vcg_session_wait", C.c_int, [_VP, C.POINTER(Result)]),
    ("vcg_session_close", None, [_VP]),
    ("vcg_device_workers", C.c_int, [_VP, C.c_int32, C.POINTER(C.c_uint32)]),
    ("vcg_mailbox_alloc", C.c_int, [C.c_uint32, C.POINTER(C.POINTER(C.c_uint32))]),
    ("vcg_mailbox_free", None, [C.POINTER(C.c_uint32)]),
    ("vcg_device_count", C.c_int, []),
    ("vcg_last_error", C.c_char_p, []),
    ("vcg_version", C.c_char_p, []),
]
EXPORTS = [s[0] for s in _SIGS]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
            "this package has no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in _SIGS:
        if "VCGPU_LIB" in os.environ and not hasattr(lib, name):
            continue  # an older library under A/B test
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


class ParseError(ValueError):
    """vcsolve.ParseError (graph.hpp:17-26); a ValueError, as pybind11 registers it
    (bindings.cpp:106)."""


def check(rc):
    """Map a status code to the exception the reference's Python binding raises."""
    if rc == VCG_OK:
        return
    msg = lib.vcg_last_error().decode(errors="replace")
    if rc == VCG_EPARSE:
        raise ParseError(msg)
    if rc in (VCG_EINVAL, VCG_ERANGE):
        raise ValueError(msg)
    if rc == VCG_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)
