"""Run report assembly: make_report (report.cpp:161-185) + collect_metrics (metrics.cpp:23-67).

The dict carries exactly the keys of the reference's report_to_dict (bindings.cpp:32-58), plus
engine extras (worklist stats as RunReport::worklist, device timing, roofline counters).
"""
from __future__ import annotations

PHASE_KEYS = (  # Phase order + phase_key (metrics.hpp:15-26, metrics.cpp:7-21)
    "worklist_remove", "worklist_add", "stack_ops", "reduce_degree_one",
    "reduce_degree_two_triangle", "reduce_high_degree", "max_degree_scan",
    "branch_remove_neighbors", "branch_remove_vertex", "prune_check",
)


def collect_metrics(worker_nodes, phase_cycles, active_cycles):
    """Load ratios = count / mean (1.0 everywhere if the mean is 0); phase shares = share of the
    workers' active cycles per phase, plus "other" (metrics.cpp:23-67). The device sums cycles
    over workers, so the share is the cycle-weighted mean of per-worker shares."""
    import numpy as np
    wn = np.asarray(worker_nodes, dtype=np.float64)  # (thousands of device workers)
    mean = float(wn.mean()) if len(wn) else 0.0
    ratios = (wn / mean).tolist() if mean > 0 else [1.0] * len(wn)
    shares = {}
    if active_cycles > 0:
        tracked = 0.0
        for key, cyc in zip(PHASE_KEYS, phase_cycles):
            s = cyc / active_cycles
            shares[key] = s
            tracked += s
        shares["other"] = 0.0 if tracked >= 1.0 else 1.0 - tracked
    else:
        shares = {key: 0.0 for key in PHASE_KEYS}
        shares["other"] = 1.0
    return ratios, shares


def make_report(graph, mode, k, strategy, workers, capacity, threshold_fraction, depth, res):
    ratios, shares = collect_metrics(res.get("_worker_nodes_np", res["worker_nodes"]),
                                     res["phase_cycles"], res["active_cycles"])
    rep = {
        "n": graph.num_vertices,
        "m": graph.num_edges,
        "mode": mode,
        "k": k if mode == "pvc" else None,
        "strategy": strategy,
        "workers": len(res["worker_nodes"]) if strategy in ("gpu", "seq") else workers,
        "capacity": capacity,
        "threshold_fraction": threshold_fraction,
        "depth": depth,
        "size": res["size"] if res["feasible"] else None,
        "feasible": res["feasible"],
        "cover": res["cover"],
        "wall_ms": res["wall_ms"],
        "status": res["status"],
        "worker_nodes": res["worker_nodes"],
        "load_ratios": ratios,
        "phase_shares": shares,
    }
    # engine extras (not in the reference dict; additive)
    rep["worklist"] = res["worklist"]
    for key in ("nodes_total", "greedy_size", "device_ms", "greedy_ms", "h2d_ms", "h2d_bytes",
                "d2h_bytes", "rounds", "maxdeg_passes", "children", "removals", "donated", "removals_deg1", "removals_deg2", "removals_high", "doomed",
                "degree_bytes",
                "n_padded", "engine", "grid_blocks", "block_threads", "kernel_launches", "cover_from_search",
                "worker_stack_high_water", "certify_nodes", "certify_ms", "timeline"):
        rep[key] = res[key]
    return rep
