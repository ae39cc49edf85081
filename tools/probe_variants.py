"""Variant sweep on one config (dev tool): capacity / threshold / donation / instrumentation."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 482
g = load_config(name)
vc.solve_pvc(g, k, strategy="gpu")  # warm
variants = [
    dict(),
    dict(instrument=True),
    dict(donate_oldest=False),
    dict(capacity=4096, threshold_fraction=0.5, instrument=True),
    dict(capacity=4096, threshold_fraction=0.5),
    dict(capacity=4096, threshold_fraction=0.5, donate_oldest=True),
    dict(capacity=4096, threshold_fraction=0.5, donate_oldest=True, instrument=True),
    dict(capacity=131072, threshold_fraction=0.5),
    dict(capacity=131072, threshold_fraction=0.5, donate_oldest=True),
    dict(capacity=131072, threshold_fraction=1.0, donate_oldest=True),
    dict(capacity=16384, threshold_fraction=0.25, donate_oldest=True),
    dict(capacity=4096, threshold_fraction=0.5, donate_oldest=True, block_warps=4),
]
for kw in variants:
    r = vc.solve_pvc(g, k, strategy="gpu", **kw)
    sh = {kk: round(v, 3) for kk, v in r["phase_shares"].items() if v > 0.001}
    print(json.dumps(dict(kw=kw, nodes=r["nodes_total"], feasible=r["feasible"],
                          dev_ms=round(r["device_ms"], 1), mnps=round(r["nodes_total"]/r["device_ms"]/1e3, 1),
                          donated=r["donated"], rm=(r["removals_deg1"], r["removals_deg2"], r["removals_high"]),
                          dooms=r["doomed"], rounds=r["rounds"], children=r["children"], maxq=r["worklist"]["max_size"],
                          workers=len(r["worker_nodes"]), grid=r["grid_blocks"],
                          minload=round(min(r["load_ratios"]), 3), maxload=round(max(r["load_ratios"]), 3),
                          shares=sh)), flush=True)
