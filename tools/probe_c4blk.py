"""C4: the global-memory node variant at several CTA sizes (dev tool)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc  # noqa: E402
from paper_2204_10402_b200.configs import load_config  # noqa: E402
g = load_config("c4")
for bw in (4, 8, 16):
    vc.solve_mvc(g, strategy="gpu", node_budget=2000, engine="sparse-global", block_warps=bw)
    for b in (20000, 100000):
        r = vc.solve_mvc(g, strategy="gpu", node_budget=b, engine="sparse-global", block_warps=bw)
        s = r["device_ms"] / 1e3
        print(json.dumps(dict(block=r["block_threads"], workers=len(r["worker_nodes"]), budget=b,
                              device_ms=round(r["device_ms"], 1), knodes_per_s=round(r["nodes_total"] / s / 1e3, 1),
                              krounds_per_s=round(r["rounds"] / s / 1e3, 1),
                              rounds_per_node=round(r["rounds"] / r["nodes_total"], 1))), flush=True)
