"""C4 sparse-engine A/B (dev tool): per-node cost in the deterministic seq order, and budgeted
full-device runs compared by their rule-round rate (node rates are schedule-dependent on C4).

usage: python tools/probe_c4ab.py ENGINE[,ENGINE...] [BUDGET ...]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc  # noqa: E402
from paper_2204_10402_b200.configs import load_config  # noqa: E402

g = load_config("c4")
engines = sys.argv[1].split(",")
budgets = [int(x) for x in sys.argv[2:]] or [20000, 100000]
for eng in engines:
    r = vc.solve_mvc(g, strategy="seq", node_budget=300, engine=eng)
    print(json.dumps(dict(engine=eng, mode="seq300", device_ms=round(r["device_ms"], 2),
                          us_per_node=round(1e3 * r["device_ms"] / r["nodes_total"], 1))), flush=True)
    vc.solve_mvc(g, strategy="gpu", node_budget=2000, engine=eng)
    for b in budgets:
        r = vc.solve_mvc(g, strategy="gpu", node_budget=b, engine=eng)
        s = r["device_ms"] / 1e3
        alg = 2 * g.num_vertices * (r["rounds"] + r["maxdeg_passes"] + r["children"])
        print(json.dumps(dict(engine=eng, budget=b, workers=len(r["worker_nodes"]), block=r["block_threads"],
                              device_ms=round(r["device_ms"], 1), knodes_per_s=round(r["nodes_total"] / s / 1e3, 1),
                              krounds_per_s=round(r["rounds"] / s / 1e3, 1), rounds_per_node=round(r["rounds"] / r["nodes_total"], 1),
                              alg_gbs=round(alg / s / 1e9, 1), size=r["size"])), flush=True)
