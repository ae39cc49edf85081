"""C4 throughput probe (dev tool): node-budgeted MVC on the BA(100k, 3) graph."""
import json, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
g = load_config("c4")
for budget in [int(x) for x in (sys.argv[1:] or ["2000", "20000", "100000"])]:
    t = time.time()
    r = vc.solve_mvc(g, strategy="gpu", node_budget=budget)
    print(json.dumps(dict(budget=budget, nodes=r["nodes_total"], size=r["size"], status=r["status"],
        device_ms=round(r["device_ms"], 1), wall_ms=round(r["wall_ms"], 1), greedy_ms=round(r["greedy_ms"], 1),
        knps=round(r["nodes_total"] / r["device_ms"], 1), rounds=r["rounds"], children=r["children"],
        rm=(r["removals_deg1"], r["removals_deg2"], r["removals_high"]), donated=r["donated"],
        hw=max(r["worker_stack_high_water"]), workers=len(r["worker_nodes"]),
        from_search=r["cover_from_search"])), flush=True)
