"""Instrumented C5 solve: per-phase shares of worker time (Fig. 6 analogue) and load ratios."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
g = load_config(sys.argv[1] if len(sys.argv) > 1 else "c5")
k = int(sys.argv[2]) if len(sys.argv) > 2 else 482
for _ in range(2):
    r = vc.solve_pvc(g, k, strategy="gpu", instrument=True)
print(json.dumps(dict(device_ms=r["device_ms"], nodes=r["nodes_total"], phase_shares=r.get("phase_shares"),
                      load_ratio_max=max(r["load_ratios"]),
                      )))
