"""Paper-analog comparison on C5 k=482 (Hybrid vs StackOnly): device time and
load ratios per strategy on the whole device."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
g = load_config("c5")
runs = [("gpu (hybrid, oldest donation)", dict(strategy="gpu")),
        ("hybrid (reference donation policy)", dict(strategy="hybrid", workers=3552)),
        ("stackonly depth 12", dict(strategy="stackonly", workers=3552, depth=12)),
        ("stackonly depth 16", dict(strategy="stackonly", workers=3552, depth=16))]
for label, kw in runs:
    try:
        for _ in range(2):
            r = vc.solve_pvc(g, 482, timeout_s=30, **kw)
        lr = r.get("load_ratios") or [0]
        print(json.dumps(dict(label=label, status=r["status"], nodes=r["nodes_total"], device_ms=round(r["device_ms"], 2),
                              load_ratio_max=round(max(lr), 2), workers=len(r["worker_nodes"]))), flush=True)
    except Exception as e:
        print(json.dumps(dict(label=label, error=str(e))), flush=True)
