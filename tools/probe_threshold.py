"""C5 k=482 device time against the worklist capacity / donation threshold (strategy gpu)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
g = load_config("c5")
for cap, frac in [(4096, 0.5), (4096, 0.25), (4096, 1.0), (8192, 0.5), (2048, 0.5), (4096, 0.5)]:
    ms = []
    for _ in range(3):
        r = vc.solve_pvc(g, 482, strategy="gpu", capacity=cap, threshold_fraction=frac)
        assert r["nodes_total"] == 21461369
        ms.append(r["device_ms"])
    print(json.dumps(dict(cap=cap, frac=frac, ms=[round(x, 2) for x in ms], donated=r["donated"],
                          load_ratio=round(max(r["load_ratios"]), 2))), flush=True)
