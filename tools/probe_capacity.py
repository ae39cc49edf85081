"""C5 device time against the worklist capacity / donation threshold (dev tool)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc  # noqa: E402
from paper_2204_10402_b200.configs import load_config  # noqa: E402
g = load_config(sys.argv[1] if len(sys.argv) > 1 else "c5")
k = int(sys.argv[2]) if len(sys.argv) > 2 else 482
for rep in range(2):
    for cap, frac in ((4096, 0.5), (8192, 0.5), (16384, 0.5), (8192, 0.25), (16384, 0.25), (4096, 1.0)):
        r = vc.solve_pvc(g, k, strategy="gpu", capacity=cap, threshold_fraction=frac)
        print(json.dumps(dict(cap=cap, frac=frac, ms=round(r["device_ms"], 3), nodes=r["nodes_total"],
                              idle=round(r["timeline"]["idle_share"], 4), donated=r["donated"])), flush=True)
