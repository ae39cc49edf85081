"""C2 (ER n=400, avg deg 6): try to establish the MVC on the GPU (dev tool)."""
import json, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
g = load_config("c2")
t = float(sys.argv[1]) if len(sys.argv) > 1 else 120
r = vc.solve_mvc(g, strategy="gpu", timeout_s=t, capacity=1 << 17)
print(json.dumps(dict(what="mvc", size=r["size"], status=r["status"], nodes=r["nodes_total"],
    device_s=r["device_ms"] / 1e3, mnps=r["nodes_total"] / r["device_ms"] / 1e3,
    greedy=r["greedy_size"], from_search=r["cover_from_search"], valid=vc.verify_cover(g, r["cover"]))), flush=True)
for k in [int(x) for x in sys.argv[2:]]:
    r = vc.solve_pvc(g, k, strategy="gpu", timeout_s=t, capacity=1 << 17)
    print(json.dumps(dict(what="pvc", k=k, feasible=r["feasible"], status=r["status"], nodes=r["nodes_total"],
        device_s=r["device_ms"] / 1e3, mnps=r["nodes_total"] / r["device_ms"] / 1e3)), flush=True)
