"""Long attempt at C2's PVC k=240 (is MVC(C2) = 241?) on one GPU."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
g = load_config("c2")
t = float(sys.argv[1])
r = vc.solve_pvc(g, 240, strategy="gpu", timeout_s=t)
out = dict(k=240, feasible=r["feasible"], status=r["status"], nodes=r["nodes_total"],
           device_s=r["device_ms"] / 1e3, cover_valid=vc.verify_cover(g, r["cover"]) if r["feasible"] else None,
           size=r["size"])
print(json.dumps(out), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/c2_k240.json", "w"))
