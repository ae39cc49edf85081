"""Quick GPU probe: times the configs through the public API (not the bench)."""
import json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config

def run(label, fn):
    t = time.time(); r = fn(); dt = time.time() - t
    print(json.dumps(dict(label=label, size=r["size"], feasible=r["feasible"], status=r["status"],
          nodes=r["nodes_total"], wall_ms=round(r["wall_ms"], 2), device_ms=round(r["device_ms"], 2),
          workers=len(r["worker_nodes"]), grid=r["grid_blocks"], rounds=r["rounds"], children=r["children"],
          mnodes_per_s=round(r["nodes_total"] / max(r["device_ms"], 1e-9) / 1e3, 2), py_s=round(dt, 3),
          greedy_ms=round(r["greedy_ms"], 3), h2d_ms=round(r["h2d_ms"], 3))), flush=True)
    return r

which = sys.argv[1:] or ["c1", "c3", "c5"]
for name in which:
    g = load_config(name)
    if name == "c1":
        run("c1 mvc gpu", lambda: vc.solve_mvc(g, strategy="gpu"))
        run("c1 mvc gpu", lambda: vc.solve_mvc(g, strategy="gpu"))
        run("c1 pvc84 gpu", lambda: vc.solve_pvc(g, 84, strategy="gpu"))
        run("c1 mvc seq", lambda: vc.solve_mvc(g, strategy="seq"))
    if name == "c3":
        run("c3 mvc gpu", lambda: vc.solve_mvc(g, strategy="gpu"))
        run("c3 pvc290 gpu", lambda: vc.solve_pvc(g, 290, strategy="gpu"))
    if name == "c5":
        run("c5 pvc483 gpu", lambda: vc.solve_pvc(g, 483, strategy="gpu"))
        run("c5 pvc482 gpu", lambda: vc.solve_pvc(g, 482, strategy="gpu"))
        run("c5 pvc482 gpu", lambda: vc.solve_pvc(g, 482, strategy="gpu"))
    if name == "c5" :
        run("c5 mvc gpu", lambda: vc.solve_mvc(g, strategy="gpu"))
    if name == "c5mvc":
        run("c5 mvc gpu", lambda: vc.solve_mvc(load_config("c5"), strategy="gpu"))
    if name == "c2":
        run("c2 mvc gpu 60s", lambda: vc.solve_mvc(g, strategy="gpu", timeout_s=60))
