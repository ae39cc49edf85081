"""Pick a C5-scale instance: for each candidate p_hat-style graph (DIMACS,
solved on its complement), the GPU MVC (with a timeout), then PVC(MVC - 1) and PVC(MVC) times.

usage: python tools/probe_scale.py TIMEOUT_S FILE.clq [FILE.clq ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc  # noqa: E402

t = float(sys.argv[1])
for path in sys.argv[2:]:
    g = vc.load_graph(path, complement_input=True)
    r = vc.solve_mvc(g, strategy="gpu", timeout_s=t, capacity=1 << 16)
    rec = dict(file=os.path.basename(path), n=g.num_vertices, m=g.num_edges,
               greedy=r["greedy_size"], mvc=r["size"], status=r["status"],
               nodes=r["nodes_total"], device_s=r["device_ms"] / 1e3,
               valid=vc.verify_cover(g, r["cover"]))
    print(json.dumps(rec), flush=True)
    if r["status"] != "complete":
        continue
    for k in (r["size"] - 1, r["size"]):
        p = vc.solve_pvc(g, k, strategy="gpu", timeout_s=t)
        print(json.dumps(dict(file=rec["file"], k=k, feasible=p["feasible"], status=p["status"],
                              nodes=p["nodes_total"], device_s=p["device_ms"] / 1e3,
                              valid=(vc.verify_cover(g, p["cover"]) if p["feasible"] else None))),
              flush=True)
