"""A/B probe: PVC no-instance node counts and device time per engine variant (dev tool).

usage: python tools/probe_ab.py ENGINE[,ENGINE...] SPEC [SPEC ...]
SPEC = c5 | c2:SECONDS | FILE.clq:K  (FILE solved on its complement)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc  # noqa: E402
from paper_2204_10402_b200.configs import load_config  # noqa: E402

engines = sys.argv[1].split(",")
for spec in sys.argv[2:]:
    t = None
    if spec == "c5":
        g, k = load_config("c5"), 482
    elif spec.startswith("c2"):
        g, k, t = load_config("c2"), 240, float(spec.split(":")[1])
    else:
        f, k = spec.rsplit(":", 1)
        g, k = vc.load_graph(f, complement_input=True), int(k)
    for eng in engines:
        for rep in range(2):
            r = vc.solve_pvc(g, k, strategy="gpu", engine=eng, timeout_s=t)
            print(json.dumps(dict(spec=spec, engine=eng, rep=rep, status=r["status"], feasible=r["feasible"],
                                  nodes=r["nodes_total"], device_ms=round(r["device_ms"], 3),
                                  mnps=round(r["nodes_total"] / r["device_ms"] / 1e3, 1),
                                  rounds=r["rounds"], children=r["children"])), flush=True)
