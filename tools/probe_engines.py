"""GPU probe: C1/C3/C5 through the public API with the compact layout on and off."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config

engines = sys.argv[1:] or ["dense", "dense-wide"]
for name, mode, k in [("c1", "mvc", None), ("c1", "pvc", 84), ("c3", "mvc", None), ("c3", "pvc", 290),
                      ("c5", "pvc", 483), ("c5", "pvc", 482), ("c5", "pvc", 482)]:
    g = load_config(name)
    for e in engines:
        r = vc.solve_mvc(g, strategy="gpu", engine=e) if mode == "mvc" else vc.solve_pvc(g, k, strategy="gpu", engine=e)
        ok = r["cover"] is None or vc.verify_cover(g, r["cover"])
        print(json.dumps(dict(cfg=name, mode=mode, k=k, engine=e, size=r["size"], feasible=r["feasible"],
                              nodes=r["nodes_total"], device_ms=round(r["device_ms"], 3), cover_ok=ok,
                              rounds=r["rounds"], children=r["children"])), flush=True)
for e in engines:  # seq order (1 warp): node counts equal the reference's
    g = load_config("c1")
    r = vc.solve_mvc(g, strategy="seq", engine=e)
    print(json.dumps(dict(cfg="c1", mode="mvc-seq", engine=e, size=r["size"], nodes=sum(r["worker_nodes"]))), flush=True)
