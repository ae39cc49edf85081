"""C2 per-phase shares (instrumented) and node rate over a bounded PVC(240) run (dev tool)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc  # noqa: E402
from paper_2204_10402_b200.configs import load_config  # noqa: E402

g = load_config("c2")
t = float(sys.argv[1]) if len(sys.argv) > 1 else 10
for eng in ("auto", "dense-wide"):
    for instr in (False, True):
        r = vc.solve_pvc(g, 240, strategy="gpu", timeout_s=t, instrument=instr, engine=eng)
        print(json.dumps(dict(engine=eng, instrument=instr, status=r["status"], nodes=r["nodes_total"],
                              device_s=r["device_ms"] / 1e3, mnps=r["nodes_total"] / r["device_ms"] / 1e3,
                              rounds=r["rounds"], children=r["children"], rm1=r["removals_deg1"],
                              rm2=r["removals_deg2"], rmh=r["removals_high"], doomed=r["doomed"],
                              phase_shares=r.get("phase_shares") if instr else None)), flush=True)
