import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
g = load_config("c2")
r = vc.solve_pvc(g, 240, strategy="gpu", timeout_s=float(sys.argv[1]) if len(sys.argv) > 1 else 1.0, instrument=len(sys.argv) > 2)
print(r["nodes_total"], r["device_ms"], r["nodes_total"] / r["device_ms"] / 1e3, "Mn/s", "rounds", r["rounds"], "rm", r["removals_deg1"], r["removals_deg2"], r["removals_high"], "children", r["children"], "dooms", r["doomed"])
print({k: round(v, 3) for k, v in r["phase_shares"].items()})
