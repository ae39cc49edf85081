"""Deterministic C4 per-node cost (dev tool): the one-CTA seq order visits the same nodes in every
build (block-parallel rules reach a schedule-independent fixpoint), so device time per node is
an A/B measure free of the schedule noise of budgeted full-device runs."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc  # noqa: E402
from paper_2204_10402_b200.configs import load_config  # noqa: E402
g = load_config("c4")
for budget in [int(x) for x in (sys.argv[1:] or ["300"])]:
    for rep in range(2):
        r = vc.solve_mvc(g, strategy="seq", node_budget=budget)
        print(json.dumps(dict(budget=budget, nodes=r["nodes_total"], device_ms=round(r["device_ms"], 2),
                              us_per_node=round(1e3 * r["device_ms"] / max(1, r["nodes_total"]), 1),
                              rounds=r["rounds"], rm=(r["removals_deg1"], r["removals_deg2"], r["removals_high"]),
                              children=r["children"])), flush=True)
