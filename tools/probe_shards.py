"""GPU probe: multi-shard solves on one device (C5 k=482) vs the single-shard solve."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
from paper_2204_10402_b200.shards import solve_sharded
g = load_config("c5")
r = vc.solve_pvc(g, 482, strategy="gpu")
print("single", r["nodes_total"], round(r["device_ms"], 2))
for devs, skew, fps, frac in [((0,), False, 0, 0.5), ((0, 0), False, 0, 0.5), ((0, 0), False, 256, 0.5),
                              ((0, 0), True, 256, 0.5), ((0, 0, 0, 0), False, 0, 0.5),
                              ((0,) * 8, False, 0, 0.5)]:
    for _ in range(2):
        r = solve_sharded(g, "pvc", 482, devices=devs, skew=skew, frontier_per_shard=fps, threshold_fraction=frac)
    print(json.dumps(dict(devs=len(devs), skew=skew, fps=fps, frac=frac, nodes=r["nodes_total"], rank_nodes=r["rank_nodes"],
          ms=[round(x, 2) for x in r["rank_device_ms"]], don=r["rank_donated"], peer=r["rank_donated_peer"],
          wall=round(r["wall_ms"], 1))), flush=True)
