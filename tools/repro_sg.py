"""Repro: the sparse engine's global-memory variant on a small graph (fuzz graph 89, seed 11)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc  # noqa: E402
g = vc.parse_edge_list(open(sys.argv[1]).read())
eng = sys.argv[2] if len(sys.argv) > 2 else "sparse-global"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
bw = int(sys.argv[4]) if len(sys.argv) > 4 else 0
cap = int(sys.argv[5]) if len(sys.argv) > 5 else 4096
for i in range(reps):
    r = vc.solve_mvc(g, strategy="gpu", engine=eng, block_warps=bw, capacity=cap)
    print(i, r["size"], r["status"], r["nodes_total"], len(r["worker_nodes"]), r["block_threads"], flush=True)
