mkdir -p gpurun_out
timeout 1200 bash tools/ab_shards_scale.sh data/cand/phat500_0.48_1.0.clq 448 gpuacq minb3 > gpurun_out/g13_shards.txt 2>&1; cat gpurun_out/g13_shards.txt
timeout 300 python -c "
import sys, json; sys.path.insert(0, '.')
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
g = load_config('c5s')
for dw in (None, 2368, 1776):
    r = vc.solve_pvc(g, 448, strategy='gpu', **({} if dw is None else dict(workers=dw)))
    print(json.dumps(dict(warps=len(r['worker_nodes']), ms=round(r['device_ms'], 1), nodes=r['nodes_total'])), flush=True)
" > gpurun_out/g13_warps.jsonl 2>&1; cat gpurun_out/g13_warps.jsonl
