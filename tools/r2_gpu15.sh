mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ipc.py -m gpu -x -q -k "shard or ipc or persistent or fill or c5" > gpurun_out/g15_pytest.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/g15_pytest.log
timeout 300 python -c "
import sys, json; sys.path.insert(0, '.')
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
for name, k in (('c5', 482), ('c1', 84), ('c5s', 448)):
    g = load_config(name)
    for _ in range(2):
        r = vc.solve_pvc(g, k, strategy='gpu')
    print(json.dumps(dict(cfg=name, ms=round(r['device_ms'], 3), nodes=r['nodes_total'], timeline=r['timeline'])), flush=True)
" > gpurun_out/g15_timeline.jsonl 2>&1; cat gpurun_out/g15_timeline.jsonl
timeout 600 bash tools/ab_shards_scale.sh data/cand/phat500_0.48_1.0.clq 448 > gpurun_out/g15_shards.txt 2>&1; cat gpurun_out/g15_shards.txt
timeout 300 bash tools/ab_shards.sh > gpurun_out/g15_shards_c5.txt 2>&1; cat gpurun_out/g15_shards_c5.txt
