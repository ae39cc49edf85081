mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g18_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/g18_pytest.log
timeout 300 python tools/probe_ab.py auto c2:5 > gpurun_out/g18_c2.jsonl 2>&1; cat gpurun_out/g18_c2.jsonl
timeout 300 python -c "
import sys, json; sys.path.insert(0, '.')
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
for name, k in (('c5', 482), ('c1', 84), ('c5s', 448)):
    g = load_config(name)
    for _ in range(2):
        r = vc.solve_pvc(g, k, strategy='gpu')
    print(json.dumps(dict(cfg=name, ms=round(r['device_ms'], 3), nodes=r['nodes_total'], timeline=r['timeline'])), flush=True)
" > gpurun_out/g18_timeline.jsonl 2>&1; cat gpurun_out/g18_timeline.jsonl
timeout 600 python tools/probe_c4ab.py sparse,sparse-global 20000 100000 > gpurun_out/g18_c4ab.jsonl 2>&1; cat gpurun_out/g18_c4ab.jsonl
