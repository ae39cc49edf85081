mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g5_pytest.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/g5_pytest.log
timeout 300 python tools/probe_c4.py 2000 20000 100000 > gpurun_out/g5_c4.jsonl 2>&1
cat gpurun_out/g5_c4.jsonl
timeout 900 python tools/probe_ab.py auto data/cand/phat500_0.45_1.0.clq:0 2>&1 | head -0
timeout 1200 python tools/probe_scale.py 60 data/cand/phat500_0.45_1.0.clq data/cand/phat500_0.4_1.0.clq data/cand/phat500_0.45_0.95.clq data/cand/phat500_0.5_0.95.clq > gpurun_out/g5_scale.jsonl 2>&1
cat gpurun_out/g5_scale.jsonl
