mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g4_pytest.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/g4_pytest.log
timeout 900 python tools/probe_ab.py auto,dense-nomid c5 c2:5 data/cand/phat500_0.35_0.95.clq:466 data/cand/phat500_0.5_1.0.clq:448 > gpurun_out/g4_ab.jsonl 2>&1
cat gpurun_out/g4_ab.jsonl
