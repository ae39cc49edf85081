mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g6_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/g6_pytest.log
timeout 1500 python tools/probe_ab.py auto,dense-mid4,dense-mid8 c5 c2:5 data/cand/phat500_0.45_1.0.clq:449 data/cand/phat500_0.5_1.0.clq:448 > gpurun_out/g6_ab.jsonl 2>&1
cat gpurun_out/g6_ab.jsonl
