mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/g1_pytest.log
timeout 300 python tools/probe.py c1 c3 c5 > gpurun_out/g1_probe.jsonl 2>&1
timeout 400 python tools/probe_c2.py 300 241 > gpurun_out/g1_c2.jsonl 2>&1
timeout 900 python tools/fuzz_parity.py 780 7 > gpurun_out/g1_fuzz.jsonl 2>&1
tail -2 gpurun_out/g1_fuzz.jsonl
cat gpurun_out/g1_probe.jsonl gpurun_out/g1_c2.jsonl
