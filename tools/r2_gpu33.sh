mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/g33_pytest.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/g33_pytest.log
timeout 1800 python tools/fuzz_parity.py 1560 11 > gpurun_out/r2_fuzz_parity_final.jsonl 2> gpurun_out/g33_fuzz.err; echo fuzz_rc=$?
tail -2 gpurun_out/r2_fuzz_parity_final.jsonl; tail -3 gpurun_out/g33_fuzz.err
