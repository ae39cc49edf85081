mkdir -p gpurun_out
timeout 300 python tools/probe_c4ab.py sparse 100000 > gpurun_out/g21_c4.jsonl 2>&1; cat gpurun_out/g21_c4.jsonl
timeout 1800 python tools/fuzz_parity.py 1560 11 > gpurun_out/r2_fuzz_parity_final.jsonl 2> gpurun_out/g21_fuzz.err; echo fuzz_rc=$?
tail -2 gpurun_out/r2_fuzz_parity_final.jsonl; tail -3 gpurun_out/g21_fuzz.err
