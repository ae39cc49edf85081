mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el sparse 3 > gpurun_out/g23_memcheck.txt 2>&1; echo rc=$?; head -80 gpurun_out/g23_memcheck.txt
