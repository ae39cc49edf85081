mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool memcheck --print-limit 10 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el sparse 80 > gpurun_out/g24_memcheck.txt 2>&1; echo rc=$?; grep -v "^[0-9]* 138 complete" gpurun_out/g24_memcheck.txt | head -60
