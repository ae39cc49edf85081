mkdir -p gpurun_out
timeout 300 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el sparse-global 20 > gpurun_out/g22_sg.txt 2>&1; echo rc=$?; tail -5 gpurun_out/g22_sg.txt
timeout 300 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el sparse 20 > gpurun_out/g22_sp.txt 2>&1; echo rc=$?; tail -3 gpurun_out/g22_sp.txt
timeout 300 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el sparse-global 20 32 > gpurun_out/g22_sg1024.txt 2>&1; echo rc=$?; tail -3 gpurun_out/g22_sg1024.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el sparse-global 3 > gpurun_out/g22_memcheck.txt 2>&1; echo rc=$?; head -60 gpurun_out/g22_memcheck.txt
