mkdir -p gpurun_out
export VCGPU_LIB=variants/sp1024x1/libvcgpu.so
timeout 600 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el sparse 300 > gpurun_out/g27_old.txt 2>&1; echo old rc=$?; tail -2 gpurun_out/g27_old.txt
unset VCGPU_LIB
timeout 600 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el sparse 300 32 > gpurun_out/g27_1024x2.txt 2>&1; echo 1024x2 rc=$?; tail -2 gpurun_out/g27_1024x2.txt
timeout 600 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el sparse 300 8 > gpurun_out/g27_256.txt 2>&1; echo 256 rc=$?; tail -2 gpurun_out/g27_256.txt
