mkdir -p gpurun_out
export VCGPU_LIB=variants/sp128x4/libvcgpu.so
timeout 600 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el sparse 300 > gpurun_out/g28_128x4.txt 2>&1; echo 128x4 rc=$?; grep -c complete gpurun_out/g28_128x4.txt
unset VCGPU_LIB
timeout 600 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el sparse 300 2 > gpurun_out/g28_64.txt 2>&1; echo 64x8 rc=$?; grep -c complete gpurun_out/g28_64.txt
timeout 600 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el sparse 300 4 65536 > gpurun_out/g28_cap.txt 2>&1; echo 128x8cap rc=$?; grep -c complete gpurun_out/g28_cap.txt
timeout 600 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el sparse 300 4 > gpurun_out/g28_128.txt 2>&1; echo 128x8 rc=$?; grep -c complete gpurun_out/g28_128.txt
