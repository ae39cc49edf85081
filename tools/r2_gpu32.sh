mkdir -p gpurun_out
export VCGPU_LIB=variants/spcheck/libvcgpu.so
for i in 1 2; do
timeout 300 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el sparse 300 4 > gpurun_out/g32_$i.txt 2>&1; echo rc=$?; grep -c complete gpurun_out/g32_$i.txt; tail -1 gpurun_out/g32_$i.txt
done
unset VCGPU_LIB
for e in sparse sparse-global; do
timeout 300 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el $e 300 > gpurun_out/g32_$e.txt 2>&1; echo $e rc=$?; grep -c complete gpurun_out/g32_$e.txt
done
