mkdir -p gpurun_out
export VCGPU_LIB=variants/spcheck/libvcgpu.so
for i in 1 2 3; do
timeout 300 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el sparse 150 4 > gpurun_out/g30_$i.txt 2>&1; echo rc=$?; grep -c complete gpurun_out/g30_$i.txt; tail -1 gpurun_out/g30_$i.txt
done
