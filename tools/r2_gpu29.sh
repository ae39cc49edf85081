mkdir -p gpurun_out
for cap in 256 64; do
timeout 300 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el sparse 100 4 $cap > gpurun_out/g29_128_$cap.txt 2>&1; echo 128x8 cap$cap rc=$?; grep -c complete gpurun_out/g29_128_$cap.txt
timeout 300 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el sparse 100 32 $cap > gpurun_out/g29_1024_$cap.txt 2>&1; echo 1024x2 cap$cap rc=$?; grep -c complete gpurun_out/g29_1024_$cap.txt
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el sparse 30 4 64 > gpurun_out/g29_memcheck.txt 2>&1; echo memcheck rc=$?; grep -v "complete" gpurun_out/g29_memcheck.txt | head -50
