mkdir -p gpurun_out
for e in sparse sparse-global; do
  timeout 600 python tools/repro_sg.py tests/data/fuzz_gnp_256_549.el $e 150 > gpurun_out/g25_$e.txt 2>&1; echo $e rc=$?; tail -2 gpurun_out/g25_$e.txt
done
