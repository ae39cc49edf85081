mkdir -p gpurun_out
for v in main d24 d32 main d24 d32; do
  if [ "$v" = main ]; then unset VCGPU_LIB; else export VCGPU_LIB=variants/$v/libvcgpu.so; fi
  echo "== $v"; timeout 200 python tools/probe_ab.py auto c5 2>&1 | cut -c1-130
done > gpurun_out/g35_ab.txt 2>&1; cat gpurun_out/g35_ab.txt
