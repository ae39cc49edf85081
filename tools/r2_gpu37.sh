mkdir -p gpurun_out
for v in main m4small main m4small; do
  if [ "$v" = main ]; then unset VCGPU_LIB; else export VCGPU_LIB=variants/$v/libvcgpu.so; fi
  echo "== $v"; timeout 300 python tools/probe_ab.py auto data/cand/phat500_0.45_1.0.clq:449 2>&1 | cut -c100-260
done > gpurun_out/g37_ab.txt 2>&1; cat gpurun_out/g37_ab.txt
