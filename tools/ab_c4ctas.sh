# C4 sparse engine: CTAs per SM (product = 8) against variants built with VCG_SPARSE_MAX_CTAS
for v in main sp4 sp6 main; do
  if [ "$v" = main ]; then unset VCGPU_LIB; else export VCGPU_LIB=variants/$v/libvcgpu.so; fi
  echo "== $v"; timeout 300 python tools/probe_c4ab.py auto 20000 100000 2>&1 | grep budget
done
