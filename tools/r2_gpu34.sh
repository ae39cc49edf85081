mkdir -p gpurun_out
for v in main smallcta main smallcta; do
  if [ "$v" = main ]; then unset VCGPU_LIB; else export VCGPU_LIB=variants/$v/libvcgpu.so; fi
  echo "== $v"; timeout 200 python tools/probe_ab.py auto c5 c2:3 2>&1 | cut -c1-150
done > gpurun_out/g34_ab.txt 2>&1; cat gpurun_out/g34_ab.txt
unset VCGPU_LIB
timeout 900 python -m pytest tests -m gpu -x -q -k "mid_layouts or c5 or c3 or corpus_hybrid or dense_widths or compact_and_wide" > gpurun_out/g34_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/g34_pytest.log
