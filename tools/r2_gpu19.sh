mkdir -p gpurun_out
for v in main nodmax notl main; do
  if [ "$v" = main ]; then unset VCGPU_LIB; else export VCGPU_LIB=variants/$v/libvcgpu.so; fi
  echo "== $v"; timeout 120 python tools/probe_ab.py auto c5 2>&1 | cut -c1-160
done > gpurun_out/g19_c5ab.txt 2>&1; cat gpurun_out/g19_c5ab.txt
unset VCGPU_LIB
timeout 600 python tools/probe_c4blk.py > gpurun_out/g19_c4blk.jsonl 2>&1; cat gpurun_out/g19_c4blk.jsonl
