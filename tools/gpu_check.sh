#!/bin/bash
# One GPU session: parity tests, then config probes for the product library and any variants.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python tools/probe.py c1 c3 c5 2>&1 | tee gpurun_out/probe_main.jsonl
for v in "$@"; do
  echo "== variant $v"
  VCGPU_LIB=variants/$v/libvcgpu.so python tools/probe.py c1 c5 2>&1 | tee gpurun_out/probe_$v.jsonl
done
