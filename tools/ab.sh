#!/bin/bash
# A/B of variant libraries on C5 (and C1): parity tests on the product lib first, then probes.
mkdir -p gpurun_out
T=${TAG:-ab}
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 120 python tools/probe.py c5 c1 2>&1 | grep -v "mvc seq" | tee gpurun_out/${T}_main.jsonl
for v in "$@"; do
  echo "== variant $v"
  VCGPU_LIB=variants/$v/libvcgpu.so timeout 120 python tools/probe.py c5 c1 2>&1 | grep -v "mvc seq" | tee gpurun_out/${T}_$v.jsonl
done
