#!/bin/bash
# A/B with correctness: for the product lib and each variant, C5/C1 probe + a GPU test subset.
for v in main "$@"; do
  if [ "$v" = main ]; then unset VCGPU_LIB; else export VCGPU_LIB=variants/$v/libvcgpu.so; fi
  echo "== $v"
  timeout 120 python tools/probe.py c5 c1 2>&1 | grep -E "pvc482|pvc84" | python3 -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(' ', d['label'], d['nodes'], d['device_ms'])"
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "config or c5 or sharded or hybrid_oracle" 2>&1 | tail -1
done
