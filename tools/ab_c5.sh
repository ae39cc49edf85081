#!/bin/bash
# C5 k=482 device time, product library vs variants, interleaved (same box, same minute).
for rep in 1 2; do
  echo "== main"; timeout 120 python tools/probe.py c5 2>&1 | grep pvc482 | cut -c1-200
  for v in "$@"; do
    echo "== $v"; VCGPU_LIB=variants/$v/libvcgpu.so timeout 120 python tools/probe.py c5 2>&1 | grep pvc482 | cut -c1-200
  done
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
