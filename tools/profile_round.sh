#!/bin/bash
# One GPU call's worth of evidence for profiles/ (run under gpurun from the repo root).
set -x
R=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${R}_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/${R}_bench_under_ncu.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dense_kernel -s 1 -c 1 \
    -o gpurun_out/${R}_c5_dense python tools/probe.py c5 > gpurun_out/${R}_ncu_c5.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sparse_kernel -c 1 \
    -o gpurun_out/${R}_c4_sparse python tools/probe_c4.py 20000 > gpurun_out/${R}_ncu_c4.log 2>&1
timeout 120 python tools/probe_c4.py 2000 20000 100000 > gpurun_out/${R}_c4_probe.jsonl 2>&1
timeout 120 python tools/probe.py c1 c3 c5 > gpurun_out/${R}_probe.jsonl 2>&1
ls -la gpurun_out
