#!/bin/bash
# ncu --set full of the C5 dense kernel (second launch of probe c5 = the k=482 solve).
R=${1:-cur}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_kernel -s 1 -c 1 \
    -o gpurun_out/${R}_c5_dense python tools/probe.py c5 > gpurun_out/${R}_ncu_c5.log 2>&1
tail -3 gpurun_out/${R}_ncu_c5.log
