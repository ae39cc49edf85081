mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g17_smi.txt 2>&1
timeout 3700 python tools/c2_long.py 3600 > gpurun_out/g17_c2_k240.log 2>&1; echo c2_rc=$?
cat gpurun_out/g17_c2_k240.log
