mkdir -p gpurun_out
timeout 600 bash tools/ab_shards_scale.sh data/cand/phat500_0.48_1.0.clq 448 > gpurun_out/g16_shards.txt 2>&1; cat gpurun_out/g16_shards.txt
