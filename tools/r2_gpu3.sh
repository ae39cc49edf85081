mkdir -p gpurun_out
timeout 300 python tools/probe_c2phase.py 10 > gpurun_out/g3_c2phase.jsonl 2>&1
cat gpurun_out/g3_c2phase.jsonl
timeout 1500 python tools/probe_scale.py 100 data/cand/phat500_0.25_0.8.clq data/cand/phat500_0.25_0.85.clq data/cand/phat500_0.3_0.9.clq data/cand/phat500_0.25_1.0.clq data/cand/phat500_0.35_0.95.clq data/cand/phat500_0.5_1.0.clq > gpurun_out/g3_scale.jsonl 2>&1
cat gpurun_out/g3_scale.jsonl
