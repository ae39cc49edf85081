mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/g10_bench.json 2> gpurun_out/g10_bench.err; echo bench_rc=$?
tail -c 4000 gpurun_out/g10_bench.json; tail -3 gpurun_out/g10_bench.err
timeout 300 python tools/probe_c4seq.py 300 1000 > gpurun_out/g10_c4seq.jsonl 2>&1; cat gpurun_out/g10_c4seq.jsonl
timeout 900 bash tools/ab_shards_scale.sh data/cand/phat500_0.48_1.0.clq 448 minb3 > gpurun_out/g10_shards.txt 2>&1; cat gpurun_out/g10_shards.txt
timeout 300 python tools/probe_ab.py dense-nomid data/cand/phat500_0.48_1.0.clq:448 > gpurun_out/g10_nomid.jsonl 2>&1; cat gpurun_out/g10_nomid.jsonl
VCG_BENCH_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --workload c5 > gpurun_out/g10_same2.json 2> gpurun_out/g10_same2.err; echo same2_rc=$?
tail -c 1500 gpurun_out/g10_same2.json; tail -3 gpurun_out/g10_same2.err
