bash tools/ab_shards.sh base mm2 2>&1
bash tools/ab_c5.sh base 2>&1 | grep -o '"device_ms": [0-9.]*\|== [a-z0-9]*' | paste -sd' '
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
VCG_BENCH_SAME_DEVICE=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --e2e-steps 2 2>&1 | tail -1 | cut -c1-600
