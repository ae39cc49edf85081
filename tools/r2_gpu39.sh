mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ipc.py -m gpu -x -q -k "shard or ipc or persistent or fill or c5 or mid" > gpurun_out/g39_pytest.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/g39_pytest.log
timeout 900 bash tools/ab_shards_scale.sh data/cand/phat500_0.48_1.0.clq 448 > gpurun_out/g39_shards.txt 2>&1; cat gpurun_out/g39_shards.txt
