mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g2_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g2_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/g2_pytest.log
timeout 300 python tools/probe.py c1 c3 c5 > gpurun_out/g2_probe.jsonl 2>&1
cat gpurun_out/g2_probe.jsonl
timeout 600 python bench.py > gpurun_out/g2_bench.json 2> gpurun_out/g2_bench.err; echo bench_rc=$?
tail -c 3000 gpurun_out/g2_bench.json
