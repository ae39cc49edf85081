mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "sparse or large_n or overflow or c4 or stackonly or frontier" > gpurun_out/g20_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/g20_pytest.log
timeout 600 python tools/probe_c4ab.py auto,sparse 20000 100000 > gpurun_out/g20_c4ab.jsonl 2>&1; cat gpurun_out/g20_c4ab.jsonl
timeout 200 python tools/probe_ab.py auto c5 > gpurun_out/g20_c5.jsonl 2>&1; cat gpurun_out/g20_c5.jsonl | cut -c1-150
