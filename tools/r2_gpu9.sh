mkdir -p gpurun_out
timeout 300 python tools/probe_c4.py 2000 20000 100000 > gpurun_out/g9_c4.jsonl 2>&1
cat gpurun_out/g9_c4.jsonl
timeout 900 python -m pytest tests -m gpu -x -q -k "sparse or large_n or overflow or c4 or stackonly" > gpurun_out/g9_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/g9_pytest.log
timeout 900 python tools/probe_ab.py auto data/cand/phat500_0.47_1.0.clq:0 2>/dev/null | head -0
timeout 900 python tools/probe_scale.py 60 data/cand/phat500_0.47_1.0.clq data/cand/phat500_0.48_1.0.clq data/cand/phat500_0.5_1.0.clq > gpurun_out/g9_scale.jsonl 2>&1
cat gpurun_out/g9_scale.jsonl
