mkdir -p gpurun_out
timeout 600 python tools/probe_ab.py auto,dense-mid4 c5 data/cand/phat500_0.45_1.0.clq:449 > gpurun_out/g8_ab.jsonl 2>&1
cat gpurun_out/g8_ab.jsonl
timeout 200 python tools/probe.py c1 c3 c5 > gpurun_out/g8_probe.jsonl 2>&1
cat gpurun_out/g8_probe.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_kernel -c 1 \
    -o gpurun_out/g8_c4_sparse python tools/probe_c4.py 100000 > gpurun_out/g8_ncu_c4.log 2>&1
tail -3 gpurun_out/g8_ncu_c4.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g8_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/g8_pytest.log
