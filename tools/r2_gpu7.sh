mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "mid_layouts or sparse_global or large_n or overflow or sparse_frontier or fill_the_device" > gpurun_out/g7_new.log 2>&1; echo newtests_rc=$?
tail -25 gpurun_out/g7_new.log
timeout 900 python tools/probe_ab.py auto,dense-mid4,dense-mid8 c5 c2:5 data/cand/phat500_0.45_1.0.clq:449 > gpurun_out/g7_ab.jsonl 2>&1
cat gpurun_out/g7_ab.jsonl
timeout 300 python tools/probe_c4.py 2000 20000 100000 > gpurun_out/g7_c4.jsonl 2>&1
cat gpurun_out/g7_c4.jsonl
