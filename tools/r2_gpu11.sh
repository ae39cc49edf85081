mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1 \
    > gpurun_out/g11_bench_under_ncu.log 2>&1; echo launches_rc=$?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:dense_kernel -s 1 -c 1 \
    -o gpurun_out/r2_c5_dense python tools/probe.py c5 > gpurun_out/g11_ncu_c5.log 2>&1; echo c5_rc=$?
timeout 500 ncu --set full --clock-control none --import-source on -k regex:dense_kernel -c 1 \
    -o gpurun_out/r2_c2_mid8 python -c "
import sys; sys.path.insert(0, '.')
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
r = vc.solve_pvc(load_config('c2'), 240, strategy='gpu', timeout_s=0.3); print(r['nodes_total'], r['device_ms'])
" > gpurun_out/g11_ncu_c2.log 2>&1; echo c2_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_kernel -c 1 \
    -o gpurun_out/r2_c5s_mid4 python -c "
import sys; sys.path.insert(0, '.')
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
r = vc.solve_pvc(load_config('c5s'), 448, strategy='gpu', timeout_s=0.5); print(r['nodes_total'], r['device_ms'])
" > gpurun_out/g11_ncu_c5s.log 2>&1; echo c5s_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_kernel -c 1 \
    -o gpurun_out/r2_c4_sparse python tools/probe_c4.py 20000 > gpurun_out/g11_ncu_c4.log 2>&1; echo c4_rc=$?
timeout 900 bash tools/ab_shards_scale.sh data/cand/phat500_0.48_1.0.clq 448 pollm32 > gpurun_out/g11_shards.txt 2>&1; cat gpurun_out/g11_shards.txt
ls -la gpurun_out/*.ncu-rep
