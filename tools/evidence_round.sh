# round evidence: bench line, launch list, ncu summaries (reduced on the box); P = file prefix
P=${P:-r2f}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${P}_gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err; echo bench_rc=$?
tail -c 600 gpurun_out/${P}_bench.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${P}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1 \
    > gpurun_out/${P}_bench_under_ncu.log 2>&1; echo launches_rc=$?
prof() {  # name, kernel regex, skip, command...
  local name=$1 kre=$2 skip=$3; shift 3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 -o /tmp/$name "$@" > gpurun_out/${name}_ncu.log 2>&1
  python tools/ncu_summary.py /tmp/$name.ncu-rep > gpurun_out/${name}_summary.json 2>&1
  python tools/ncu_lines.py /tmp/$name.ncu-rep > gpurun_out/${name}_lines.txt 2>&1
}
prof ${P}_c5_dense dense_kernel 1 python tools/probe.py c5
prof ${P}_c4_sparse sparse_kernel 1 python tools/probe_c4.py 2000 100000
prof ${P}_c2_mid8 dense_kernel 0 python -c "
import sys; sys.path.insert(0, '.')
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
r = vc.solve_pvc(load_config('c2'), 240, strategy='gpu', timeout_s=0.3); print(r['nodes_total'], r['device_ms'])
"
prof ${P}_c5s_mid4 dense_kernel 0 python -c "
import sys; sys.path.insert(0, '.')
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
r = vc.solve_pvc(load_config('c5s'), 448, strategy='gpu', timeout_s=0.5); print(r['nodes_total'], r['device_ms'])
"
timeout 600 python tools/probe_c4ab.py auto 20000 100000 > gpurun_out/${P}_c4.jsonl 2>&1
VCG_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 1 --warmup 1 > gpurun_out/${P}_same2.json 2> gpurun_out/${P}_same2.err; echo same2_rc=$?
tail -c 800 gpurun_out/${P}_same2.json
du -sh gpurun_out
