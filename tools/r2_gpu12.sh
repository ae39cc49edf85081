# profiles with on-box reduction (ncu reports are ~24 MB each; gpurun_out must stay < 64 MiB)
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1 \
    > gpurun_out/g12_bench_under_ncu.log 2>&1; echo launches_rc=$?
prof() {  # name, kernel regex, command...
  local name=$1 kre=$2; shift 2
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kre -s ${SKIP:-0} -c 1 -o /tmp/$name "$@" > gpurun_out/${name}_ncu.log 2>&1
  python tools/ncu_summary.py /tmp/$name.ncu-rep > gpurun_out/${name}_summary.json 2>&1
  python tools/ncu_lines.py /tmp/$name.ncu-rep > gpurun_out/${name}_lines.txt 2>&1
  python tools/ncu_lines.py /tmp/$name.ncu-rep 0 > gpurun_out/${name}_lines_by_inst.txt 2>&1
}
SKIP=1 prof r2_c5_dense dense_kernel python tools/probe.py c5
cp /tmp/r2_c5_dense.ncu-rep gpurun_out/
prof r2_c2_mid8 dense_kernel python -c "
import sys; sys.path.insert(0, '.')
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
r = vc.solve_pvc(load_config('c2'), 240, strategy='gpu', timeout_s=0.3); print(r['nodes_total'], r['device_ms'])
"
prof r2_c5s_mid4 dense_kernel python -c "
import sys; sys.path.insert(0, '.')
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
r = vc.solve_pvc(load_config('c5s'), 448, strategy='gpu', timeout_s=0.5); print(r['nodes_total'], r['device_ms'])
"
prof r2_c4_sparse sparse_kernel python tools/probe_c4.py 20000
du -sh gpurun_out
