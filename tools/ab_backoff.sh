mkdir -p gpurun_out
for v in main bo500 bo200 main bo500 bo200; do
  if [ "$v" = main ]; then unset VCGPU_LIB; else export VCGPU_LIB=variants/$v/libvcgpu.so; fi
  timeout 200 python -c "
import sys, json; sys.path.insert(0, '.')
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
g = load_config('c5')
for _ in range(3):
    r = vc.solve_pvc(g, 482, strategy='gpu')
    print('$v', round(r['device_ms'], 3), round(r['timeline']['idle_share'], 4), flush=True)
"
done
