#!/bin/bash
# C5 (and C5-scale-class) device time, product library against variants, interleaved on one box.
# usage: tools/ab_c5.sh v1 [v2 ...]   (variants/NAME/libvcgpu.so from build_variant.sh)
for round in 1 2; do
for v in main "$@"; do
  if [ "$v" = main ]; then unset VCGPU_LIB; else export VCGPU_LIB=variants/$v/libvcgpu.so; fi
  timeout 300 python -c "
import sys, json; sys.path.insert(0, '.')
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
g = load_config('c5')
t = []
for _ in range(4):
    r = vc.solve_pvc(g, 482, strategy='gpu'); t.append(round(r['device_ms'], 2))
g2 = vc.load_graph('data/cand/phat500_0.45_1.0.clq', complement_input=True) if len(sys.argv) > 0 else None
r = vc.solve_pvc(g2, 449, strategy='gpu')
print('$v', 'c5', t, 'p45', round(r['device_ms'], 1), flush=True)
"
done
done
