#!/bin/bash
# Device time / node rate across builds (the product library, historical worktrees under
# variants/, block_warps overrides, variant libraries), interleaved on one box.
# usage: [WL=c5|c5s] [REPS=6] tools/ab_hist.sh "label:dir:kwargs[:variant lib]" ...
#   c5: PVC k=482 exact solves (device ms); c5s: C5-scale PVC k=448 for 2 s (M nodes/s)
cd ${GRAFT_REPO_ROOT:-.}
WL=${WL:-c5}; REPS=${REPS:-6}
for round in 1 2 3; do
for spec in "$@"; do
  IFS=: read label d kw lib <<< "$spec"
  if [ -n "$lib" ]; then export VCGPU_LIB=$PWD/$lib; else unset VCGPU_LIB; fi
  (cd $d && timeout 300 python -c "
import sys; sys.path.insert(0, '.')
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
g = load_config('$WL')
t = []
for _ in range($REPS):
    if '$WL' == 'c5':
        r = vc.solve_pvc(g, 482, strategy='gpu', $kw); t.append(round(r['device_ms'], 2))
    else:
        r = vc.solve_pvc(g, 448, strategy='gpu', timeout_s=2.0, $kw); t.append(round(r['nodes_total'] / r['device_ms'] / 1e3, 1))
print('$WL', '$label', r['nodes_total'], r['grid_blocks'], r['block_threads'], sorted(t), flush=True)
")
done
done
