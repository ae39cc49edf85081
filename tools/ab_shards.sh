#!/bin/bash
# Multi-shard A/B on one device: 2 and 4 shards of C5 k=482 (root start), product lib vs variants.
for v in main "$@"; do
  if [ "$v" = main ]; then unset VCGPU_LIB; else export VCGPU_LIB=variants/$v/libvcgpu.so; fi
  echo "== $v"
  timeout 120 python -c "
import sys, json; sys.path.insert(0, '.')
from paper_2204_10402_b200.configs import load_config
from paper_2204_10402_b200.shards import solve_sharded
g = load_config('c5')
for devs in ((0, 0), (0, 0), (0, 0, 0, 0), (0, 0, 0, 0)):
    r = solve_sharded(g, 'pvc', 482, devices=devs)
    assert r['nodes_total'] == 21461369
    print(len(devs), round(max(r['rank_device_ms']), 2), r['rank_donated_peer'])
"
done
