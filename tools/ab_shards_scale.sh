#!/bin/bash
# Multi-shard overhead on one device for a C5-scale candidate: one full-device solve vs 2 and 4
# linked shards sharing the device (root start), product lib vs variants.
# usage: tools/ab_shards_scale.sh FILE.clq K [variant ...]
F=$1; K=$2; shift 2
for v in main "$@"; do
  if [ "$v" = main ]; then unset VCGPU_LIB; else export VCGPU_LIB=variants/$v/libvcgpu.so; fi
  echo "== $v"
  timeout 900 python -c "
import sys, json; sys.path.insert(0, '.')
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.shards import solve_sharded
g = vc.load_graph('$F', complement_input=True)
r = vc.solve_pvc(g, $K, strategy='gpu')
print(json.dumps(dict(shards=1, nodes=r['nodes_total'], ms=round(r['device_ms'], 1), idle=r['timeline']['idle_share'])), flush=True)
for devs in ((0, 0), (0, 0, 0, 0)):
    r = solve_sharded(g, 'pvc', $K, devices=devs)
    print(json.dumps(dict(shards=len(devs), nodes=r['nodes_total'], ms=round(max(r['rank_device_ms']), 1),
                          rank_nodes=r['rank_nodes'], peer=r['rank_donated_peer'], idle=r['rank_idle_share'])), flush=True)
"
done
