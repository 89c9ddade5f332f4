#!/bin/bash
# JIT tile kernel variants on the tile probe: CTAs per SM, ring depth, tile order.
for dt in ${DTS:-c128 c64}; do
  for cfg in ${CFGS:-"2 1 c" "2 1 b" "2 2 b" "1 2 b" "1 3 b" "1 3 c"}; do
    set -- $cfg
    echo "== $dt blocks=$1 depth=$2 order=$3"
    QJ_TILE_BLOCKS=$1 QJ_TILE_DEPTH=$2 QJ_TILE_ORDER=$3 timeout 300 python tools/tile_probe.py $dt 2>&1 | python -c "
import json,sys
t=sys.stdin.read()
try:
    d=json.loads(t[t.index('{'):])
    print(' '.join('%s=%.3f' % (k, v.get('frac', 0)) for k, v in d.items()))
except Exception as e:
    print('ERR', t[-400:])
"
  done
done
