#!/bin/bash
# new ring defaults (short rows: 2 buffers, no pairs) vs the old (3 buffers, pairs) on the c128 workloads
mkdir -p gpurun_out/ringab2
python -m paper_2203_08826_b200.build > gpurun_out/ringab2/build.log 2>&1 || exit 1
for rep in 1; do
for v in "new:" "old:QJ_TILE_NBUF=3,QJ_RING_PAIRS=1"; do
  name=${v%%:*}; envs=${v#*:}
  for w in qft30_c128 bv30_c128 qaoa30_c128; do
  ( IFS=","; for kv in $envs; do [ -n "$kv" ] && export "$kv"; done; IFS=" "
    timeout 300 python tools/sim_probe.py $w > gpurun_out/ringab2/s.json 2>/dev/null
    echo "$rep $name $w $(python3 -c "
import json; d=json.load(open('gpurun_out/ringab2/s.json')); print('sim %.3f sep %.3f' % (d['simulate'], d['separate']), [round(x[1],3) for x in d['separate_launches']][-7:])")" )
  done
done; done
