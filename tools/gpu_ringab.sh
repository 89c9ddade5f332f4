#!/bin/bash
# repeated A/B of ring-form knobs on the QFT30 every-tile passes
mkdir -p gpurun_out/ringab
python -m paper_2203_08826_b200.build > gpurun_out/ringab/build.log 2>&1 || exit 1
for rep in 1 2 3; do
for v in "base:" "nopairs:QJ_RING_PAIRS=0" "nbuf2:QJ_TILE_NBUF=2" "both:QJ_RING_PAIRS=0,QJ_TILE_NBUF=2"; do
  name=${v%%:*}; envs=${v#*:}
  ( IFS=","; for kv in $envs; do [ -n "$kv" ] && export "$kv"; done; IFS=" "
    timeout 300 python tools/sim_probe.py qft30_c128 > gpurun_out/ringab/s.json 2>/dev/null
    echo "$rep $name $(python3 -c "
import json; d=json.load(open('gpurun_out/ringab/s.json')); print('sep %.3f' % d['separate'], [round(x[1],3) for x in d['separate_launches']][-3:])")" )
done; done
