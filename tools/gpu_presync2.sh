#!/bin/bash
mkdir -p gpurun_out/ps2
python -m paper_2203_08826_b200.build > gpurun_out/ps2/build.log 2>&1 || exit 1
for rep in 1 2 3; do for v in new:0 old:1; do n=${v%%:*}; e=${v#*:}
for w in qft30_c128 bv30_c128; do QJ_TILE_PRESYNC=$e timeout 300 python tools/sim_probe.py $w > gpurun_out/ps2/s.json 2>&1; echo "$rep $n $w $(python3 -c "
import json; d=json.load(open('gpurun_out/ps2/s.json')); print('sim %.3f sep %.3f' % (d['simulate'], d['separate']), [round(x[1],3) for x in d['separate_launches']][-4:])" 2>&1 | tail -1)"; done; done; done
