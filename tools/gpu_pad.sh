#!/bin/bash
mkdir -p gpurun_out/pad
python -m paper_2203_08826_b200.build > gpurun_out/pad/build.log 2>&1 || exit 1
for v in high: low:QJ_TILE_PAD=low; do n=${v%%:*}; e=${v#*:}
for w in sup32_c64 qaoa30_c128 bv30_c128 var20_c128; do ( [ -n "$e" ] && export $e; timeout 300 python tools/sim_probe.py $w > gpurun_out/pad/sim_${n}_$w.json 2>&1 ); echo "$n $w $(python3 -c "
import json; d=json.load(open('gpurun_out/pad/sim_${n}_$w.json')); print('sim %.3f sep %.3f' % (d['simulate'], d['separate']))" 2>&1 | tail -1)"; done; done
