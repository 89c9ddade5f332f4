#!/bin/bash
mkdir -p gpurun_out/budget
python -m paper_2203_08826_b200.build > gpurun_out/budget/build.log 2>&1 || exit 1
for b in 64 96 128 192; do
for w in sup32_c64 qaoa30_c128 var20_c64 tfim20_c128; do QJ_TILE_BUDGET=$b timeout 300 python tools/sim_probe.py $w > gpurun_out/budget/sim_${b}_$w.json 2>&1; echo "budget $b $w $(python3 -c "
import json; d=json.load(open('gpurun_out/budget/sim_${b}_$w.json')); print('sim %.3f sep %.3f passes %d' % (d['simulate'], d['separate'], len(d['separate_launches'])))" 2>&1 | tail -1)"; done; done
