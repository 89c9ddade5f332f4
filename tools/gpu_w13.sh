#!/bin/bash
# build-time window width experiment: W = 13 (4 low bits + 9, 512 threads) vs the default 12
mkdir -p gpurun_out/w13
QJ_TILE_W=13 python -m paper_2203_08826_b200.build --force > gpurun_out/w13/build.log 2>&1 || { echo build failed; tail gpurun_out/w13/build.log; exit 1; }
for w in qft30_c128 qaoa30_c128 sup32_c64; do timeout 600 python tools/sim_probe.py $w > gpurun_out/w13/sim_$w.json 2>&1; echo "w13 $w $(python3 -c "
import json; d=json.load(open('gpurun_out/w13/sim_$w.json')); print('sim %.3f sep %.3f' % (d['simulate'], d['separate']), [x[1] for x in d['separate_launches']][:6])" 2>&1 | tail -1)"; done
python -m paper_2203_08826_b200.build --force > /dev/null 2>&1
