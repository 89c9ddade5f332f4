#!/bin/bash
mkdir -p gpurun_out/operm2
python -m paper_2203_08826_b200.build > gpurun_out/operm2/build.log 2>&1 || exit 1
for w in qft30_c128 qaoa30_c128 bv30_c128; do timeout 300 python tools/sim_probe.py $w > gpurun_out/operm2/sim_$w.json 2>&1; echo "final-only $w $(python3 -c "
import json; d=json.load(open('gpurun_out/operm2/sim_$w.json')); print('sim %.3f sep %.3f' % (d['simulate'], d['separate']))" 2>&1 | tail -1)"; done
bash tools/gpu_final_r02.sh
