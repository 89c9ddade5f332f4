#!/bin/bash
mkdir -p gpurun_out/budget2
python -m paper_2203_08826_b200.build > gpurun_out/budget2/build.log 2>&1 || exit 1
for w in qft30_c128 bv30_c128 sup32_c64 qaoa30_c128; do timeout 300 python tools/sim_probe.py $w > gpurun_out/budget2/sim_$w.json 2>&1; echo "$w $(python3 -c "
import json; d=json.load(open('gpurun_out/budget2/sim_$w.json')); print('sim %.3f sep %.3f passes %d' % (d['simulate'], d['separate'], len(d['separate_launches'])))" 2>&1 | tail -1)"; done
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/budget2/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/budget2/pytest.log
