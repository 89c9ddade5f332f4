#!/bin/bash
mkdir -p gpurun_out/ab3
python -m paper_2203_08826_b200.build > gpurun_out/ab3/build.log 2>&1 || exit 1
for w in qft30_c128 bv30_c128 qaoa30_c128 sup32_c64; do timeout 300 python tools/sim_probe.py $w > gpurun_out/ab3/sim_$w.json 2>&1; echo "$w $(python3 -c "
import json; d=json.load(open('gpurun_out/ab3/sim_$w.json')); print('sim %.3f sep %.3f' % (d['simulate'], d['separate']), [x[1] for x in d['simulate_launches']][-4:])")"; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "simulate or live or tile or fused or fsim" > gpurun_out/ab3/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab3/pytest.log
