#!/bin/bash
mkdir -p gpurun_out/ab4
python -m paper_2203_08826_b200.build > gpurun_out/ab4/build.log 2>&1 || exit 1
for v in early:1 late:0; do n=${v%%:*}; e=${v#*:}
for w in qft30_c128 bv30_c128 qaoa30_c128; do QJ_EARLY_SLOTS=$e timeout 300 python tools/sim_probe.py $w > gpurun_out/ab4/sim_${n}_$w.json 2>&1; echo "$n $w $(python3 -c "
import json; d=json.load(open('gpurun_out/ab4/sim_${n}_$w.json')); print('sim %.3f sep %.3f' % (d['simulate'], d['separate']), [x[1] for x in d['simulate_launches']][-4:])")"; done; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/ab4/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab4/pytest.log
