#!/bin/bash
# packed f32x2 complex64 arithmetic: simulate timings, then the GPU suite
mkdir -p gpurun_out/f2
python -m paper_2203_08826_b200.build > gpurun_out/f2/build.log 2>&1 || exit 1
for w in sup32_c64 var20_c64 var20_c128 qft30_c128; do timeout 600 python tools/sim_probe.py $w > gpurun_out/f2/sim_$w.json 2>&1; echo "$w $(python3 -c "
import json; d=json.load(open('gpurun_out/f2/sim_$w.json')); print('sim %.4f sep %.4f' % (d['simulate'], d['separate']))" 2>&1 | tail -1)"; done
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/f2/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/f2/pytest_gpu.log
