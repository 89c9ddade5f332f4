#!/bin/bash
# live staging A/B + parity of the simulate paths + checked kernels
mkdir -p gpurun_out/ls
python -m paper_2203_08826_b200.build > gpurun_out/ls/build.log 2>&1 || exit 1
for rep in 1 2; do for v in on:1 off:0; do n=${v%%:*}; e=${v#*:}
for w in qft30_c128 bv30_c128 qaoa30_c128; do QJ_LIVE_STAGE=$e timeout 300 python tools/sim_probe.py $w > gpurun_out/ls/s.json 2>&1; echo "$rep $n $w $(python3 -c "
import json; d=json.load(open('gpurun_out/ls/s.json')); print('sim %.3f' % d['simulate'], [round(x[1],3) for x in d['simulate_launches']][-3:])" 2>&1 | tail -1)"; done; done; done
timeout 1800 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q -k "simulate or live or qft" > gpurun_out/ls/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ls/pytest.log
QJ_JIT_CHECK=1 timeout 600 python tools/sanitize_driver.py > gpurun_out/ls/checked.log 2>&1; echo "checked rc=$?"; tail -2 gpurun_out/ls/checked.log
