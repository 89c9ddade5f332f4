#!/bin/bash
mkdir -p gpurun_out/operm
python -m paper_2203_08826_b200.build > gpurun_out/operm/build.log 2>&1 || exit 1
for v in on:1 off:0; do n=${v%%:*}; e=${v#*:}
for w in qft30_c128 qaoa30_c128 bv30_c128 sup32_c64; do QJ_TILE_OPERM=$e timeout 300 python tools/sim_probe.py $w > gpurun_out/operm/sim_${n}_$w.json 2>&1; echo "$n $w $(python3 -c "
import json; d=json.load(open('gpurun_out/operm/sim_${n}_$w.json')); print('sim %.3f sep %.3f' % (d['simulate'], d['separate']), [x[1] for x in d['simulate_launches']][-3:], [x[1] for x in d['separate_launches']][:3])" 2>&1 | tail -1)"; done; done
timeout 2000 python -m pytest tests -m gpu -x -q > gpurun_out/operm/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/operm/pytest.log
QJ_JIT=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or circuits or tiles" > gpurun_out/operm/pytest_interp.log 2>&1; echo "pytest interpreter rc=$?"; tail -2 gpurun_out/operm/pytest_interp.log
