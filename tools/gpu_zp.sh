#!/bin/bash
# paired live tiles + early scale: A/B on the simulate workloads, then parity
mkdir -p gpurun_out/zp
python -m paper_2203_08826_b200.build > gpurun_out/zp/build.log 2>&1 || exit 1
for v in on:1:1 off:0:1 noscale:1:0; do IFS=: read n e s <<< "$v"
for w in qft30_c128 qaoa30_c128 bv30_c128 qft30_c64; do QJ_ZPAIR=$e QJ_EARLY_SCALE=$s timeout 300 python tools/sim_probe.py $w > gpurun_out/zp/sim_${n}_$w.json 2>&1; echo "$n $w $(python3 -c "
import json; d=json.load(open('gpurun_out/zp/sim_${n}_$w.json')); print('sim %.3f' % d['simulate'], [round(x[1],3) for x in d['simulate_launches']][-3:])" 2>&1 | tail -1)"; done; done
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q -k "simulate or live" > gpurun_out/zp/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/zp/pytest.log
