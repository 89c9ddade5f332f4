#!/bin/bash
# programmatic dependent launch of the tile passes: A/B on the simulate workloads, then the GPU suite
mkdir -p gpurun_out/pdl
python -m paper_2203_08826_b200.build > gpurun_out/pdl/build.log 2>&1 || exit 1
for rep in 1 2; do for v in on:1 off:0; do n=${v%%:*}; e=${v#*:}
for w in var20_c128 var20_c64 tfim20_c128 qft30_c128 qaoa30_c128; do QJ_PDL=$e timeout 300 python tools/sim_probe.py $w > gpurun_out/pdl/s.json 2>&1; echo "$rep $n $w $(python3 -c "
import json; d=json.load(open('gpurun_out/pdl/s.json')); print('sim %.4f sep %.4f' % (d['simulate'], d['separate']))" 2>&1 | tail -1)"; done; done; done
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pdl/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pdl/pytest_gpu.log
