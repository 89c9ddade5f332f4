#!/bin/bash
# barrier before each transpose's write: dropped (default) vs kept (QJ_TILE_PRESYNC=1); then the GPU suite
mkdir -p gpurun_out/ps
python -m paper_2203_08826_b200.build > gpurun_out/ps/build.log 2>&1 || exit 1
for v in new:0 old:1; do n=${v%%:*}; e=${v#*:}
for w in qft30_c128 qaoa30_c128 bv30_c128 sup32_c64; do QJ_TILE_PRESYNC=$e timeout 300 python tools/sim_probe.py $w > gpurun_out/ps/sim_${n}_$w.json 2>&1; echo "$n $w $(python3 -c "
import json; d=json.load(open('gpurun_out/ps/sim_${n}_$w.json')); print('sim %.3f sep %.3f' % (d['simulate'], d['separate']), [round(x[1],3) for x in d['separate_launches']][-4:])" 2>&1 | tail -1)"; done; done
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/ps/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ps/pytest_gpu.log
