#!/bin/bash
mkdir -p gpurun_out/rp
python -m paper_2203_08826_b200.build > gpurun_out/rp/build.log 2>&1 || exit 1
for v in base:0 pairs:1; do n=${v%%:*}; e=${v#*:}
for w in qft30_c128 qaoa30_c128 sup32_c64; do QJ_RING_PAIRS=$e timeout 300 python tools/sim_probe.py $w > gpurun_out/rp/sim_${n}_$w.json 2>&1; echo "$n $w $(python3 -c "
import json; d=json.load(open('gpurun_out/rp/sim_${n}_$w.json')); print('sim %.3f sep %.3f' % (d['simulate'], d['separate']), [x[1] for x in d['separate_launches']][:4])" 2>&1 | tail -1)"; done; done
QJ_RING_PAIRS=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q -k "fused or apply_circuit or supremacy or shard" > gpurun_out/rp/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/rp/pytest.log
