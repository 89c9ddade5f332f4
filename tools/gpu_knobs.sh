#!/bin/bash
mkdir -p gpurun_out/knobs
python -m paper_2203_08826_b200.build > gpurun_out/knobs/build.log 2>&1 || exit 1
QJ_AB="base: blocks3:QJ_TILE_BLOCKS=3 cyclic:QJ_TILE_ORDER=c nostage:QJ_JIT_STAGE=0 noterms:QJ_JIT_STAGE_TERMS=0 depth2:QJ_TILE_DEPTH=2" QJ_WL="qft30_c128" bash tools/ab_tile.sh 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    name=l.split()[0]; j=l[l.find('{'):]
    try:
        d=json.loads(j); print(name, 'sim %.3f'%d['simulate'], [x[1] for x in d['simulate_launches']], 'sep %.2f'%d['separate'])
    except Exception as e: print(l[:200])
"
python tools/qft_step.py simulate 4 > gpurun_out/knobs/plain_sim.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:qj_tile_jit -s 8 -c 1 -o gpurun_out/knobs/live_pass3 -f \
    python tools/qft_step.py simulate 4 > gpurun_out/knobs/ncu_sim.log 2>&1; echo "ncu sim rc=$?"
