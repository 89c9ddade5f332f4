#!/bin/bash
# ncu --set full of the QFT30 tile passes: the live headline pass 3 and the every-tile (ring) pass 3
mkdir -p gpurun_out/ncu
python -m paper_2203_08826_b200.build > gpurun_out/ncu/build.log 2>&1 || exit 1
python tools/qft_step.py simulate 4 > gpurun_out/ncu/plain_sim.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:qj_tile_jit -s 8 -c 1 -o gpurun_out/ncu/live_pass3 -f \
    python tools/qft_step.py simulate 4 > gpurun_out/ncu/ncu_sim.log 2>&1; echo "ncu sim rc=$?"
python tools/qft_step.py separate 3 > gpurun_out/ncu/plain_sep.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:qj_tile_jit -s 6 -c 3 -o gpurun_out/ncu/ring_passes -f \
    python tools/qft_step.py separate 3 > gpurun_out/ncu/ncu_sep.log 2>&1; echo "ncu sep rc=$?"
