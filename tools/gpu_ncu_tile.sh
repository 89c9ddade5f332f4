#!/bin/bash
# ncu --set full on the three QFT30 tile passes of one qj_simulate step (after
# the plain run exited 0); summary rows for the tile kernels.
python -m paper_2203_08826_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python tools/sim_probe.py > gpurun_out/sim.json 2>&1 || { echo sim failed; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qj_tile_jit -s ${SKIP:-9} -c 3 \
    -o gpurun_out/prof_tile13 -f python tools/sim_probe.py > gpurun_out/ncu_tile13.log 2>&1; echo "ncu rc=$?"
