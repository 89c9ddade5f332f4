#!/bin/bash
# ncu --set full of the QFT30 live pass 3 (the headline's dominant kernel)
mkdir -p gpurun_out/nl
python -m paper_2203_08826_b200.build > gpurun_out/nl/build.log 2>&1 || exit 1
python tools/qft_step.py simulate 4 > gpurun_out/nl/plain_sim.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qj_tile_jit -s 8 -c 1 -o gpurun_out/nl/live_pass3 -f \
    python tools/qft_step.py simulate 4 > gpurun_out/nl/ncu_sim.log 2>&1; echo "ncu sim rc=$?"
