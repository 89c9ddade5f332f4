#!/bin/bash
# ncu --set full of sup32 c64 simulate passes 4..8 (cyclic form; 4 to 10 dense 2-qubit ops each)
mkdir -p gpurun_out/ns
python -m paper_2203_08826_b200.build > gpurun_out/ns/build.log 2>&1 || exit 1
python tools/qft_step.py simulate 2 sup32_c64 > gpurun_out/ns/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qj_tile_jit -s 47 -c 5 -o gpurun_out/ns/sup_passes -f \
    python tools/qft_step.py simulate 2 sup32_c64 > gpurun_out/ns/ncu.log 2>&1; echo "ncu rc=$?"
