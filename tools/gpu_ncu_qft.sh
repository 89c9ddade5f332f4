#!/bin/bash
python -m paper_2203_08826_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python tools/qft_passes.py 30 2 > gpurun_out/qft.log 2>&1 || { echo qft failed; exit 1; }
for m in 1 0; do
QJ_TILE_PIPE=$m timeout 900 ncu --set full --clock-control none --import-source on -k regex:qj_tile_jit -s 3 -c 3 \
    -o gpurun_out/prof_qft_pipe$m -f python tools/qft_passes.py 30 2 > gpurun_out/ncu_qft$m.log 2>&1; echo "ncu $m rc=$?"
done
