#!/bin/bash
mkdir -p gpurun_out/l2
python -m paper_2203_08826_b200.build > gpurun_out/l2/build.log 2>&1 || exit 1
QJ_AB="auto: none:QJ_TMAP_L2=0 l128:QJ_TMAP_L2=1 l256:QJ_TMAP_L2=2" QJ_WL="qft30_c128" bash tools/ab_tile.sh 2>&1 | cut -c 1-400
python tools/qft_step.py separate 3 > gpurun_out/l2/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:qj_tile_jit --csv \
    --log-file gpurun_out/l2/launches_auto.csv python tools/qft_step.py separate 3 > gpurun_out/l2/ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 python tools/sweep_passes.py > gpurun_out/l2/sweep.jsonl 2> gpurun_out/l2/sweep.err; echo "sweep rc=$?"; tail -3 gpurun_out/l2/sweep.err
