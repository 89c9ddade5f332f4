#!/bin/bash
# ncu --set full on the fused tile kernel (QFT30 c128), after a plain run.
CMD="python bench.py --fuse --steps 1 --warmup 1 --no-cpu-baseline"
QJ_DEBUG_PLAN=1 $CMD > gpurun_out/plain_tile.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:tile -s 3 -c 1 \
    -o gpurun_out/prof_tile $CMD > gpurun_out/ncu_tile.log 2>&1
echo done
