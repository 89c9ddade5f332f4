#!/bin/bash
CMD="python bench.py --workload sup32_c64 --steps 1 --warmup 1 --no-cpu-baseline --no-unfused"
$CMD > gpurun_out/plain_sup.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:qj_tile_jit -s 40 -c 1 -o gpurun_out/prof_sup $CMD > gpurun_out/ncu_sup.log 2>&1
echo done
