#!/bin/bash
# ncu evidence for round 1 (run under gpurun, 1 GPU): plain run first, then the
# launch list (time + DRAM bytes per launch) of the same command, then
# --set full on the dominant kernels of the fused and the unfused paths.
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:qj_tile_jit -s 3 -c 2 \
    -o gpurun_out/prof_tile $CMD > gpurun_out/ncu_tile.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:diag_kernel -s 100 -c 1 \
    -o gpurun_out/prof_diag $CMD > gpurun_out/ncu_diag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gate_warp -s 0 -c 1 \
    -o gpurun_out/prof_gate $CMD > gpurun_out/ncu_gate.log 2>&1
echo done
