#!/bin/bash
# ncu evidence for round 1 (run under gpurun, 1 GPU).  Plain run first, then
# the launch list, then --set full on the dominant kernels.
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:diag_kernel -s 100 -c 2 \
    -o gpurun_out/prof_diag $CMD > gpurun_out/ncu_diag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gate_warp -s 0 -c 1 \
    -o gpurun_out/prof_gate_hi $CMD > gpurun_out/ncu_gate_hi.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gate_warp -s 26 -c 2 \
    -o gpurun_out/prof_gate_lo $CMD > gpurun_out/ncu_gate_lo.log 2>&1
echo done
