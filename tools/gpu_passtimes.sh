#!/bin/bash
# per-pass durations (ncu launch list) of the fused QFT30 under planner/kernel variants
# VARIANTS: ';'-separated env assignments per variant, e.g. "QJ_TILE_CARRY=0;QJ_TILE_CARRY=0 QJ_JIT_SKIP=s"
python -m paper_2203_08826_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python tools/qft_passes.py 30 2 > gpurun_out/qft.log 2>&1 || { echo qft failed; exit 1; }
IFS=';' read -ra VS <<< "${VARIANTS:-QJ_TILE_CARRY=0;QJ_TILE_CARRY=1}"
for v in "${VS[@]}"; do
  env $v timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,launch__grid_size,launch__shared_mem_per_block_dynamic,launch__occupancy_limit_shared_mem --clock-control none -k regex:qj_tile_jit -s 3 -c 3 --csv \
    python tools/qft_passes.py ${NQ:-30} 2 2>/dev/null | grep -E '"qj_tile_jit"' | awk -F'","' -v v="${v// /,}" '{print v, $(NF-2), $NF}' | sed 's/"//g'
done
