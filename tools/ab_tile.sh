#!/bin/bash
# A/B of tile-pass knobs on QFT30 c128 (simulate + separate per-pass times) and sup32-lite
# usage: QJ_AB="name1:ENV=..,ENV2=.. name2:..." bash tools/ab_tile.sh
mkdir -p gpurun_out/ab
python -m paper_2203_08826_b200.build > gpurun_out/ab/build.log 2>&1 || { echo build failed; tail gpurun_out/ab/build.log; exit 1; }
for spec in ${QJ_AB:-base:}; do
  name=${spec%%:*}; envs=${spec#*:}
  ( IFS=","; for kv in $envs; do [ -n "$kv" ] && export "$kv"; done; IFS=" "
    for w in ${QJ_WL:-qft30_c128}; do
      timeout 300 python tools/sim_probe.py $w > gpurun_out/ab/sim_${name}_$w.json 2> gpurun_out/ab/sim_${name}_$w.err
      echo "$name $w rc=$? $(cat gpurun_out/ab/sim_${name}_$w.json | head -c 1500)"
    done )
done
