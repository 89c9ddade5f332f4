#!/bin/bash
mkdir -p gpurun_out/jit
QJ_DUMP_JIT=gpurun_out/jit timeout 300 python tools/dump_jit.py qft30 > gpurun_out/dump.log 2>&1; echo "dump rc=$?"
for b in 1 2; do for d in 1 2 3; do
  QJ_TILE_BLOCKS=$b QJ_TILE_DEPTH=$d timeout 300 python tools/tile_probe.py c128 > gpurun_out/probe_b${b}_d${d}.json 2>&1; echo "b=$b d=$d rc=$?"
done; done
