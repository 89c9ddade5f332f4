#!/bin/bash
for c in 3 4 5; do
  QJ_TILE_C=$c timeout 300 python tools/tile_probe.py c128 > gpurun_out/probe_c$c.json 2>&1; echo "c=$c rc=$?"
  QJ_TILE_C=$c timeout 300 python tools/sim_probe.py > gpurun_out/sim_c$c.json 2>&1; echo "sim c=$c rc=$?"
done
