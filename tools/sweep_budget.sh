#!/bin/bash
for w in sup32_c64 var20_c128 qft30_c128; do
  for b in 48 96 192 100000; do
    for dag in 1 0; do
      QJ_TILE_BUDGET=$b QJ_TILE_DAG=$dag python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --no-unfused > gpurun_out/sw.log 2>&1
      tail -1 gpurun_out/sw.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$w budget=$b dag=$dag', round(d['value'],5), 'passes', d['kinds'].get('tile',{}).get('launches_per_step'), 'frac', round(d['kinds'].get('tile',{}).get('frac',0),3), 'dry', round(d['dry_run_s'],2))"
    done
  done
done
