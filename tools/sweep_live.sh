#!/bin/bash
# qj_simulate QFT30 c128 (live tiles): tile-kernel knobs, headline leg only
mkdir -p gpurun_out/sweep
timeout 600 python -m pytest tests -m gpu -x -q -k "simulate or smoke" > gpurun_out/sweep/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/sweep/pytest.log
for env in "X=0" "QJ_TILE_BLOCKS=1" "QJ_TILE_BLOCKS=3" "QJ_JIT_STAGE_TERMS=0" "QJ_JIT_STAGE=0" "QJ_TILE_ORDER=b" "QJ_TILE_PAIR=0" "QJ_TILE_DEPTH=2"; do
  env $env timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-unfused > gpurun_out/sweep/s.log 2>&1
  tail -1 gpurun_out/sweep/s.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$env', round(d['value']*1e3,3), 'ms', 'tile', d['kinds'].get('tile'))" || tail -3 gpurun_out/sweep/s.log
done
