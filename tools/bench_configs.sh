#!/bin/bash
# All BASELINE.json single-GPU configs through bench.py (one JSON line each).
for w in qft10_c128 var20_c128 var20_c64 sup32_c64; do
  python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; echo "$w rc=$?"
done
