#!/bin/bash
# All BASELINE.json single-GPU configs (+ the paper's TFIM sizes) through
# bench.py, one JSON line each, into gpurun_out/bench_<workload>.log.
for w in qft10_c128 var20_c128 var20_c64 tfim10_c128 tfim20_c128 sup32_c64; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; echo "$w rc=$?"
done
