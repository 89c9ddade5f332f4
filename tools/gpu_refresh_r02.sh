#!/bin/bash
# refresh after the binding change: default bench line (+ clocks), configs, e2e breakdown, HBM write ceiling
mkdir -p gpurun_out/fin3 gpurun_out/configs3
python -m paper_2203_08826_b200.build > gpurun_out/fin3/build.log 2>&1 || { echo build failed; exit 1; }
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/fin3/clocks.csv &
SMI=$!
timeout 900 python bench.py > gpurun_out/fin3/bench.log 2>&1; echo "bench rc=$?"
kill $SMI
for w in qft10_c128 var20_c128 var20_c64 tfim10_c128 tfim20_c128 qft30_c128 bv30_c128 qaoa30_c128 sup32_c64; do
  timeout 900 python bench.py --workload $w > gpurun_out/configs3/bench_$w.log 2>&1; echo "config $w rc=$?"
done
python tools/e2e_probe.py > gpurun_out/fin3/e2e_probe.json 2>&1; echo "e2e probe rc=$?"
python tools/write_bw.py > gpurun_out/fin3/write_bw.json 2>&1; echo "write bw rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin3/smoke.log 2>&1; echo "smoke rc=$?"
