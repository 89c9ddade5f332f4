#!/bin/bash
# Every BASELINE.json single-GPU config (+ BV / QAOA north-star extras and the
# paper's TFIM sizes) through bench.py, one JSON line each, into
# gpurun_out/configs/bench_<workload>.log; then per-section ncu DRAM traffic
# (tools/step_probe.py + tools/ncu_traffic.py) into gpurun_out/configs/ncu_traffic.json.
mkdir -p gpurun_out/configs
for w in ${QJ_CONFIGS:-qft10_c128 var20_c128 var20_c64 tfim10_c128 tfim20_c128 qft30_c128 bv30_c128 qaoa30_c128 sup32_c64}; do
  timeout 900 python bench.py --workload $w > gpurun_out/configs/bench_$w.log 2>&1; echo "$w rc=$?"
done
if [ -n "$QJ_TRAFFIC" ]; then
  for ws in $QJ_TRAFFIC; do
    w=${ws%%:*}; sec=${ws#*:}
    python tools/step_probe.py $w $sec 2 > gpurun_out/configs/probe_${w}_$sec.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
        --log-file gpurun_out/configs/ncu_${w}_$sec.csv python tools/step_probe.py $w $sec 2 > /dev/null 2>&1; echo "ncu $w $sec rc=$?"
    python tools/ncu_traffic.py gpurun_out/configs/ncu_traffic.json $w $sec gpurun_out/configs/ncu_${w}_$sec.csv
  done
fi
