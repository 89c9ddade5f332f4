#!/bin/bash
bash tools/gpu_ringab2.sh
mkdir -p gpurun_out/fin6
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/fin6/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fin6/pytest_gpu.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/fin6/clocks.csv &
SMI=$!
timeout 900 python bench.py > gpurun_out/fin6/bench.log 2>&1; echo "bench rc=$?"
kill $SMI
for w in qft30_c128 bv30_c128 qaoa30_c128; do timeout 900 python bench.py --workload $w > gpurun_out/fin6/bench_$w.log 2>&1; echo "config $w rc=$?"; done
python tools/qft_step.py separate 3 > gpurun_out/fin6/plain_sep.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:qj_tile_jit -s 6 -c 3 -o gpurun_out/fin6/ring_passes -f \
    python tools/qft_step.py separate 3 > gpurun_out/fin6/ncu_sep.log 2>&1; echo "ncu sep rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin6/smoke.log 2>&1; echo "smoke rc=$?"
