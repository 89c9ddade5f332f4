#!/bin/bash
# round-2 final evidence at HEAD, one box:
#  1. per-section DRAM traffic launch lists -> profiles/r02/ncu_traffic.json (read by bench.py for roofline.traffic)
#  2. GPU suite, smoke
#  3. default bench line (+ nvidia-smi clocks during it), reference arm, sharded path at N=1
#  4. one bench line per BASELINE config
#  5. launch list of the bench command; ncu --set full of the headline pass and of the ring passes
mkdir -p gpurun_out/fin gpurun_out/configs
python -m paper_2203_08826_b200.build > gpurun_out/fin/build.log 2>&1 || { echo build failed; exit 1; }
rm -f gpurun_out/configs/ncu_traffic.json
for ws in qft30_c128:simulate qft30_c128:separate qft30_c128:unfused sup32_c64:simulate qaoa30_c128:simulate bv30_c128:simulate var20_c128:simulate tfim20_c128:simulate; do
  w=${ws%%:*}; sec=${ws#*:}
  python tools/step_probe.py $w $sec 2 > gpurun_out/configs/probe_${w}_$sec.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/configs/ncu_${w}_$sec.csv python tools/step_probe.py $w $sec 2 > /dev/null 2>&1; echo "ncu $w $sec rc=$?"
  python tools/ncu_traffic.py gpurun_out/configs/ncu_traffic.json $w $sec gpurun_out/configs/ncu_${w}_$sec.csv
done
cp gpurun_out/configs/ncu_traffic.json profiles/r02/ncu_traffic.json && echo "traffic json updated"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/fin/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fin/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo "smoke rc=$?"
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/fin/clocks.csv &
SMI=$!
timeout 900 python bench.py > gpurun_out/fin/bench.log 2>&1; echo "bench rc=$?"; tail -c 400 gpurun_out/fin/bench.log
kill $SMI
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin/reference.log 2>&1; echo "reference rc=$?"
timeout 600 python bench.py --sharded-n 30 --steps 3 --warmup 3 --no-replicas > gpurun_out/fin/sharded1.log 2>&1; echo "sharded rc=$?"
for w in qft10_c128 var20_c128 var20_c64 tfim10_c128 tfim20_c128 qft30_c128 bv30_c128 qaoa30_c128 sup32_c64; do
  timeout 900 python bench.py --workload $w > gpurun_out/configs/bench_$w.log 2>&1; echo "config $w rc=$?"
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-unfused"
$CMD > gpurun_out/fin/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/fin/launches.csv $CMD > gpurun_out/fin/ncu_list.log 2>&1; echo "ncu list rc=$?"
python tools/qft_step.py simulate 4 > gpurun_out/fin/plain_sim.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:qj_tile_jit -s 8 -c 1 -o gpurun_out/fin/live_pass3 -f \
    python tools/qft_step.py simulate 4 > gpurun_out/fin/ncu_sim.log 2>&1; echo "ncu sim rc=$?"
python tools/qft_step.py separate 3 > gpurun_out/fin/plain_sep.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:qj_tile_jit -s 6 -c 3 -o gpurun_out/fin/ring_passes -f \
    python tools/qft_step.py separate 3 > gpurun_out/fin/ncu_sep.log 2>&1; echo "ncu sep rc=$?"
