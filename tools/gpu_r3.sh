#!/bin/bash
mkdir -p gpurun_out/r3
python -m paper_2203_08826_b200.build > gpurun_out/r3/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "simulate or live or tile or fused" > gpurun_out/r3/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r3/pytest.log
for w in qft30_c128 bv30_c128 qaoa30_c128; do timeout 300 python tools/sim_probe.py $w > gpurun_out/r3/sim_r4_$w.json 2>&1; echo "r4 $w $(head -c 300 gpurun_out/r3/sim_r4_$w.json)"; done
QJ_TILE_R=3 python -m paper_2203_08826_b200.build --force > gpurun_out/r3/build_r3.log 2>&1 || { echo r3 build failed; tail gpurun_out/r3/build_r3.log; }
for w in qft30_c128 qaoa30_c128; do timeout 300 python tools/sim_probe.py $w > gpurun_out/r3/sim_r3_$w.json 2>&1; echo "r3 $w $(head -c 300 gpurun_out/r3/sim_r3_$w.json)"; done
python -m paper_2203_08826_b200.build --force > /dev/null 2>&1
