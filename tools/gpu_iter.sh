#!/bin/bash
# quick iteration: build, fused-path GPU tests, tile probes (c128 + c64), QFT30 step
python -m paper_2203_08826_b200.build > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
mkdir -p gpurun_out/jit
QJ_DUMP_JIT=gpurun_out/jit timeout 300 python tools/dump_jit.py qft30 > gpurun_out/dump.log 2>&1; echo "dump rc=$?"; tail -3 gpurun_out/dump.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "${QJ_K:-circuits or fused or simulate or qft30 or supremacy or shard or host or cache or tiles}" > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_iter.log
timeout 300 python tools/tile_probe.py c128 > gpurun_out/probe_c128.json 2>&1; echo "probe rc=$?"
timeout 300 python tools/sim_probe.py > gpurun_out/sim.json 2>&1; echo "sim rc=$?"
