#!/bin/bash
# round-2 baseline: full GPU suite, bench line, per-pass timings, JIT sources of QFT30 / sup32
mkdir -p gpurun_out/base
python -m paper_2203_08826_b200.build > gpurun_out/base/build.log 2>&1 || { echo build failed; exit 1; }
mkdir -p gpurun_out/base/jit
QJ_DUMP_JIT=gpurun_out/base/jit timeout 300 python tools/dump_jit.py qft30 > gpurun_out/base/dump.log 2>&1; echo "dump rc=$?"
timeout 300 python tools/sim_probe.py > gpurun_out/base/sim.json 2>&1; echo "sim rc=$?"
timeout 900 python bench.py > gpurun_out/base/bench.log 2>&1; echo "bench rc=$?"; tail -c 600 gpurun_out/base/bench.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/base/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/base/pytest.log
