#!/bin/bash
mkdir -p gpurun_out/repro
python -m paper_2203_08826_b200.build > gpurun_out/repro/build.log 2>&1 || exit 1
timeout 300 python tools/repro_diag.py 24 > gpurun_out/repro/plain.log 2>&1; echo "repro24 rc=$?"; tail -3 gpurun_out/repro/plain.log
timeout 300 python tools/repro_diag.py 30 > gpurun_out/repro/plain30.log 2>&1; echo "repro30 rc=$?"; tail -3 gpurun_out/repro/plain30.log
QJ_AB="ring:" QJ_WL="qft30_c128 qaoa30_c128 sup32_c64" bash tools/ab_tile.sh 2>&1 | cut -c 1-300
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q > gpurun_out/repro/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/repro/pytest.log
timeout 900 python tools/sweep_passes.py > gpurun_out/repro/sweep.jsonl 2> gpurun_out/repro/sweep.err; echo "sweep rc=$?"; tail -3 gpurun_out/repro/sweep.err
