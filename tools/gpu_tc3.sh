#!/bin/bash
mkdir -p gpurun_out/tc3
python -m paper_2203_08826_b200.build > gpurun_out/tc3/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "dense5 or fuse_gates" > gpurun_out/tc3/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/tc3/pytest.log
SWEEP_FILTER=5q timeout 600 python tools/sweep_passes.py 2>&1 | cut -c 1-160
