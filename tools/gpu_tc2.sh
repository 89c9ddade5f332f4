#!/bin/bash
mkdir -p gpurun_out/tc2
python -m paper_2203_08826_b200.build > gpurun_out/tc2/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q -k "dense5 or nccl or fuse_gates or checked" > gpurun_out/tc2/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/tc2/pytest.log
timeout 900 python tools/sweep_passes.py > gpurun_out/tc2/sweep_passes.jsonl 2> gpurun_out/tc2/sweep.err; echo "sweep rc=$?"; grep "5q" gpurun_out/tc2/sweep_passes.jsonl | cut -c 1-200
