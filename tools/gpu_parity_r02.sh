#!/bin/bash
# round-2 parity: the new full-size / controlled-fSim / sharded-amplitude tests, then smoke
mkdir -p gpurun_out/par
python -m paper_2203_08826_b200.build > gpurun_out/par/build.log 2>&1 || { echo build failed; exit 1; }
nproc; free -g | head -2
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -v -s -x ${QJ_K:+-k "$QJ_K"} > gpurun_out/par/pytest_fullsize.log 2>&1; echo "fullsize rc=$?"; tail -5 gpurun_out/par/pytest_fullsize.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/par/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/par/smoke.log
