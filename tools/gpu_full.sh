#!/bin/bash
# round evidence: GPU tests, smoke, default bench, all single-GPU configs
python -m paper_2203_08826_b200.build > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
bash tools/bench_configs.sh
