#!/bin/bash
# round-2 evidence: GPU tests, default bench line, per-pass sweep
mkdir -p gpurun_out/r02
python -m paper_2203_08826_b200.build > gpurun_out/r02/build.log 2>&1 || { echo build failed; exit 1; }
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke.log 2>&1; echo "smoke rc=$?"
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/r02/clocks.csv &
SMI=$!
timeout 900 python bench.py > gpurun_out/r02/bench.log 2>&1; echo "bench rc=$?"; tail -c 300 gpurun_out/r02/bench.log
kill $SMI
timeout 900 python tools/sweep_passes.py > gpurun_out/r02/sweep_passes.jsonl 2> gpurun_out/r02/sweep.err; echo "sweep rc=$?"
