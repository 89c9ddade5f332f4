#!/bin/bash
mkdir -p gpurun_out/live2
python -m paper_2203_08826_b200.build > gpurun_out/live2/build.log 2>&1 || echo "build rc=$?"
QJ_DEBUG_JIT=1 timeout 900 python -m pytest tests -m gpu -x -q -k "simulate or smoke or qft" 2>&1 > gpurun_out/live2/pytest_sim.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/live2/pytest_sim.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/live2/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/live2/bench.log 2>&1; echo "bench rc=$?"
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/live2/launches.csv $CMD > gpurun_out/live2/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qj_tile_jit -s 3 -c 3 \
    -o gpurun_out/live2/prof_tile -f $CMD > gpurun_out/live2/ncu_tile.log 2>&1; echo "ncu tile rc=$?"
