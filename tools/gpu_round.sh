#!/bin/bash
# One gpurun call: GPU tests, smoke, the default bench line, the ncu launch list
# of the same bench command, and one --set full capture of the fused tile kernel.
mkdir -p gpurun_out
python -m paper_2203_08826_b200.build > gpurun_out/build.log 2>&1 || echo "build rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qj_tile_jit -s 3 -c 2 \
    -o gpurun_out/prof_tile -f $CMD > gpurun_out/ncu_tile.log 2>&1; echo "ncu tile rc=$?"
