#!/bin/bash
# final round-1 evidence for the live-tile headline: simulate parity, smoke, bench line, launch list
mkdir -p gpurun_out/fin
timeout 600 python -m pytest tests -m gpu -x -q -k "simulate or smoke or qft" > gpurun_out/fin/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/fin/pytest.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/fin/bench.log 2>&1; echo "bench rc=$?"
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/fin/launches.csv $CMD > gpurun_out/fin/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qj_tile_jit -s 3 -c 3 \
    -o gpurun_out/fin/prof_tile -f $CMD > gpurun_out/fin/ncu_tile.log 2>&1; echo "ncu tile rc=$?"
