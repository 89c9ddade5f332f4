#!/bin/bash
# bench smoke: default line, the sharded path on one NCCL rank, reference arm, BV/QAOA configs
mkdir -p gpurun_out/bench
python -m paper_2203_08826_b200.build > gpurun_out/bench/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python bench.py > gpurun_out/bench/default.log 2>&1; echo "default rc=$?"; tail -c 400 gpurun_out/bench/default.log
timeout 600 python bench.py --sharded-n 30 --steps 3 --warmup 3 > gpurun_out/bench/sharded1.log 2>&1; echo "sharded rc=$?"; tail -c 400 gpurun_out/bench/sharded1.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench/reference.log 2>&1; echo "ref rc=$?"; tail -c 300 gpurun_out/bench/reference.log
for w in bv30_c128 qaoa30_c128 var20_c128; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench/$w.log 2>&1; echo "$w rc=$?"
done
