#!/bin/bash
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/membench tools/membench.cu || exit 1  # built on the box, never committed
mkdir -p gpurun_out
out=gpurun_out/membench.jsonl; : > $out
for cfg in "3 21" "3 18" "3 12" "3 3" "4 22" "5 23" "6 24" "8 26" "12 12"; do
  for B in 1 2 4; do for o in c b; do
    timeout 60 ./tools/membench 30 $cfg $B $o 5 >> $out
  done; done
done
echo done
