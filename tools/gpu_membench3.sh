#!/bin/bash
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/membench tools/membench.cu || exit 1  # built on the box, never committed
out=gpurun_out/membench3.jsonl; : > $out
for cfg in "3 21" "3 12" "4 22"; do for B in 1 2; do for pm in 0 1 2; do
  timeout 60 ./tools/membench 30 $cfg $B c 5 $pm >> $out
done; done; done
echo done
