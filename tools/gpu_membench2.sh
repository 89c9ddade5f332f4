#!/bin/bash
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/membench2 tools/membench2.cu || exit 1  # built on the box, never committed
out=gpurun_out/membench2.jsonl; : > $out
for cfg in "13 4 21" "13 4 3" "13 5 21" "12 4 22" "12 3 21"; do
  for m in 0 1; do
    for w in "0 0" "2 0" "3 0" "0 16" "2 16" "3 32"; do
      timeout 60 ./tools/membench2 30 $cfg $m $w >> $out
    done
  done
done
echo done
