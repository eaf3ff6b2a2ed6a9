#!/bin/bash
mkdir -p gpurun_out
for v in "GD_WARP_EXPAND=1" "GD_WARP_EXPAND=0" "GD_LOOP_SPLIT=1 GD_INSERT_PER=8" "GD_LOOP_SPLIT=1 GD_INSERT_PER=4" "GD_LOOP_SPLIT=1 GD_INSERT_PER=2" "GD_WARP_EXPAND=0 GD_LOOP_SPLIT=1 GD_INSERT_PER=2"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
done
