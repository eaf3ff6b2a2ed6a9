#!/bin/bash
mkdir -p gpurun_out
for v in "GD_WARP_EXPAND=1 GD_XP_PER=4" "GD_WARP_EXPAND=1 GD_XP_PER=4 GD_INSERT_WAVES=7" "GD_WARP_EXPAND=0"; do
  tag=$(echo $v | tr ' =.' '___')
  env $v timeout 300 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
done
