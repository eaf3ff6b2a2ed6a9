#!/bin/bash
mkdir -p gpurun_out
for v in "GD_INSERT_WAVES=1" "GD_INSERT_WAVES=2" "GD_INSERT_WAVES=3" "GD_INSERT_WAVES=4"; do
  tag=$(echo $v | tr ' =.' '___')
  env $v timeout 300 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
done
