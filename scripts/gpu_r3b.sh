#!/bin/bash
mkdir -p gpurun_out
for v in "GD_COUNT_CTAS=1" "GD_COUNT_CTAS=2" "GD_COUNT_CTAS=4" "GD_COUNT_CTAS=8"; do
  tag=$(echo $v | tr ' =.' '___')
  env $v timeout 300 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
done
