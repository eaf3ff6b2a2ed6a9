#!/bin/bash
mkdir -p gpurun_out
for v in "GD_WARP_EXPAND=1 GD_XP_PER=4" "GD_WARP_EXPAND=1 GD_XP_PER=8" "GD_WARP_EXPAND=0"; do
  tag=$(echo $v | tr ' =.' '___')
  env $v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
done
timeout 300 python -m pytest tests/test_gpu_loop.py -q -x -k "xp or heavy" -p no:cacheprovider > gpurun_out/pytest_xp.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_xp.log
