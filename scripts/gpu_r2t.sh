#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sort.py tests/test_gpu_ra.py -q -x -p no:cacheprovider > gpurun_out/pytest_sort.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sort.log
for v in "GD_WARP_APPEND=0" "GD_WARP_APPEND=1"; do
  tag=$(echo $v | tr ' =.' '___')
  env $v timeout 300 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
done
timeout 300 python scripts/sort_micro.py 771 > gpurun_out/sort_micro.log 2>&1
