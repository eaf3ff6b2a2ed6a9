#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_download.py -q -rf -p no:cacheprovider > gpurun_out/pytest_dl.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dl.log
for v in "GD_DL_DELTA=1" "GD_DL_DELTA=1 GD_DL_DIRECT_FRAC=0" "GD_DL_DELTA=1 GD_DL_DIRECT_FRAC=0.1" "GD_DL_DELTA=0"; do
  tag=$(echo $v | tr ' =.' '___')
  env GD_DL_TRACE=1 $v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-profile > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
done
