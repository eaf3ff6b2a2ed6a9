#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_loop.py tests/test_gpu_engine.py tests/test_gpu_scale.py -q -rf -x -p no:cacheprovider -k "not full_scale" > gpurun_out/pytest_pre.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pre.log
for v in "GD_PRECOUNT=1" "GD_PRECOUNT=0"; do
  tag=$(echo $v | tr ' =.' '___')
  env $v timeout 300 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
done
