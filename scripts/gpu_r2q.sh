#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_download.py -q -rf -p no:cacheprovider > gpurun_out/pytest_dl.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dl.log
for v in "GD_DL_DIRECT_FRAC=0.1" "GD_DL_DIRECT_FRAC=0.15" "GD_DL_DIRECT_FRAC=0.2" "GD_SORT_PIPE=1 GD_SORT_DIGIT_BITS=8"; do
  tag=$(echo $v | tr ' =.' '___')
  env GD_DL_TRACE=1 $v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 --master-port=29537 bench.py --steps 3 --warmup 2 --no-cpu-baseline --partitioned > gpurun_out/bench_part1.json 2> gpurun_out/bench_part1.err
