#!/bin/bash
# Round 2f: partition tests (loopback P=2..8 both exchanges), insert variants, C2 bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_partition.py -x -q -k "native_driver" > gpurun_out/pytest_part.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_part.log
for v in "GD_INSERT_SLOTS=1" "GD_INSERT_SLOTS=0" "GD_INSERT_SLOTS=1 GD_LOOP_SPLIT=1"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 --master-port=29533 bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --partitioned > gpurun_out/bench_part1.json 2> gpurun_out/bench_part1.err
