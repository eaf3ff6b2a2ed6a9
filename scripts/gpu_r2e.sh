#!/bin/bash
# Round 2e: L2 hints on the head index, sort pipe with static tiles, loopback P=8 peer exchange.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python scripts/sort_micro.py 200 771 > gpurun_out/sort_micro.log 2>&1
for v in "GD_L2_HINTS=1" "GD_L2_HINTS=0" "GD_L2_HINTS=2" "GD_L2_HINTS=1 GD_INSERT_SLOTS=2" "GD_L2_HINTS=1 GD_LOOP_SPLIT=1"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
done
timeout 600 python -m pytest tests/test_gpu_partition.py -x -q -k "multi_rank_loopback and 8-46" > gpurun_out/pytest_p8.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p8.log
