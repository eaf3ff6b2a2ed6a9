#!/bin/bash
# Round 2h: L2 fetch granularity (micro + C2), batched expansion variants.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
for g in 32 64 128; do timeout 120 ./scripts/micro/random_access $g 8192 > gpurun_out/ra_gran$g.txt 2>&1; done
for v in "GD_L2_FETCH=32" "GD_L2_FETCH=64" "GD_L2_FETCH=128" "GD_INSERT_SLOTS=1" "GD_LOOP_SPLIT=1" "GD_LOOP_SPLIT=1 GD_L2_FETCH=32"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
done
