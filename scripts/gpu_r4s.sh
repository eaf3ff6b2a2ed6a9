#!/bin/bash
# Big step outliers vs the nvidia-smi sampler: full default bench (20 steps), 3x with and 3x without sampling.
mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sp2_smi_$i.json 2>/dev/null
  GD_BENCH_CLOCK_MS=0 timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sp2_nosmi_$i.json 2>/dev/null
done
