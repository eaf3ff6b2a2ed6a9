#!/bin/bash
# Step spikes: bench with and without the nvidia-smi clock sampler in the timed region.
mkdir -p gpurun_out
for i in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/spk_smi_$i.json 2>/dev/null
  GD_BENCH_CLOCK_MS=0 timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/spk_nosmi_$i.json 2>/dev/null
done
GD_BENCH_CLOCK_MS=1000 timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/spk_smi1000.json 2>/dev/null
