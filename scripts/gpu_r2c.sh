#!/bin/bash
# Round 2c: sort variants (micro), full GPU suite, C2 bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 600 python scripts/sort_micro.py 16 200 771 > gpurun_out/sort_micro.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf -x --durations=20 -k "not full_scale" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
