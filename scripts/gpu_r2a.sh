#!/bin/bash
# Round-2 first GPU session: full-scale golden records, GPU parity suite, bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/gpu.txt
timeout 1500 python tests/golden/make_scale_golden.py > gpurun_out/golden.log 2>&1; echo "golden rc=$?" >> gpurun_out/golden.log
cp tests/golden/scale_digests.json gpurun_out/ 2>/dev/null
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
