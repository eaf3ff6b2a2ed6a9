#!/bin/bash
# Overlapped packing for the byte-offset download: tests, sweep, e2e with and without.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_download.py -x -q > gpurun_out/pytest_ov.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ov.log
GD_DL_TRACE=1 timeout 600 python scripts/dl_sweep.py > gpurun_out/dl_sweep_ov.txt 2> gpurun_out/dl_sweep_ov.err
GD_DL_OVERLAP=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-profile > gpurun_out/bench_ov1.json 2>/dev/null
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-profile > gpurun_out/bench_ov0.json 2>/dev/null
