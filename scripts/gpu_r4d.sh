#!/bin/bash
# Byte-offset download: download tests, C2 download sweep, bench line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_download.py -x -q > gpurun_out/pytest_dl.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dl.log
timeout 600 python scripts/dl_sweep.py > gpurun_out/dl_sweep.txt 2> gpurun_out/dl_sweep.err
timeout 900 python bench.py > gpurun_out/bench_dl.json 2> gpurun_out/bench_dl.err
