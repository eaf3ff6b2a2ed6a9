#!/bin/bash
# Pipelined download with run() returning before the segment sorts finish.
mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_pipe2.json 2> gpurun_out/bench_pipe2.err
GD_DL_PIPELINE=0 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_nopipe2.json 2> gpurun_out/bench_nopipe2.err
GD_DL_TRACE=1 timeout 600 python scripts/dl_sweep.py > gpurun_out/dl_sweep3.txt 2> gpurun_out/dl_sweep3.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
