#!/bin/bash
# Segmented final sort + pipelined download: download tests, loop tests, sweep, bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_download.py -x -q > gpurun_out/pytest_dl2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dl2.log
timeout 600 python scripts/dl_sweep.py > gpurun_out/dl_sweep2.txt 2> gpurun_out/dl_sweep2.err
timeout 900 python bench.py > gpurun_out/bench_pipe.json 2> gpurun_out/bench_pipe.err
GD_DL_PIPELINE=0 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_nopipe.json 2> gpurun_out/bench_nopipe.err
