#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_download.py -x -q > gpurun_out/pytest_dl4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dl4.log
GD_DL_TRACE=1 timeout 600 python scripts/dl_sweep.py > gpurun_out/dl_sweep6.txt 2> gpurun_out/dl_sweep6.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_chunk2.json 2> gpurun_out/bench_chunk2.err
