#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_download.py -x -q > gpurun_out/pytest_dl.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dl.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-profile > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
GD_HOST_UNPACK=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-profile > gpurun_out/bench_quick0.json 2>> gpurun_out/bench_quick.err
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
