#!/bin/bash
mkdir -p gpurun_out
GD_SORT_TRACE=1 timeout 300 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_sortadapt.json 2> gpurun_out/bench_sortadapt.err
GD_SORT_BALLOT=0 timeout 300 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_sortmatch.json 2> gpurun_out/bench_sortmatch.err
GD_SORT_TRACE=1 timeout 300 python scripts/sort_micro.py 200 > gpurun_out/sort_micro.log 2> gpurun_out/sort_micro.err
timeout 600 python -m pytest tests/test_gpu_sort.py -q -x -p no:cacheprovider > gpurun_out/pytest_sort.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sort.log
