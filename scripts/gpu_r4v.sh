#!/bin/bash
# Unrolled log-growth copy: growth trace + A/B-free bench (same box comparisons via the trace's gpu times).
mkdir -p gpurun_out
GD_LOOP_TRACE=1 timeout 300 python scripts/prof_case.py c2 > gpurun_out/trace_copy.txt 2>&1
timeout 900 python scripts/ab.py 'x=' 'y=' 4 > gpurun_out/ab_copy.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_loop.py -x -q > gpurun_out/pytest_copy.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_copy.log
