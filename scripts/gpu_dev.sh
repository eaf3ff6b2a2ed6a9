#!/bin/bash
GD_LOOP_TRACE=1 timeout 300 python scripts/diag.py 5e6 1.05 9 > gpurun_out/diag_trace.log 2>&1
timeout 600 python -m pytest tests/test_gpu_loop.py -x -q > gpurun_out/pytest_loop.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_loop.log
