#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_loop.py -x -q > gpurun_out/pytest_loop.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_loop.log
timeout 300 python scripts/diag.py 5e6 1.05 1 > gpurun_out/diag.log 2>&1
timeout 300 python scripts/run_configs.py c4_cspa > gpurun_out/c4.log 2>&1
