#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_loop.py -x -q > gpurun_out/pytest_loop.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_loop.log
GD_LOOP_TRACE=1 timeout 900 python scripts/run_configs.py c5_tc_dag > gpurun_out/c5.log 2>&1
nvidia-smi --query-gpu=memory.total,memory.used --format=csv >> gpurun_out/c5.log
