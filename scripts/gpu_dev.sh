#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_loop.py -x -q -k "hash_predup or c1_all" > gpurun_out/pytest_loop.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_loop.log
timeout 300 python scripts/run_configs.py c4_cspa > gpurun_out/c4.log 2>&1
GD_HASH_DEDUP=0 timeout 300 python scripts/run_configs.py c4_cspa >> gpurun_out/c4.log 2>&1
