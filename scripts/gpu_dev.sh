#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_loop.py -x -q -k "hash_predup" > gpurun_out/pytest_loop.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_loop.log
timeout 300 python scripts/configs_bench.py c4_cspa > gpurun_out/c4.jsonl 2>&1
GD_DEDUP_SPLIT=0 timeout 300 python scripts/configs_bench.py c4_cspa >> gpurun_out/c4.jsonl 2>&1
timeout 300 python scripts/diag_config.py c4_cspa > gpurun_out/diag_c4.log 2>&1
