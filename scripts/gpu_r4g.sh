#!/bin/bash
# Stamp update by atomicMax in the fast path; index load limit / growth sweep.
mkdir -p gpurun_out
timeout 900 python scripts/ab.py 'base=' 'l40g6=index_load_pct:40,index_growth:6' 'l35g8=index_load_pct:35,index_growth:8' 'l25g8=index_load_pct:25,index_growth:8' 'l25g12=index_load_pct:25,index_growth:12' 4 > gpurun_out/ab_load.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_loop.py -x -q > gpurun_out/pytest_loop.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_loop.log
