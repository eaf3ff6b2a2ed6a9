#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf -x -p no:cacheprovider -k "not full_scale" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1800 python -m pytest tests/test_gpu_scale.py -q -rf -p no:cacheprovider -k "full_scale" > gpurun_out/pytest_scale.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_scale.log
