#!/bin/bash
# Count ahead (no loop_count in the graph iteration): loop/engine/scale tests + A/B on C2.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_loop.py tests/test_gpu_engine.py tests/test_gpu_scale.py -x -q > gpurun_out/pytest_ca.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ca.log
timeout 900 python scripts/ab.py 'a1=count_ahead:1' 'a0=count_ahead:0' 'b1=count_ahead:1' 'b0=count_ahead:0' 5 > gpurun_out/ab_ca.txt 2>&1
timeout 300 python scripts/loop_modes.py > gpurun_out/loop_modes_ca.txt 2>&1
