#!/bin/bash
# Round 2g: P=8 tiny peer loopback diagnostics (isolated), split-mode launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_partition.py -x -q -k "multi_rank_loopback and 8-46 and True" > gpurun_out/pytest_p8t.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p8t.log
GD_LOOP_MODE=eager GD_LOOP_SPLIT=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_split.csv python scripts/prof_case.py c2 > gpurun_out/launches_split.log 2>&1
