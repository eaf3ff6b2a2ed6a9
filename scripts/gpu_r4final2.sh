#!/bin/bash
# End-of-round validation with the final defaults: full GPU suite, smoke, bench line, launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_end.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_end.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_end.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_end.json 2> gpurun_out/bench_end.err
GD_LOOP_MODE=eager timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_end.csv python scripts/prof_case.py c2 > gpurun_out/launches_end.log 2>&1
