#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_loop.py tests/test_gpu_engine.py -q -rf -x -p no:cacheprovider > gpurun_out/pytest_zone.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_zone.log
timeout 300 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_zone.json 2> gpurun_out/bench_zone.err
GD_LOOP_MODE=eager timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"table_zone" --csv --log-file gpurun_out/zone.csv python scripts/prof_case.py c2 > /dev/null 2>&1
