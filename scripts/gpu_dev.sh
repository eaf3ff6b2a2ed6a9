#!/bin/bash
timeout 600 python scripts/run_configs.py c1_tc_rand c3_sg_tree c4_cspa > gpurun_out/configs.log 2>&1
GD_LOOP_MODE=eager timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/bench_ncu.log 2>&1
