#!/bin/bash
# Per-iteration cost analysis of C2: iteration log, eager launch list with
# per-launch durations, near-empty-iteration cost (chain of 3000).
mkdir -p gpurun_out
timeout 300 python scripts/iter_log_dump.py > gpurun_out/iter_log.txt 2>&1
timeout 300 python scripts/loop_modes.py > gpurun_out/loop_modes.txt 2>&1
GD_LOOP_MODE=eager timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r4.csv python scripts/prof_case.py c2 > gpurun_out/launches_r4.log 2>&1
