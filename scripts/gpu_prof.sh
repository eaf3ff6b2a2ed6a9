#!/bin/bash
export GD_LOOP_MODE=eager
python scripts/prof_case.py c2log > gpurun_out/c2log.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:loop_ -s 30 -c 30 --csv --log-file gpurun_out/chain_launches.csv python scripts/prof_case.py chain > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loop_materialize_insert -s 300 -c 1 -o gpurun_out/insert_c2 python scripts/prof_case.py c2 > gpurun_out/ncu_insert.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loop_scan -s 300 -c 1 -o gpurun_out/scan_c2 python scripts/prof_case.py c2 > gpurun_out/ncu_scan.log 2>&1
