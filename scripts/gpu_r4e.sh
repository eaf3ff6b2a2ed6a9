#!/bin/bash
# ncu --set full of the warp-expanded insert at a mid-run C2 iteration (J ~ 0.72 M) and of the count kernel.
mkdir -p gpurun_out
GD_LOOP_MODE=eager timeout 900 ncu --set full --clock-control none --import-source on -k regex:"loop_expand_insert" -s 505 -c 1 -o gpurun_out/prof_xins_r4 python scripts/prof_case.py c2 > gpurun_out/ncu_xins_r4.log 2>&1
GD_LOOP_MODE=eager timeout 900 ncu --set full --clock-control none --import-source on -k regex:"loop_count" -s 505 -c 1 -o gpurun_out/prof_cnt_r4 python scripts/prof_case.py c2 > gpurun_out/ncu_cnt_r4.log 2>&1
