#!/bin/bash
mkdir -p gpurun_out
for b in 0 1; do
GD_SORT_BALLOT=$b timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"onesweep" --csv --log-file gpurun_out/sortpass_$b.csv python scripts/prof_case.py c2 > /dev/null 2>&1
done
GD_SORT_PIPE=4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"onesweep" --csv --log-file gpurun_out/sortpass_4.csv python scripts/prof_case.py c2 > /dev/null 2>&1
