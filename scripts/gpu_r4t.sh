#!/bin/bash
# Log growth factor A/B on C2 (fewer rollbacks), trace of the rollbacks at 2x and 4x.
mkdir -p gpurun_out
timeout 900 python scripts/ab.py 'l2=log_growth:2' 'l4=log_growth:4' 'l8=log_growth:8' 'm2=log_growth:2' 'm4=log_growth:4' 5 > gpurun_out/ab_loggrowth.txt 2>&1
GD_LOOP_TRACE=1 GD_LOG_GROWTH=4 timeout 300 python scripts/prof_case.py c2 > gpurun_out/trace_lg4.txt 2>&1
