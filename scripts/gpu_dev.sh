#!/bin/bash
timeout 900 ncu --set full --clock-control none -k regex:"dedup_insert|part_scatter" -s 40 -c 2 -o gpurun_out/prof_dedup python scripts/configs_bench.py c4_cspa > gpurun_out/ncu_dedup.log 2>&1
