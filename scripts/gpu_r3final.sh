#!/bin/bash
# Round 2 closing measurements with the final defaults.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err
: > gpurun_out/configs2.jsonl
for c in c1_tc_rand c3_sg_tree c3_sg_tree_w1000 c3_sg_tree_w4000 c4_cspa c5_tc_dag; do
  timeout 600 python scripts/configs_bench.py $c >> gpurun_out/configs2.jsonl 2>> gpurun_out/configs2.err
done
GD_LOOP_MODE=eager timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches2.csv python scripts/prof_case.py c2 > gpurun_out/launches2.log 2>&1
GD_LOOP_MODE=eager timeout 900 ncu --set full --clock-control none --import-source on -k regex:"loop_expand_insert" -s 400 -c 2 -o gpurun_out/prof_xins2 python scripts/prof_case.py c2 > gpurun_out/ncu_xins2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"onesweep" -s 33 -c 2 -o gpurun_out/prof_sort2 python scripts/prof_case.py c2 > gpurun_out/ncu_sort2.log 2>&1
