#!/bin/bash
# Round 2 closing measurements with the byte-offset download default.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final4.json 2> gpurun_out/bench_final4.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref4.json 2> gpurun_out/bench_ref4.err
GD_DL_TRACE=1 timeout 600 python scripts/dl_sweep.py > gpurun_out/dl_sweep4.txt 2> gpurun_out/dl_sweep4.err
: > gpurun_out/configs4.jsonl
for c in c1_tc_rand c3_sg_tree c3_sg_tree_w1000 c3_sg_tree_w4000 c4_cspa c5_tc_dag; do
  timeout 600 python scripts/configs_bench.py $c >> gpurun_out/configs4.jsonl 2>> gpurun_out/configs4.err
done
GD_LOOP_MODE=eager timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches4.csv python scripts/prof_case.py c2 > gpurun_out/launches4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"byte_pack|byte_class" -c 2 -o gpurun_out/prof_pack4 python scripts/prof_case.py c2dl > gpurun_out/ncu_pack4.log 2>&1
