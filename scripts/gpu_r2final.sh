#!/bin/bash
# Round 2 measurement session: full GPU suite (incl. full-scale digests), bench line, configs, launch list, ncu.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
: > gpurun_out/configs.jsonl
for c in c1_tc_rand c3_sg_tree c3_sg_tree_w1000 c3_sg_tree_w4000 c4_cspa c5_tc_dag; do
  timeout 600 python scripts/configs_bench.py $c >> gpurun_out/configs.jsonl 2>> gpurun_out/configs.err
done
GD_LOOP_MODE=eager timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/prof_case.py c2 > gpurun_out/launches.log 2>&1
GD_LOOP_MODE=eager timeout 900 ncu --set full --clock-control none --import-source on -k regex:"loop_materialize_insert" -s 400 -c 2 -o gpurun_out/prof_mins python scripts/prof_case.py c2 > gpurun_out/ncu_mins.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"onesweep" -s 30 -c 2 -o gpurun_out/prof_sort python scripts/prof_case.py c2 > gpurun_out/ncu_sort.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -rf --durations=30 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
