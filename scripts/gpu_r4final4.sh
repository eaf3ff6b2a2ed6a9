#!/bin/bash
# Closing validation with the final defaults (log_growth 4, gate in the insert, byte-offset download).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_last.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_last.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_last.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_last.json 2> gpurun_out/bench_last.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_last.json 2> gpurun_out/bench_ref_last.err
: > gpurun_out/configs_last.jsonl
for c in c1_tc_rand c3_sg_tree c3_sg_tree_w1000 c3_sg_tree_w4000 c4_cspa c5_tc_dag; do
  timeout 600 python scripts/configs_bench.py $c >> gpurun_out/configs_last.jsonl 2>> gpurun_out/configs_last.err
done
GD_LOOP_MODE=eager timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_last.csv python scripts/prof_case.py c2 > gpurun_out/launches_last.log 2>&1
