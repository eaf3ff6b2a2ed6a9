#!/bin/bash
# log_growth = 4 default: loop/scale tests, C5/C3 configs, bench line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_loop.py tests/test_gpu_scale.py tests/test_gpu_engine.py -x -q > gpurun_out/pytest_lg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lg.log
: > gpurun_out/configs_lg.jsonl
for c in c1_tc_rand c3_sg_tree c3_sg_tree_w1000 c3_sg_tree_w4000 c5_tc_dag; do
  timeout 600 python scripts/configs_bench.py $c >> gpurun_out/configs_lg.jsonl 2>> gpurun_out/configs_lg.err
done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_lg.json 2> gpurun_out/bench_lg.err
