#!/bin/bash
# One process per config (allocator caches do not carry between workloads).
: > gpurun_out/configs.jsonl
for c in c1_tc_rand c3_sg_tree c3_sg_tree_w1000 c3_sg_tree_w4000 c4_cspa c5_tc_dag; do
  timeout 600 python scripts/configs_bench.py $c >> gpurun_out/configs.jsonl 2>> gpurun_out/configs.err
done
timeout 900 python scripts/configs_bench.py c3_sg_tree_w4000 c5_tc_dag > gpurun_out/configs_shared.jsonl 2>> gpurun_out/configs.err
timeout 600 python -m pytest tests/test_gpu_loop.py tests/test_gpu_engine.py -x -q > gpurun_out/pytest_loop.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_loop.log
