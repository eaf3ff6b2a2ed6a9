#!/bin/bash
# Round 2d: targeted hang check, insert variants, sort variants on C2.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
GD_LOOP_TRACE=1 timeout 120 python -m pytest tests/test_gpu_loop.py -x -q -k "sg_corpus_modes and window" > gpurun_out/pytest_window.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_window.log
timeout 300 python scripts/sort_micro.py 200 771 > gpurun_out/sort_micro.log 2>&1
for v in "GD_INSERT_SLOTS=2" "GD_INSERT_SLOTS=1" "GD_INSERT_SLOTS=4" "GD_LOOP_SPLIT=1" "GD_LOOP_SPLIT=1 GD_INSERT_SLOTS=1" "GD_SORT_PIPE=4"; do
  tag=$(echo $v | tr ' =' '__')
  env GD_SORT_PIPE=0 $v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
done
