#!/bin/bash
# Round 2d: insert variants (bucket slots 1/2/4, split insert) and sort variants on C2.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_loop.py tests/test_gpu_sort.py -q -x -k "c1_all_modes or sg_corpus or sort" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
for v in "GD_INSERT_SLOTS=2" "GD_INSERT_SLOTS=1" "GD_INSERT_SLOTS=4" "GD_LOOP_SPLIT=1" "GD_SORT_PIPE=0" "GD_SORT_PIPE=1 GD_SORT_DIGIT_BITS=8" "GD_SORT_PIPE=2"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
done
