#!/bin/bash
mkdir -p gpurun_out
for v in "GD_LOOP_SPLIT=1 GD_INSERT_PIPE=1" "GD_LOOP_SPLIT=1 GD_INSERT_PIPE=0"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
done
GD_LOOP_MODE=eager GD_LOOP_SPLIT=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"insert_keys" -s 500 -c 2 -o gpurun_out/prof_ikp python scripts/prof_case.py c2 > gpurun_out/ncu_ikp.log 2>&1
