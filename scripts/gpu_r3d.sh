#!/bin/bash
# Flakiness check: the whole GPU suite twice, plus the round's bench line with the e2e warm-up.
mkdir -p gpurun_out
for k in 1 2; do
timeout 2400 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/pytest_gpu_$k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$k.log
done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final3.json 2> gpurun_out/bench_final3.err
