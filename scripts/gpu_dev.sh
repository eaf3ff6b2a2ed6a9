#!/bin/bash
for i in 1 2; do GD_BENCH_CANARY=1 GD_BENCH_CLOCK_MS=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-profile --no-e2e 2>/dev/null; done > gpurun_out/bench_q8.jsonl
