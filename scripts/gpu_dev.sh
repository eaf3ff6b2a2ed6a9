#!/bin/bash
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_t.json 2> gpurun_out/bench_t.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_t.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['step_ms'], d['roofline']['kernel_ms_per_step'])"
