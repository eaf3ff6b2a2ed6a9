#!/bin/bash
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_t.json 2> gpurun_out/bench_t.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_t.json').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms_per_step']; print(round(d['ms_per_step'],1), d['step_ms'], k['sort_hist'], k['sort_pass'])"
timeout 900 python -m pytest tests/test_gpu_ra.py -x -q 2>&1 | tail -1
