#!/bin/bash
for it in 16 8; do
GD_SORT_ITEMS=$it timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_s.json 2> gpurun_out/bench_s.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_s.json').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms_per_step']; print('items=$it', round(d['ms_per_step'],1), k['sort_pass'])"
done
