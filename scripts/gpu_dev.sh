#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_download.py -x -q 2>&1 | tail -3
for f in 0 0.25 0.35; do
GD_DL_DIRECT_FRAC=$f GD_DL_TRACE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-profile > gpurun_out/bench_dl.json 2> gpurun_out/bench_dl.err
grep download gpurun_out/bench_dl.err | tail -2
python -c "
import json; d=json.loads(open('gpurun_out/bench_dl.json').read().strip().splitlines()[-1]); print('frac=$f', round(d['ms_per_step'],1), d['e2e']['seconds_per_step'], d['e2e']['d2h_bytes_per_step'])"
done
