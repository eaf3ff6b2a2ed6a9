#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_loop.py tests/test_gpu_partition.py -x -q > gpurun_out/pytest_loop.log 2>&1; tail -3 gpurun_out/pytest_loop.log
for m in 1 0; do
GD_PROBE_SCAN=$m timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_ps$m.json 2> gpurun_out/bench_ps$m.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_ps$m.json').read().strip().splitlines()[-1]); print('fused=$m', d['ms_per_step'], d['step_ms'], d['gpu_launches'], d['roofline']['kernel_ms_per_step'])"
done
