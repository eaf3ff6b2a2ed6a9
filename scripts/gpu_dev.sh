#!/bin/bash
GD_LOOP_TRACE=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/bench_z0.json 2> gpurun_out/bench_z0.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_z0.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['step_ms'], [x['index'] for x in d['step_phases_ms']])"
grep -E "block|tab-|log " gpurun_out/bench_z0.err | awk '{ if ($0 ~ /gpu/ && $(NF-1)+0 > 15) print "BIG", $0; }' | tail -50
grep block gpurun_out/bench_z0.err | tail -2
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_full.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['step_ms'], d['e2e']['seconds_per_step'], [x['index'] for x in d['step_phases_ms']])"
