#!/bin/bash
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_s.json 2> gpurun_out/bench_s.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_s.json').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms_per_step']; print('portion28', round(d['ms_per_step'],1), d['step_ms'], k['sort_pass'])"
timeout 900 python scripts/configs_bench.py c5_tc_dag 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['workload'], round(d['time_to_fixpoint_s']*1e3,1), 'ms')"
timeout 900 python -m pytest tests/test_gpu_ra.py -x -q -k "sort or canonical" 2>&1 | tail -1
