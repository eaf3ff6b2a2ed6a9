#!/bin/bash
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_w.json 2> gpurun_out/bench_w.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_w.json').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms_per_step']; print('C2', round(d['ms_per_step'],1), d['step_ms'], k['join_insert'])"
timeout 900 python scripts/configs_bench.py c1_tc_rand c3_sg_tree c3_sg_tree_w4000 c5_tc_dag 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['workload'], round(d['time_to_fixpoint_s']*1e3,1), 'ms')"
timeout 900 python -m pytest tests/test_gpu_loop.py -x -q 2>&1 | tail -1
