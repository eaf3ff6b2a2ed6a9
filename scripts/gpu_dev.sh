#!/bin/bash
timeout 900 python scripts/configs_bench.py c4_cspa c3_sg_tree_w4000 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['workload'], round(d['time_to_fixpoint_s']*1e3,1), 'ms')"
timeout 900 python -m pytest tests/test_gpu_engine.py -x -q -k "cspa or dedup" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_loop.py -x -q -k "dedup" 2>&1 | tail -1
