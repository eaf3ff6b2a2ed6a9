#!/bin/bash
for s in 8388608 16777216 33554432 67108864; do
GD_DEDUP_L2_SLOTS=$s timeout 900 python scripts/configs_bench.py c4_cspa 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('slots=$s', d['workload'], round(d['time_to_fixpoint_s']*1e3,1), 'ms')"
done
GD_DEDUP_SPLIT=0 timeout 900 python scripts/configs_bench.py c4_cspa 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('nosplit', d['workload'], round(d['time_to_fixpoint_s']*1e3,1), 'ms')"
