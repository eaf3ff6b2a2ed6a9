#!/bin/bash
for gf in 6 8; do
GD_TAB_GROWTH=$gf timeout 900 python scripts/configs_bench.py c1_tc_rand c3_sg_tree c3_sg_tree_w1000 c3_sg_tree_w4000 c5_tc_dag 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('gf=$gf', d['workload'], round(d['time_to_fixpoint_s']*1e3,1), 'ms')"
done
