#!/bin/bash
cp paper_2311_02206_b200/lib/libgdlog_b200.so /tmp/libgd_orig.so
for v in occ6 occ5 occ7 occ6; do
cp paper_2311_02206_b200/lib/variants/lib_$v.so paper_2311_02206_b200/lib/libgdlog_b200.so
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_v.json 2> gpurun_out/bench_v.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_v.json').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms_per_step']; print('$v', round(d['ms_per_step'],1), k['join_insert'])"
done
cp /tmp/libgd_orig.so paper_2311_02206_b200/lib/libgdlog_b200.so
