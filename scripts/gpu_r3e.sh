#!/bin/bash
# A/B (builds under exp/, made locally for this call): (1) next-round row prefetch in the warp-expanded insert: exp/base (without) vs the default build;
# (2) the download's dynamic work units: exp/pf (barrier per chunk) vs the default build, e2e;
# (3) C4 calibration sweep.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_download.py -x -q > gpurun_out/pytest_dl.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dl.log
for k in 1 2; do
GDLOG_B200_LIB=exp/base/libgdlog_b200.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_base_$k.json 2> gpurun_out/ab_base_$k.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_pf_$k.json 2> gpurun_out/ab_pf_$k.err
done
for k in 1 2; do
GDLOG_B200_LIB=exp/pf/libgdlog_b200.so timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_old_$k.json 2> gpurun_out/e2e_old_$k.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_new_$k.json 2> gpurun_out/e2e_new_$k.err
done
timeout 2400 python scripts/cspa_calibrate.py 1.45 1.4 1.35 1.3 1.25 1.2 1.15 1.1 > gpurun_out/cspa_cal.jsonl 2> gpurun_out/cspa_cal.err
