#!/bin/bash
mkdir -p gpurun_out
for v in "GD_SORT_BALLOT=1" "GD_SORT_BALLOT=0" "GD_SORT_BALLOT=1 GD_SORT_MIN_CTAS=4"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
done
timeout 900 python -m pytest tests/test_gpu_partition.py tests/test_gpu_sort.py -q -rf -k "native_driver or sort" -p no:cacheprovider > gpurun_out/pytest_part.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_part.log
timeout 1200 python tests/golden/make_scale_golden.py c5_tc_dag > gpurun_out/golden_c5.log 2>&1; echo "rc=$?" >> gpurun_out/golden_c5.log
cp tests/golden/scale_digests.json gpurun_out/scale_digests.json
