#!/bin/bash
# Round 2: peer-memory partition driver + pipelined sort: parity first, then the sort micro and C2 A/B.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_partition.py -x -q -k "native_driver" > gpurun_out/pytest_part.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_part.log
timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_download.py tests/test_gpu_reftests.py -x -q > gpurun_out/pytest_sort.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sort.log
timeout 600 python scripts/sort_micro.py 16 771 > gpurun_out/sort_micro.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pipe.json 2> gpurun_out/bench_pipe.err
GD_SORT_PIPE=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_classic.json 2> gpurun_out/bench_classic.err
GD_WARP_EXPAND=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_noxp.json 2> gpurun_out/bench_noxp.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 --master-port=29531 bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --partitioned > gpurun_out/bench_part1.json 2> gpurun_out/bench_part1.err
GD_LOOP_MODE=eager timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/prof_case.py c2 > gpurun_out/launches.log 2>&1
GD_LOOP_MODE=eager timeout 900 ncu --set full --clock-control none --import-source on -k regex:"loop_expand_insert" -s 400 -c 2 -o gpurun_out/prof_xins python scripts/prof_case.py c2 > gpurun_out/ncu_xins.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"onesweep" -s 2 -c 2 -o gpurun_out/prof_sort python scripts/prof_case.py c2 > gpurun_out/ncu_sort.log 2>&1
