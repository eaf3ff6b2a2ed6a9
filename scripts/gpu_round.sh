#!/bin/bash
# Round measurement session: parity suite, smoke, bench line, launch list,
# full ncu captures of the dominant loop kernels and of the final sort.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
GD_LOOP_MODE=eager timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/bench_ncu.log 2>&1
GD_LOOP_MODE=eager timeout 900 ncu --set full --clock-control none --import-source on -k regex:"loop_materialize_insert|loop_probe|loop_scan" -s 1500 -c 3 -o gpurun_out/prof_loop python scripts/prof_case.py c2 > gpurun_out/ncu_loop.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:onesweep -s 30 -c 1 -o gpurun_out/prof_sort python scripts/prof_case.py c2 > gpurun_out/ncu_sort.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:table_zone -s 2 -c 1 -o gpurun_out/prof_zone python scripts/prof_case.py c2 > gpurun_out/ncu_zone.log 2>&1
