#!/bin/bash
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt; lscpu | grep -E "Socket|NUMA|Thread|Core" >> gpurun_out/host.txt
GD_DL_TRACE=1 timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_dl.json 2> gpurun_out/bench_dl.err
python - > gpurun_out/hostbw.txt 2>&1 <<'PY'
import numpy as np, time, threading
n = 1 << 30  # 8 GB of u64
a = np.empty(n, dtype=np.uint64)
t = time.perf_counter(); a.fill(1); dt = time.perf_counter() - t
print(f"1-thread fill 8 GB: {8/dt:.1f} GB/s")
PY
