#!/bin/bash
# Host side of the download: topology and write bandwidth into pinned memory.
mkdir -p gpurun_out
( lscpu; echo; nproc; cat /sys/fs/cgroup/cpu.max 2>/dev/null; numactl -H 2>/dev/null; free -g ) > gpurun_out/host_topo.txt 2>&1
timeout 300 scripts/micro/host_bw 12 > gpurun_out/host_bw.txt 2>&1
