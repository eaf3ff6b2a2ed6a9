#!/bin/bash
# heavy_rows sweep on C2 (warp-expanded insert: per-warp work imbalance).
mkdir -p gpurun_out
timeout 900 python scripts/ab.py 'h4096=heavy_rows:4096' 'h1024=heavy_rows:1024' 'h512=heavy_rows:512' 'h256=heavy_rows:256' 'h128=heavy_rows:128' 'h64=heavy_rows:64' 'h32=heavy_rows:32' 4 > gpurun_out/ab_heavy.txt 2>&1
