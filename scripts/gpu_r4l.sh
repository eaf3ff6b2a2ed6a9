#!/bin/bash
# Download packed per 16 M-row chunk with events (host rebuild starts on chunk 0 while the device packs the rest).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_download.py -x -q > gpurun_out/pytest_dl3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dl3.log
GD_DL_TRACE=1 timeout 600 python scripts/dl_sweep.py > gpurun_out/dl_sweep5.txt 2> gpurun_out/dl_sweep5.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_chunk.json 2> gpurun_out/bench_chunk.err
timeout 900 ncu --set full --clock-control none -k regex:"byte_pack|byte_class" -c 2 -o gpurun_out/prof_pack5 python scripts/prof_case.py c2dl > gpurun_out/ncu_pack5.log 2>&1
