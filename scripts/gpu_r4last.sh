#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_zz.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_zz.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_zz.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_zz.json 2> gpurun_out/bench_zz.err
