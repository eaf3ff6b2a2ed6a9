#!/bin/bash
# PDL A/B + loop tests; step-spike hunt with the loop trace.
mkdir -p gpurun_out
: > gpurun_out/spike_trace.txt
timeout 900 python scripts/spike_hunt.py 40 > gpurun_out/spike_hunt.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_loop.py -x -q > gpurun_out/pytest_pdl.log 2>&1; echo "default rc=$?" >> gpurun_out/pytest_pdl.log
GD_PDL=1 timeout 900 python -m pytest tests/test_gpu_loop.py tests/test_gpu_engine.py -x -q >> gpurun_out/pytest_pdl.log 2>&1; echo "pdl rc=$?" >> gpurun_out/pytest_pdl.log
timeout 900 python scripts/ab.py 'p1=pdl:1' 'p0=pdl:0' 'q1=pdl:1' 'q0=pdl:0' 5 > gpurun_out/ab_pdl.txt 2>&1
