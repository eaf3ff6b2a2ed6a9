#!/bin/bash
# Gate evaluated inside the insert kernel (gate_in_insert): loop tests + A/B on C2.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_loop.py tests/test_gpu_engine.py -x -q > gpurun_out/pytest_gate.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gate.log
timeout 900 python scripts/ab.py 'g1=gate_in_insert:1' 'g0=gate_in_insert:0' 'h1=gate_in_insert:1' 'h0=gate_in_insert:0' 5 > gpurun_out/ab_gate.txt 2>&1
timeout 300 python scripts/loop_modes.py > gpurun_out/loop_modes_gate.txt 2>&1
