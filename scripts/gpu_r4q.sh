#!/bin/bash
# Chunked final steps in the host-driven loop: parity tests, then C4 at and beyond the size that exhausted HBM.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py -x -q -k "chunked or cspa or budget" > gpurun_out/pytest_chunk.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_chunk.log
timeout 300 python scripts/configs_bench.py c4_cspa > gpurun_out/c4_default.jsonl 2> gpurun_out/c4_default.err
for n in 1.15 1.1 1.05; do
  GD_LOOP_TRACE=0 timeout 420 python scripts/c4_probe.py $n 2 > gpurun_out/c4_chunk_$n.jsonl 2> gpurun_out/c4_chunk_$n.err
done
