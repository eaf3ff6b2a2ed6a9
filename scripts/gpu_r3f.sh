#!/bin/bash
# C4 near the explosion point: run-to-run behaviour at n = 1.2M (with and without trimming the cache between runs), 1.25M for contrast.
mkdir -p gpurun_out
timeout 600 python scripts/c4_probe.py 1.2 4 > gpurun_out/c4_probe_12.jsonl 2> gpurun_out/c4_probe_12.err
timeout 600 python scripts/c4_probe.py 1.2 4 --trim > gpurun_out/c4_probe_12t.jsonl 2> gpurun_out/c4_probe_12t.err
timeout 600 python scripts/c4_probe.py 1.25 4 > gpurun_out/c4_probe_125.jsonl 2> gpurun_out/c4_probe_125.err
timeout 600 python scripts/c4_probe.py 1.5 4 > gpurun_out/c4_probe_15.jsonl 2> gpurun_out/c4_probe_15.err
