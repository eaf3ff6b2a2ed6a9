#!/bin/bash
GD_HOST_UNPACK=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-profile > gpurun_out/bench_dl.json 2> gpurun_out/bench_dl.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_dl.json').read().strip().splitlines()[-1]); print('direct', d['ms_per_step'], d['e2e'])"
nvidia-smi -q | grep -A3 -i "Link Width\|PCIe Generation" | head -12
