#!/bin/bash
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --partitioned --steps 3 --warmup 3 --no-cpu-baseline 2> gpurun_out/bench_part_native.err | tail -1 > gpurun_out/bench_part_native.json
python -c "
import json; d=json.loads(open('gpurun_out/bench_part_native.json').read()); print(round(d['ms_per_step'],1), d['step_ms'], d['config']['parallelism'], d['config']['reach'], round(d['e2e']['seconds_per_step'],3))"
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 2>/dev/null | tail -1 | cut -c1-300
