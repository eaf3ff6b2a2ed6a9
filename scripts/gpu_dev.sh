#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_partition.py -x -q 2>&1 | tail -4
for drv in native python; do
GD_PART_DRIVER=$drv timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --partitioned --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_part.json 2> gpurun_out/bench_part.err
tail -2 gpurun_out/bench_part.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_part.json').read().strip().splitlines()[-1]); print('$drv', d['ms_per_step'], d['step_ms'], d['config']['parallelism'], d['config']['reach'], d['config']['iterations'], d['e2e']['seconds_per_step'])"
done
