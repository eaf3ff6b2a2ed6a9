#!/bin/bash
# N > 1 bench path at one rank (torchrun): native driver vs torch.distributed protocol
for drv in native python; do
GD_PART_DRIVER=$drv timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --partitioned --steps 3 --warmup 3 --no-cpu-baseline 2> gpurun_out/bench_part_$drv.err | tail -1 > gpurun_out/bench_part_$drv.json
done
