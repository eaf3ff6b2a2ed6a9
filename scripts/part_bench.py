"""Partitioned mode on one GPU (LoopbackCluster, P logical shards) on C2:
time to fixpoint per P, loop-kernel path vs the sort/merge host path
(python scripts/part_bench.py [P ...])."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_02206_b200 import arraylog as al  # noqa: E402
from paper_2311_02206_b200 import workloads as W  # noqa: E402
from paper_2311_02206_b200.partition import LoopbackCluster  # noqa: E402

edges = W.tc_pl(5_000_000, 5_000_000, 200, 1.05, 1)
d = torch.from_numpy(edges.view(np.int64)).cuda()
ctx = al.Context(0, torch.cuda.current_stream().cuda_stream)
for P in [int(x) for x in sys.argv[1:]] or [1, 2]:
    for path in ("loop", "host"):
        os.environ["GD_PART_LOOP"] = "1" if path == "loop" else "0"
        ts = []
        for rep in range(2):
            engines = []
            for r in range(P):
                e = al.engine("reach", ctx=ctx)
                e.set_partition(r, P)
                e.load_edb_device("Edge", d.data_ptr(), len(edges))
                e.seed()
                engines.append(e)
            torch.cuda.synchronize()
            t = time.perf_counter()
            it = LoopbackCluster(engines).run()
            n = sum(e.relation_count("Reach") for e in engines)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t)
            for e in engines:
                e.close()
        print(f"P={P} {path:5s}: {min(ts)*1e3:8.1f} ms, {it} iterations, |Reach| {n} "
              f"({min(ts)/it*1e6:.0f} us/iteration for all shards, sequential on one GPU)", flush=True)
