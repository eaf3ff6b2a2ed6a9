"""Wall time of the resident loop per launch mode (graph / batch / eager /
host-driven) on a long chain (tiny iterations: pure per-iteration
overhead) and on C2 (python scripts/loop_modes.py [c2])."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_02206_b200 import arraylog as al  # noqa: E402
from paper_2311_02206_b200 import workloads as W  # noqa: E402

_s = torch.cuda.Stream()
torch.cuda.set_stream(_s)
ctx = al.Context(0, _s.cuda_stream)
cases = {"chain3000": np.stack([np.arange(2999), np.arange(1, 3000)], 1).astype(np.uint64)}
if len(sys.argv) > 1:
    cases["c2"] = W.tc_pl(5_000_000, 5_000_000, 200, 1.05, 1)
modes = {"graph": {"loop_mode": 0}, "batch16": {"loop_mode": 2, "loop_batch": 16},
         "batch64": {"loop_mode": 2, "loop_batch": 64}, "eager": {"loop_mode": 1},
         "host": {"resident_loop": 0}, "graph_noxp": {"loop_mode": 0, "warp_expand": 0}}
for name, edges in cases.items():
    d = torch.from_numpy(edges.view(np.int64)).cuda()
    for m, kv in modes.items():
        ctx.set_config(**{"loop_mode": 0, "loop_batch": 16, "resident_loop": 1, "warp_expand": 1, **kv})
        ts = []
        for rep in range(3):
            e = al.engine("reach", ctx=ctx)
            e.load_edb_device("Edge", d.data_ptr(), len(edges))
            torch.cuda.synchronize()
            t = time.perf_counter()
            e.run()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t)
            it = e.stats().iterations
            cnt = e.relation_count("Reach")
            e.close()
        print(f"{name:10s} {m:8s} iters {it:5d} |Reach| {cnt:11d}  best {min(ts)*1e3:8.1f} ms  "
              f"({min(ts)/it*1e6:7.1f} us/iter)", flush=True)
