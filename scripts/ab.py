"""A/B of gd_device_config options on C2 (same box, config after config,
best of N after the first):  python scripts/ab.py 'A=' 'B=split_insert:1,insert_waves:2' [reps]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_02206_b200 import arraylog as al  # noqa: E402
from paper_2311_02206_b200 import workloads as W  # noqa: E402

args = [a for a in sys.argv[1:] if "=" in a.split(",")[0] or a.endswith("=")]
reps = int(sys.argv[-1]) if sys.argv[-1].isdigit() else 4
configs = {}
for a in args:
    name, _, kv = a.partition("=")
    configs[name] = dict(x.split(":", 1) for x in kv.split(",") if x) if kv else {}
edges = W.tc_pl(5_000_000, 5_000_000, 200, 1.05, 1)
d = torch.from_numpy(edges.view(np.int64)).cuda()
ctx = al.Context(0, torch.cuda.current_stream().cuda_stream)
best = {k: 1e9 for k in configs}
for name, env in configs.items():  # config-major: alternating configs thrash the allocator
    for rep in range(reps):
        cfg = {k: (float(v) if "." in v else int(v)) for k, v in env.items()}
        with ctx.configured(**cfg):
            e = al.engine("reach", ctx=ctx)
            e.load_edb_device("Edge", d.data_ptr(), len(edges))
            torch.cuda.synchronize()
            t = time.perf_counter()
            e.run()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            n = e.relation_count("Reach")
            e.close()
        if rep > 0:
            best[name] = min(best[name], dt)
        print(f"rep {rep} {name:10s} {dt*1e3:8.1f} ms |Reach| {n}", flush=True)
print({k: round(v * 1e3, 1) for k, v in best.items()})
