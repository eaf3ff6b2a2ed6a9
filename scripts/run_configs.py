"""Time-to-fixpoint of the BASELINE configs on one B200 (EDB resident in
HBM): python scripts/run_configs.py c3_sg_tree c4_cspa ..."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_02206_b200 import arraylog as al  # noqa: E402
from paper_2311_02206_b200 import workloads as W  # noqa: E402

ctx = al.Context(0, torch.cuda.current_stream().cuda_stream)
for name in sys.argv[1:]:
    cfg = W.CONFIGS[name]
    edbs = cfg["gen"]()
    dev = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int64)).cuda() for k, v in edbs.items()}
    for rep in range(2):
        e = al.engine(cfg["program"], ctx=ctx)
        for k, v in edbs.items():
            e.load_edb_device(k, dev[k].data_ptr(), len(v))
        torch.cuda.synchronize()
        t = time.perf_counter()
        try:
            e.run()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            s = e.raw_stats()
            sizes = {n: e.relation_count(n) for n in e.idb_relations()}
            print(f"{name} rep {rep}: {dt*1e3:.1f} ms iterations {s.iterations} join_tuples {s.join_tuples} "
                  f"sizes {sizes} phases {e.stats().phase_seconds}", flush=True)
        except Exception as ex:  # noqa: BLE001
            print(f"{name} rep {rep}: FAILED after {time.perf_counter()-t:.1f}s: {ex}", flush=True)
        e.close()
