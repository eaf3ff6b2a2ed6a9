"""Per-kernel-class device time of one BASELINE config
(python scripts/diag_config.py c4_cspa)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_02206_b200 import arraylog as al  # noqa: E402
from paper_2311_02206_b200 import workloads as W  # noqa: E402

name = sys.argv[1]
cfg = W.CONFIGS[name]
edbs = cfg["gen"]()
dev = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int64)).cuda() for k, v in edbs.items()}
ctx = al.Context(0, torch.cuda.current_stream().cuda_stream)
for rep in range(3):
    prof = rep == 2
    ctx.set_profiling(prof)
    ctx.profile_reset()
    e = al.engine(cfg["program"], ctx=ctx)
    for k, v in edbs.items():
        e.load_edb_device(k, dev[k].data_ptr(), len(v))
    torch.cuda.synchronize()
    t = time.perf_counter()
    e.run()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"rep {rep}{' (profiled)' if prof else ''}: {dt*1e3:.1f} ms, launches {ctx.kernel_launches}", flush=True)
    if prof:
        p = ctx.profile()
        print({k: (round(v[0], 1), v[1]) for k, v in p.items() if v[1]})
    e.close()
