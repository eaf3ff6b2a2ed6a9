"""Per-phase host wall time vs device kernel time of one C2 run
(diagnostics: python scripts/diag.py [n] [alpha] [profile_rep])."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_02206_b200 import arraylog as al  # noqa: E402
from paper_2311_02206_b200 import workloads as W  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 5_000_000
alpha = float(sys.argv[2]) if len(sys.argv) > 2 else 1.05
prof_rep = int(sys.argv[3]) if len(sys.argv) > 3 else 3
edges = W.tc_pl(n, n, 200, alpha, 1)
d = torch.from_numpy(edges.view(np.int64)).cuda()
ctx = al.Context(0, torch.cuda.current_stream().cuda_stream)
for rep in range(4):
    ctx.set_profiling(rep == prof_rep)
    ctx.profile_reset()
    h0 = ctx.host_counters()
    l0 = ctx.kernel_launches
    e = al.engine("reach", ctx=ctx)
    e.load_edb_device("Edge", d.data_ptr(), len(edges))
    torch.cuda.synchronize()
    t = time.perf_counter()
    e.run()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    s = e.stats()
    h1 = ctx.host_counters()
    print(f"rep {rep}: wall {dt*1e3:.1f} ms  iters {s.iterations}  reach {e.relation_count('Reach')}  "
          f"phases(ms) " + " ".join(f"{k}={v*1e3:.1f}" for k, v in s.phase_seconds.items()) +
          f" | allocs {h1['allocs']-h0['allocs']} ({(h1['alloc_s']-h0['alloc_s'])*1e3:.1f} ms)"
          f" syncs {h1['syncs']-h0['syncs']} ({(h1['sync_s']-h0['sync_s'])*1e3:.1f} ms)"
          f" launches {ctx.kernel_launches-l0}", flush=True)
    if rep == prof_rep:
        pr = ctx.profile()
        print("kernels(ms):", {k: round(v[0], 1) for k, v in pr.items()})
    e.close()
