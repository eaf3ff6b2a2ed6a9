"""Host-side timeline of the segmented final sort on C2 (GD_SORT_TRACE=1):
when run() returns relative to the device work it queued."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_02206_b200 import arraylog as al  # noqa: E402
from paper_2311_02206_b200 import workloads as W  # noqa: E402

s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = al.Context(0, s.cuda_stream, config={"trace": 4})
edges = W.tc_pl(5_000_000, 5_000_000, 200, 1.05, 1)
d = torch.from_numpy(edges.view(np.int64)).cuda()
for rep in range(3):
    e = al.engine("reach", ctx=ctx)
    e.load_edb_device("Edge", d.data_ptr(), len(edges))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e.run()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rep {rep}: run() returned after {1e3 * (t1 - t0):.1f} ms, device done after {1e3 * (t2 - t0):.1f} ms",
          file=sys.stderr, flush=True)
    e.close()
