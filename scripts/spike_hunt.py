"""Repeated C2 runs with the loop trace on (GD_LOOP_TRACE): device time per
run (CUDA events on the engine stream) and the host-side trace of the run,
printed whenever a run is more than 5% slower than the median so far
(python scripts/spike_hunt.py [runs])."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_02206_b200 import arraylog as al  # noqa: E402
from paper_2311_02206_b200 import workloads as W  # noqa: E402

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 30
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = al.Context(0, s.cuda_stream, config={"trace": 1})
edges = W.tc_pl(5_000_000, 5_000_000, 200, 1.05, 1)
d = torch.from_numpy(edges.view(np.int64)).cuda()
log = Path("gpurun_out/spike_trace.txt")
times = []
for r in range(runs):
    fd = os.open("/tmp/spike_run.txt", os.O_WRONLY | os.O_CREAT | os.O_TRUNC)
    saved = os.dup(2)
    os.dup2(fd, 2)
    try:
        e = al.engine("reach", ctx=ctx)
        e.load_edb_device("Edge", d.data_ptr(), len(edges))
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        e.run()
        b.record(s)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        e.close()
    finally:
        os.dup2(saved, 2)
        os.close(fd)
    times.append(ms)
    med = float(np.median(times))
    print(f"run {r}: {ms:.1f} ms (median {med:.1f})", flush=True)
    if r >= 3 and ms > 1.05 * med:
        with log.open("a") as f:
            f.write(f"=== run {r}: {ms:.1f} ms vs median {med:.1f}\n")
            f.write(Path("/tmp/spike_run.txt").read_text())
    if r == 3:
        with log.open("a") as f:
            f.write(f"=== reference run {r}: {ms:.1f} ms\n")
            f.write(Path("/tmp/spike_run.txt").read_text())
