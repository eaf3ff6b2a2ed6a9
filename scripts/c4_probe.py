"""CSPA run-to-run probe: cspa_local(n) run several times in one process
(EDB resident), printing per run the device time, the engine's phase and
kernel-class times (profiling on for the runs after the first two), the
allocator / sync host counters and free HBM — to see what a later run does
differently from the first one near the memory limit.

    python scripts/c4_probe.py 1.2 [runs] [--trim]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_02206_b200 import arraylog as al  # noqa: E402
from paper_2311_02206_b200 import workloads as W  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
n = int(float(args[0]) * 1e6) if args else 1_200_000
runs = int(args[1]) if len(args) > 1 else 3
trim = "--trim" in sys.argv
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = al.Context(0, s.cuda_stream)
a, d = W.cspa_local(n, 362_000, 1_140_000, 256, 1)
dev = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int64)).cuda() for k, v in (("assign", a), ("dereference", d))}
for rep in range(runs):
    prof = rep >= 2
    if prof:
        ctx.set_profiling(True)
        ctx.profile_reset()
    h0 = ctx.host_counters()
    free0 = torch.cuda.mem_get_info()[0]
    e = al.engine("cspa", ctx=ctx)
    for k, v in dev.items():
        e.load_edb_device(k, v.data_ptr(), v.numel() // 2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    e.run()
    e1.record(s)
    torch.cuda.synchronize()
    st = e.stats()
    raw = e.raw_stats()
    h1 = ctx.host_counters()
    rec = {"n": n, "run": rep, "time_s": e0.elapsed_time(e1) / 1e3, "iterations": st.iterations,
           "phases_s": {k: round(v, 4) for k, v in st.phase_seconds.items()},
           "device_bytes_peak": int(raw.device_bytes_peak), "peak_temp_bytes": int(raw.peak_temp_bytes),
           "host": {k: round(h1[k] - h0[k], 4) for k in h0}, "free_before_gb": round(free0 / 1e9, 2),
           "sizes": {r: e.relation_count(r) for r in e.idb_relations()}}
    if prof:
        rec["kernels_ms"] = {k: round(v[0], 2) for k, v in ctx.profile().items() if v[0]}
        ctx.set_profiling(False)
    e.close()
    if trim:
        ctx.trim()
    print(json.dumps(rec), flush=True)
