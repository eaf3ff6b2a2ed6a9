"""e2e download sweep on C2: direct-tail share x compression, 4 downloads each
(GD_DL_TRACE output on stderr): python scripts/dl_sweep.py"""
import ctypes as C
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
ctx = al.Context(0, s.cuda_stream, config={"trace": 2})
edges = W.tc_pl(5_000_000, 5_000_000, 200, 1.05, 1)
e = al.engine("reach", ctx=ctx)
e.load_edb("Edge", al.tuple_array(2, edges))
e.run()
n = e.relation_count("Reach")
out = torch.empty((n, 2), dtype=torch.int64).pin_memory().numpy().view(np.uint64)
rid = e._rid("Reach")
want = None
for delta, ov in ((2, 1), (2, 0), (1, 0), (0, 0)):
    for frac in ((0.0, 0.1) if delta == 2 else (0.0,)):
        ts = []
        for _ in range(4):
            with ctx.configured(download_delta=delta, download_direct_frac=frac, download_overlap_pack=ov):
                t = time.perf_counter()
                ctx.check(ctx.lib.gd_engine_relation_download(e.h, rid, out.ctypes.data_as(C.c_void_p), n))
                ts.append(time.perf_counter() - t)
        dig = int(out[::9973].sum())
        want = dig if want is None else want
        assert dig == want, "download differs between modes"
        print(f"delta={delta} overlap={ov} frac={frac}: " + " ".join(f"{x * 1e3:.0f}" for x in ts) + " ms", flush=True)
