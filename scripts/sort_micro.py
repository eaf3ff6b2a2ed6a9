"""Radix sort micro-benchmark on device keys (gd_sort_keys_device):
classic onesweep (sort_pipeline=0) vs the pipelined kernel at 8/9/10-bit
digits, on uniform 46-bit keys and on C2-shaped keys (the final Reach
relation's packed keys when --c2 is given).  Checks every result against
torch.sort.  CUDA-event times on the context stream, L2 flushed between
runs.

    python scripts/sort_micro.py [n_millions ...] [--c2]
"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2311_02206_b200 import arraylog as al


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    sizes = [int(float(a) * 1e6) for a in args] or [16_000_000, 771_000_000]
    stream = torch.cuda.Stream()  # a real stream: the context must launch where the events are recorded
    torch.cuda.set_stream(stream)
    ctx = al.Context(0, stream.cuda_stream)
    lib = ctx.lib
    flush = torch.empty(256 << 20 >> 2, dtype=torch.int32, device="cuda")
    modes = [("classic", {"sort_pipeline": 0, "sort_pipeline_min_keys": 0}), ("pipe8", {"sort_pipeline": 1, "sort_digit_bits": 8}),
             ("pipe9", {"sort_pipeline": 1, "sort_digit_bits": 9}),
             ("pipe10", {"sort_pipeline": 1, "sort_digit_bits": 10}),
             ("pipe8s", {"sort_pipeline": 2, "sort_digit_bits": 8}),
             ("pipe10s", {"sort_pipeline": 2, "sort_digit_bits": 10}),
             ("pipe10m", {"sort_pipeline": 3, "sort_digit_bits": 10}),
             ("classicb", {"sort_pipeline": 4})]
    out = []
    for n in sizes:
        g = torch.Generator(device="cuda").manual_seed(1)
        src = torch.randint(0, 1 << 46, (n,), dtype=torch.int64, device="cuda", generator=g)
        ref = torch.sort(src).values
        a = torch.empty_like(src)
        b = torch.empty_like(src)
        for name, cfg in modes:
            ctx.set_config(**cfg)
            ts = []
            for rep in range(4):
                a.copy_(src)
                flush.add_(1)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                it = C.c_int(0)
                e0.record(stream)
                ctx.check(lib.gd_sort_keys_device(ctx.h, a.data_ptr(), b.data_ptr(), n, 46, C.byref(it)))
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res = b if it.value else a
            ok = bool(torch.equal(res, ref))
            ms = float(np.median(ts[1:]))
            nb = 46
            npass = {"classic": 6, "classicb": 6}.get(name, -(-nb // cfg.get("sort_digit_bits", 8)))
            rec = {"n": n, "mode": name, "ms": round(ms, 3), "ok": ok, "passes": npass,
                   "gbs_per_pass": round(2 * 8 * n * npass / (ms / 1e3) / 1e9 / npass, 1)}
            print(json.dumps(rec), flush=True)
            out.append(rec)
        del src, ref, a, b
        torch.cuda.empty_cache()
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/sort_micro.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
