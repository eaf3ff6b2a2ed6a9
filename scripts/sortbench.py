"""Radix sort microbenchmark: canonicalize-style sort of random packed keys
through the engine's kernels (GD_SORT_ITEMS selects the tile size)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2311_02206_b200 import arraylog as al
ctx = al.default_context()
for n in (1 << 16, 1 << 18, 1 << 20, 1 << 22, 1 << 24):
    a = np.random.default_rng(1).integers(0, 1 << 23, size=(n, 2), dtype=np.uint64)
    t = al.tuple_array(2, a)
    al.canonicalize(t)
    ctx.set_profiling(True); ctx.profile_reset()
    for _ in range(5):
        al.canonicalize(t)
    p = ctx.profile(); ctx.set_profiling(False)
    sp = p["sort_pass"]
    print(f"n={n:9d} sort_pass avg {sp[0]/sp[1]*1e3:8.1f} us  ({sp[2]/sp[1]/(sp[0]/sp[1]/1e3)/1e9:7.1f} GB/s)  hist {p['sort_hist'][0]/5*1e3:6.1f} us/sort", flush=True)
