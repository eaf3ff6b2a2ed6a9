"""Δ-size distribution of C2's iterations (how much of the run is
launch-bound): prints iteration counts and row shares per Δ-size band."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import bench
from paper_2311_02206_b200 import arraylog as al
torch.cuda.set_device(0)
ctx = al.Context(0, torch.cuda.current_stream().cuda_stream)
edges = bench.gen_workload()
e = al.engine("reach", ctx=ctx)
e.load_edb("Edge", al.tuple_array(2, edges))
e.run()
h = np.array(e.delta_history("Reach"), dtype=np.int64)
print("iterations", len(h), "sum", h.sum())
for lo, hi in [(0, 1e3), (1e3, 1e4), (1e4, 1e5), (1e5, 1e6), (1e6, 1e7), (1e7, 1e9)]:
    m = (h >= lo) & (h < hi)
    print(f"delta in [{lo:.0e},{hi:.0e}): iters {m.sum():4d} rows {h[m].sum()/h.sum():.4f}")
print("first 20", h[:20].tolist())
print("every 50th", h[::50].tolist())
