"""Distribution of C2's Reach keys over top-bit buckets (sizing an MSD
final sort).  Prints, per bucket width, max bucket size and the share of
keys in buckets above smem-sortable sizes."""
import sys, numpy as np
sys.path.insert(0, ".")
import bench
from paper_2311_02206_b200 import arraylog as al
import torch
torch.cuda.set_device(0)
ctx = al.Context(0, torch.cuda.current_stream().cuda_stream)
edges = bench.gen_workload()
e = al.engine("reach", ctx=ctx)
e.load_edb("Edge", al.tuple_array(2, edges))
e.run()
print("encoding", e.encoding())
r = e.relation("Reach")
rows = r.data
src = rows[:, 0].astype(np.int64); dst = rows[:, 1].astype(np.int64)
bits = int(e.encoding()["bits"])
key = (src << bits) | dst
tb = 2 * bits
print("n", len(key), "key bits", tb)
for k in range(10, 22):
    h = np.bincount(key >> (tb - k), minlength=1 << k)
    for cap in (6144, 12288, 24576):
        big = h[h > cap]
        print(f"top{k:2d} cap{cap:6d}: max {h.max():9d} buckets>cap {len(big):6d} keys_in_big {big.sum()/len(key):.4f}")
deg = np.bincount(src)
print("max reach per src", deg.max(), "srcs>12288", (deg > 12288).sum(), "share", deg[deg > 12288].sum() / len(key))
