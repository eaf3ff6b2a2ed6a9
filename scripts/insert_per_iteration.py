"""Per-iteration cost of C2's insert and count kernels: the ncu launch list
of one eager C2 run (gpu__time_duration per launch) against that run's
iteration log (scripts/iter_log_dump.py) -> markdown on stdout.
python scripts/insert_per_iteration.py gpurun_out/launches_r4.csv gpurun_out/c2_iter_log.npy"""
import csv
import sys

import numpy as np


def launches(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    r = csv.reader(lines)
    h = next(r)
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    return [(x[ki], float(x[vi].replace(",", "")) * scale[x[ui]]) for x in r]


rows = launches(sys.argv[1])
log = np.load(sys.argv[2])
ins = np.array([v for k, v in rows if "expand_insert" in k])
cnt = np.array([v for k, v in rows if "loop_count" in k])
# launches of iterations rolled back for a growth: the insert stops at once
# (the gate flagged the overflow); they are the extra launches beyond the log
extra = len(ins) - len(log)
J = log[:, 1].astype(float)
drop = sorted(np.argsort(ins)[: max(extra, 0)]) if extra > 0 else []
keep = np.setdiff1d(np.arange(len(ins)), drop)
t, c = ins[keep], cnt[keep]
print("# C2 insert / count cost per iteration (ncu launch list vs iteration log)\n")
print(f"{len(ins)} insert launches, {len(log)} iterations ({extra} rolled-back launches dropped: "
      f"{ins[drop].sum():.0f} us); insert total {t.sum() / 1e3:.1f} ms, count total {c.sum() / 1e3:.1f} ms "
      "(ncu: cold caches, serialised)\n")
print("| join rows J | iterations | share of J | insert ms | count ms | G rows/s | mean insert us |")
print("|---|---|---|---|---|---|---|")
for lo, hi in [(0, 1e3), (1e3, 1e4), (1e4, 1e5), (1e5, 3e5), (3e5, 1e6), (1e6, 3e6), (3e6, 1e9)]:
    m = (J >= lo) & (J < hi)
    if m.sum():
        print(f"| [{lo:.0e}, {hi:.0e}) | {m.sum()} | {J[m].sum() / J.sum():.3f} | {t[m].sum() / 1e3:.2f} | "
              f"{c[m].sum() / 1e3:.2f} | {J[m].sum() / t[m].sum() / 1e3:.2f} | {t[m].mean():.1f} |")
A = np.stack([np.ones_like(J), J], 1)
co = np.linalg.lstsq(A, t, rcond=None)[0]
print(f"\nleast-squares fit: insert = {co[0]:.1f} us + J / {1 / co[1] / 1e3:.2f} G rows/s; "
      f"count mean {c.mean():.1f} us (min {c.min():.1f})")
