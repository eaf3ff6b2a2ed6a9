"""Calibrates synthetic workload parameters on the GPU (SURVEY §8d asks
C2 to land at |Reach| in [0.5, 2]e9).  Usage: python scripts/calibrate.py tc_pl"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_2311_02206_b200 import arraylog as al  # noqa: E402
from paper_2311_02206_b200 import workloads as W  # noqa: E402


def run(prog, edbs):
    e = al.engine(prog)
    for k, v in edbs.items():
        e.load_edb(k, al.tuple_array(2, v))
    t = time.time()
    e.run()
    al.default_context().synchronize()
    dt = time.time() - t
    s = e.raw_stats()
    out = {n: e.relation_count(n) for n in e.idb_relations()}
    e.close()
    return dt, s.iterations, s.join_tuples, out, s.device_bytes_peak


kind = sys.argv[1]
if kind == "tc_pl":
    grid = [tuple(map(float, x.split(","))) for x in sys.argv[2:]] or [
        (5e6, 200, 1.0), (5e6, 32, 1.5), (5e6, 64, 1.5), (2e7, 200, 2.0), (2e7, 64, 3.0), (5e6, 16, 2.0)]
    for n, w, a in grid:
        n, w = int(n), int(w)
        e = W.tc_pl(n, 5_000_000, w, a, 1)
        try:
            dt, it, j, out, peak = run("reach", {"Edge": e})
            print(f"tc_pl n={n} W={w} a={a} edges={len(e)} -> {out} iters={it} J={j} t={dt:.3f}s "
                  f"peak={peak/1e9:.1f}GB", flush=True)
        except Exception as ex:  # noqa: BLE001
            print(f"tc_pl n={n} W={w} a={a}: {type(ex).__name__}: {str(ex)[:120]}", flush=True)
elif kind == "sg_tree":
    for n, w in [(1_000_001, int(x)) for x in sys.argv[2:]] or [(1_000_001, 1000), (1_000_001, 3000)]:
        e = W.sg_tree(n, w, 1)
        dt, it, j, out, peak = run("sg", {"Edge": e})
        print(f"sg_tree n={n} W={w} -> {out} iters={it} J={j} t={dt:.3f}s peak={peak/1e9:.1f}GB", flush=True)
elif kind == "cspa":
    for n in [int(float(x)) for x in sys.argv[2:]] or [3_000_000, 2_500_000, 2_000_000]:
        a, d = W.cspa_local(n, 362_000, 1_140_000, 256, 1)
        try:
            dt, it, j, out, peak = run("cspa", {"assign": a, "dereference": d})
            print(f"cspa n={n} -> {out} iters={it} J={j} t={dt:.3f}s peak={peak/1e9:.1f}GB", flush=True)
        except Exception as ex:  # noqa: BLE001
            print(f"cspa n={n}: {type(ex).__name__}: {str(ex)[:120]}", flush=True)
