"""Synthetic workloads of SURVEY §8(d) (the configs of BASELINE.json).

Vectorised numpy generators (seeded, deterministic).  These define the
benchmark inputs; they are not bit-identical to the survey's libstdc++
mt19937 probes (tests reproduce C1 exactly through the compiled reference
generator), but follow the same shapes.  Duplicate draws are kept: they
collapse when the engine canonicalizes at load (engine.hpp:107-128).

  tc_rand   C1  uniform random graph, n nodes, m draws
  tc_pl     C2  power-law DAG: src = floor((n-1) U^alpha), dst = src+1+U{0..W-1}
  sg_tree   C3  random tree/DAG: node v in [1, n) gets parent U{max(0,v-W)..v-1}
  cspa_local C4 assign/dereference inside modules of S variables
  tc_dag    C5  alpha = 1 variant of tc_pl at 10^8 edges
"""
from __future__ import annotations

import numpy as np


def tc_rand(n: int, m: int, seed: int = 1) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.integers(0, n, size=(m, 2), dtype=np.uint64)


def tc_pl(n: int, m: int, window: int, alpha: float, seed: int = 1) -> np.ndarray:
    rng = np.random.default_rng(seed)
    u = rng.random(m)
    src = np.floor((n - 1) * u ** alpha).astype(np.uint64)
    dst = src + np.uint64(1) + rng.integers(0, window, size=m, dtype=np.uint64)
    dst = np.minimum(dst, np.uint64(n - 1))
    keep = src < dst
    return np.ascontiguousarray(np.column_stack([src[keep], dst[keep]]))


def tc_dag(n: int, m: int, window: int = 200, seed: int = 1) -> np.ndarray:
    return tc_pl(n, m, window, 1.0, seed)


def sg_tree(n: int, window: int, seed: int = 1) -> np.ndarray:
    rng = np.random.default_rng(seed)
    v = np.arange(1, n, dtype=np.int64)
    lo = np.maximum(0, v - window)
    parent = lo + (rng.random(n - 1) * (v - lo)).astype(np.int64)
    return np.ascontiguousarray(np.column_stack([parent, v]).astype(np.uint64))


def cspa_local(n: int, n_assign: int, n_deref: int, module: int = 256, seed: int = 1):
    rng = np.random.default_rng(seed)
    nmod = max(1, n // module)

    def draw(k):
        mod = rng.integers(0, nmod, size=k, dtype=np.uint64) * np.uint64(module)
        a = mod + rng.integers(0, module, size=k, dtype=np.uint64)
        b = mod + rng.integers(0, module, size=k, dtype=np.uint64)
        return np.ascontiguousarray(np.column_stack([a, b]))

    return draw(n_assign), draw(n_deref)


# Named configurations (BASELINE.json "configs").
CONFIGS = {
    "c1_tc_rand": dict(program="reach", gen=lambda: {"Edge": tc_rand(10_000, 10_000, 1)},
                       desc="TC on a random graph, n=m=1e4"),
    "c2_tc_pl": dict(program="reach", gen=lambda: {"Edge": tc_pl(5_000_000, 5_000_000, 200, 1.05, 1)},
                     desc="TC on a power-law DAG, 5e6 edge draws (n=5e6, W=200, alpha=1.05; bench.py)"),
    "c3_sg_tree": dict(program="sg", gen=lambda: {"Edge": sg_tree(1_000_001, 40, 1)},
                       desc="SG on a random tree, 1e6 edges (W=40)"),
    "c3_sg_tree_w1000": dict(program="sg", gen=lambda: {"Edge": sg_tree(1_000_001, 1000, 1)},
                             desc="SG on a random tree, 1e6 edges (W=1000)"),
    "c3_sg_tree_w4000": dict(program="sg", gen=lambda: {"Edge": sg_tree(1_000_001, 4000, 1)},
                             desc="SG on a random tree, 1e6 edges (W=4000)"),
    "c4_cspa": dict(program="cspa", gen=lambda: dict(zip(("assign", "dereference"),
                                                        cspa_local(1_500_000, 362_000, 1_140_000, 256, 1))),
                    desc="CSPA, httpd-sized EDB (assign 3.62e5, dereference 1.14e6, modules of 256)"),
    "c5_tc_dag": dict(program="reach", gen=lambda: {"Edge": tc_dag(100_000_000, 100_000_000, 200, 1)},
                      desc="TC on a 1e8-edge DAG (W=200, alpha=1)"),
}
