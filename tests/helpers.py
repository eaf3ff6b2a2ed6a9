"""Test helpers: seeded inputs (numpy), plan conversion, comparisons."""
from __future__ import annotations

import ctypes as C

import numpy as np

from paper_2311_02206_b200 import abi as A
from paper_2311_02206_b200.builtins import Program, Rule, Step, Variant

U64MAX = (1 << 64) - 1


def rows(flat, arity):
    return np.asarray(flat, dtype=np.uint64).reshape(-1, arity)


def random_relation(rng: np.random.Generator, arity: int, n: int, domain: int, high: int = 0) -> np.ndarray:
    """Random rows with values in [high, high + domain)."""
    return (rng.integers(0, domain, size=(n, arity), dtype=np.uint64) + np.uint64(high)).astype(np.uint64)


def set_rows(a: np.ndarray) -> np.ndarray:
    """Canonical (sorted, unique) rows of a — numpy lexicographic order."""
    if len(a) == 0:
        return a.reshape(0, a.shape[1] if a.ndim == 2 else 1)
    return np.unique(a, axis=0)


def chain_edges(nodes: int) -> np.ndarray:
    """engine_test.cpp:21-28 — 1->2->...->nodes."""
    return rows([v for i in range(1, nodes) for v in (i, i + 1)], 2)


def operand_str(op) -> str:
    return {0: "o", 1: "i", 2: "c"}[op.kind] + (str(op.column) if op.kind < 2 else str(op.value))


def program_from_ref(ref_engine) -> Program:
    """Builds a Program (relations + plans) from the reference planner's
    output for programs outside the built-ins (test-only: the planner is
    not part of the hot path)."""
    names, ar = ref_engine.names, ref_engine.arities
    # EDBs are the relations no plan has as head
    heads = set()
    plans = ref_engine.plans()
    for p in plans:
        heads.add(names[p.head_rel])
    rels = [(n, a, n not in heads) for n, a in zip(names, ar)]
    rules = []
    for p in plans:
        variants = []
        for v in p.variants[: p.nvariants]:
            sa = ar[v.src_rel]
            steps = []
            for s in v.steps[: v.nsteps]:
                ia = ar[s.inner_rel]
                steps.append(Step(names[s.inner_rel], list(s.inner_perm[:ia]), s.join_column_count,
                                  [operand_str(o) for o in s.proj[: s.proj_arity]],
                                  [(operand_str(f.lhs), operand_str(f.rhs), bool(f.require_equal))
                                   for f in s.filters[: s.nfilters]]))
            variants.append(Variant(names[v.src_rel], "delta" if v.src_version else "full", list(v.src_perm[:sa]),
                                    steps, [operand_str(o) for o in v.sel_proj[: v.sel_arity]],
                                    [(operand_str(f.lhs), operand_str(f.rhs), bool(f.require_equal))
                                     for f in v.sel_filters[: v.nsel_filters]]))
        rules.append(Rule(p.rule_index, names[p.head_rel], bool(p.recursive), variants))
    return Program("custom", rels, rules)


def spec(jcc, proj, filters=()):
    g = A.gd_join_spec()
    g.join_column_count = jcc
    g.proj_arity = len(proj)
    for i, o in enumerate(proj):
        g.proj[i] = o
    g.nfilters = len(filters)
    for i, f in enumerate(filters):
        g.filters[i] = f
    return g


def O(c):
    return A.gd_operand(A.GD_OUTER_COL, c, 0)


def I(c):
    return A.gd_operand(A.GD_INNER_COL, c, 0)


def K(v):
    return A.gd_operand(A.GD_CONSTANT, 0, v)


def F(lhs, rhs, eq=False):
    return A.gd_filter(lhs, rhs, int(eq), 0)


_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _rotl(x, r):
    return (x << np.uint64(r)) | (x >> np.uint64(64 - r))


def fmix64(k: np.ndarray) -> np.ndarray:
    """Murmur3 finalizer (hash.hpp:13-20), vectorised, wrapping u64."""
    k = k ^ (k >> np.uint64(33))
    k = k * np.uint64(0xFF51AFD7ED558CCD)
    k = k ^ (k >> np.uint64(33))
    k = k * np.uint64(0xC4CEB9FE1A85EC53)
    return k ^ (k >> np.uint64(33))


def prefix_hash_np(a: np.ndarray) -> np.ndarray:
    """prefix_hash over every column of each row (hash.hpp:28-53: the
    Murmur3-x64-128-style mix, seed 0, h1 + h2), vectorised."""
    a = np.asarray(a, dtype=np.uint64)
    n = a.shape[1]
    c1, c2 = np.uint64(0x87C37B91114253D5), np.uint64(0x4CF5AD432745937F)
    h1 = np.zeros(len(a), dtype=np.uint64)
    h2 = np.zeros(len(a), dtype=np.uint64)
    with np.errstate(over="ignore"):
        for i in range(0, n - 1, 2):
            k1 = _rotl(a[:, i] * c1, 31) * c2
            h1 ^= k1
            h1 = _rotl(h1, 27) + h2
            h1 = h1 * np.uint64(5) + np.uint64(0x52DCE729)
            k2 = _rotl(a[:, i + 1] * c2, 33) * c1
            h2 ^= k2
            h2 = _rotl(h2, 31) + h1
            h2 = h2 * np.uint64(5) + np.uint64(0x38495AB5)
        if n % 2:
            h1 ^= _rotl(a[:, n - 1] * c1, 31) * c2
        ln = np.uint64(n * 8)
        h1 ^= ln
        h2 ^= ln
        h1 = h1 + h2
        h2 = h2 + h1
        return fmix64(h1) + fmix64(h2)


def digest_rows(a: np.ndarray) -> int:
    """Host twin of the device relation digest (gd_engine_relation_digest,
    primitives.cu digest_kernel): the order-independent sum, mod 2^64, of
    fmix64(prefix_hash(row)) over the rows."""
    a = np.asarray(a, dtype=np.uint64)
    if len(a) == 0:
        return 0
    with np.errstate(over="ignore"):
        return int(np.sum(fmix64(prefix_hash_np(a)), dtype=np.uint64))
