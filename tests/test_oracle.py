"""CPU: pins the plain-C oracle (oracle/gdlog_oracle.c) against the
reference's known answers, the committed golden fixtures and the reference
engine itself (oracle/_ref).  No GPU involved."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2311_02206_b200.builtins import BUILTINS, CSPA, REACH, SG, to_blob
from tests.helpers import F, I, K, O, U64MAX, chain_edges, random_relation, rows, spec

GOLD = Path(__file__).resolve().parent / "golden"
KA = json.loads((GOLD / "known_answers.json").read_text())


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint64).tobytes()).hexdigest()


def run_port(port, prog, edbs):
    ids = {prog.rid(k): np.asarray(v, dtype=np.uint64) for k, v in edbs.items()}
    return port.run_engine([a for _, a, _ in prog.relations], [int(e) for _, _, e in prog.relations],
                           to_blob(prog), ids)


def test_known_answers_kernels(port):
    k = KA["canonicalize"]
    assert port.canonicalize(k["in"], 2).reshape(-1).tolist() == k["out"]
    k = KA["permute"]
    assert port.permute_columns(port.canonicalize(k["in"], 2), 2, k["perm"]).reshape(-1).tolist() == k["out"]
    for name in ("group_starts", "range_lookup"):
        k = KA[name]
        a = port.canonicalize(k["in"], 2)
        keys = [[int(x)] for x in k["lookups"]]
        st, ct, _, _ = port.index_lookup(a, 2, 1, keys)
        assert [[int(s), int(c)] for s, c in zip(st, ct)] == list(k["lookups"].values())
    k = KA["join_count"]
    assert port.join(port.canonicalize(k["outer"], 2), 2, port.canonicalize(k["inner"], 2), 2,
                     spec(1, [O(1), I(1)]), materialize=False) == k["count"]
    k = KA["star_self_join"]
    r = port.canonicalize(k["rel"], 2)
    assert len(port.join(r, 2, r, 2, spec(1, [O(1), I(1)]))) == k["count"]
    k = KA["inequality"]
    r = port.canonicalize(k["rel"], 2)
    out = port.join(r, 2, r, 2, spec(1, [O(1), I(1)], [F(O(1), I(1), False)]))
    assert port.canonicalize(out, 2).tolist() == k["out"]
    k = KA["merge"]
    assert port.merge_sorted(k["full"], k["delta"], 2).reshape(-1).tolist() == k["out"]
    k = KA["difference"]
    assert port.difference(k["new"], k["full"], 1).reshape(-1).tolist() == k["out"]


def test_known_answers_engine(port):
    rels, hist, _, iters = run_port(port, REACH, {"Edge": chain_edges(5)})
    k = KA["reach_path5"]
    assert len(rels[1]) == k["count"] and iters == k["iterations"] and hist[1] == k["delta_history"]
    rels, _, _, iters = run_port(port, REACH, {"Edge": rows([1, 1], 2)})
    assert rels[1].tolist() == KA["reach_self_loop"]["out"] and iters == 1
    rels, _, _, _ = run_port(port, SG, {"Edge": rows(KA["sg_binary_tree"]["edges"], 2)})
    assert len(rels[1]) == 14
    k = KA["cspa_seed"]
    rels, _, _, _ = run_port(port, CSPA, {"assign": rows([1, 2], 2)})
    for name in ("ValueFlow", "MemoryAlias", "ValueAlias"):
        assert rels[CSPA.rid(name)].tolist() == k[name]


def test_c1_golden(port):
    g = np.load(GOLD / "c1_tc_rand.npz")
    rels, hist, log, iters = run_port(port, REACH, {"Edge": g["edges"]})
    assert np.array_equal(rels[1], g["reach"])
    assert hist[1] == g["delta_history"].tolist()
    assert iters == int(g["iterations"]) == KA["c1"]["iterations"]
    assert len(rels[1]) == KA["c1"]["reach"]
    assert [list(x) for x in log[1][:3]] == KA["c1"]["first_iterations"]


@pytest.mark.parametrize("kind", ["reach", "sg", "cspa"])
def test_corpora_golden(port, kind):
    corp = json.loads((GOLD / "corpora.json").read_text())[kind]
    prog = BUILTINS[kind]
    for rec in corp[:: 3 if kind == "reach" else 2]:
        if kind == "cspa":
            edbs = {"assign": rows(np.asarray(rec["assign"]).reshape(-1), 2),
                    "dereference": rows(np.asarray(rec["dereference"]).reshape(-1), 2)}
            names = ("ValueFlow", "ValueAlias", "MemoryAlias")
        else:
            edbs = {"Edge": rows(np.asarray(rec["edges"]).reshape(-1), 2)}
            names = ("Reach",) if kind == "reach" else ("SG",)
        rels, _, _, iters = run_port(port, prog, edbs)
        assert iters == rec["iterations"]
        for n in names:
            assert [len(rels[prog.rid(n)]), sha(rels[prog.rid(n)])] == rec[n], n


@pytest.mark.parametrize("seed", range(6))
def test_port_matches_reference_kernels(port, ref, seed):
    rng = np.random.default_rng(seed)
    a = random_relation(rng, 2, 3000, 60 + seed * 40, U64MAX - 5000 if seed == 5 else 0)
    ca = port.canonicalize(a, 2)
    assert np.array_equal(ca, ref.canonicalize(a, 2))
    assert np.array_equal(port.permute_columns(ca, 2, [1, 0]), ref.permute_columns(ca, 2, [1, 0]))
    assert np.array_equal(port.prefix_hash(a, 2, 1), ref.prefix_hash(a, 2, 1))
    assert np.array_equal(port.prefix_hash(a, 2, 2), ref.prefix_hash(a, 2, 2))
    keys = np.vstack([ca[:, :1], random_relation(rng, 1, 200, 100)])
    pst, pct, psc, poc = port.index_lookup(ca, 2, 1, keys)
    rst, rct, rsc, roc = ref.index_lookup(ca, 2, 1, keys)
    assert np.array_equal(pct, rct) and np.array_equal(pst, rst) and (psc, poc) == (rsc, roc)
    b = port.canonicalize(random_relation(rng, 2, 2000, 60 + seed * 40), 2)
    for s in (spec(1, [O(1), I(1)]), spec(1, [I(1), O(0), K(9)], [F(O(1), I(1), False)]), spec(0, [O(0), I(0)])):
        jb = b[:40] if s.join_column_count == 0 else b
        assert np.array_equal(port.join(ca, 2, jb, 2, s), ref.join(ca, 2, jb, 2, s))
    f = port.difference(b, ca, 2)
    assert np.array_equal(f, ref.difference(b, ca, 2))
    assert np.array_equal(port.merge_sorted(ca, f, 2), ref.merge_sorted(ca, f, 2))


@pytest.mark.parametrize("kind,seed", [("reach", 1), ("reach", 2), ("sg", 3), ("cspa", 4), ("cspa", 5)])
def test_port_engine_matches_reference(port, ref, kind, seed):
    rng = np.random.default_rng(seed)
    prog = BUILTINS[kind]
    if kind == "cspa":
        edbs = {"assign": random_relation(rng, 2, 120, 40), "dereference": random_relation(rng, 2, 150, 40)}
    else:
        edbs = {"Edge": random_relation(rng, 2, 400, 150)}
    rels, hist, _, iters = run_port(port, prog, edbs)
    r = ref.engine(kind)
    for k, v in edbs.items():
        r.load_edb(k, v)
    r.run()
    assert iters == r.stats().iterations
    for n in prog.idbs:
        assert np.array_equal(rels[prog.rid(n)], r.relation(n)), n
        if any(p.head == n and p.recursive for p in prog.rules):
            assert hist[prog.rid(n)] == r.delta_history(n)


def test_host_digest_twin_matches_reference_hash(ref):
    """tests/helpers.prefix_hash_np (the host twin behind digest_rows, which
    pins the device relation digest) equals the reference's slot_key on
    random rows, arities 1-5."""
    from tests.helpers import prefix_hash_np
    rng = np.random.default_rng(5)
    for arity in range(1, 6):
        rows = rng.integers(0, 1 << 63, size=(500, arity), dtype=np.uint64) * np.uint64(2)
        got = prefix_hash_np(rows)
        exp = ref.prefix_hash(rows, arity, arity)
        # slot_key remaps the sentinel to sentinel - 1 (hash.hpp:57-60)
        got = np.where(got == np.uint64((1 << 64) - 1), np.uint64((1 << 64) - 2), got)
        assert np.array_equal(got, exp), arity
