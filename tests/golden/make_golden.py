"""Generates the committed golden fixtures of tests/golden/ from the
reference engine compiled in oracle/_ref (the unmodified arraylog headers).

Run here (where oracle/_ref was built from /root/reference):
    python tests/golden/make_golden.py
Outputs:
  c1_tc_rand.npz       SURVEY §8d C1 input (mt19937_64 seed 1, n = m = 1e4)
                       and the reference's canonical Reach + per-iteration Δ
  corpora.json         acceptance corpora (acceptance_test.cpp:58-89) inputs
                       and sha256 of the reference's canonical outputs
  known_answers.json   known-answer vectors of the reference gtest suites,
                       each with its file:line, re-verified against _ref
"""
import ctypes as C
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle.bindings import RefOracle  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint64).tobytes()).hexdigest()


def corpus(ref, kind, idx):
    out = np.zeros((400, 2), dtype=np.uint64)
    counts = np.zeros(2, dtype=np.uint64)
    rc = ref.lib.ref_acceptance_corpus(C.c_int(kind), C.c_uint32(idx), out.ctypes.data_as(C.c_void_p),
                                       C.c_uint64(400), counts.ctypes.data_as(C.c_void_p))
    assert rc == 0
    a = int(counts[0])
    return out[:a], out[a: a + int(counts[1])]


def main():
    ref = RefOracle()
    # ---- C1 ---------------------------------------------------------------
    raw = np.zeros((10000, 2), dtype=np.uint64)
    assert ref.lib.ref_gen_tc_rand(C.c_uint64(10000), C.c_uint64(10000), C.c_uint64(1),
                                   raw.ctypes.data_as(C.c_void_p)) == 0
    e = ref.engine("reach")
    e.load_edb("Edge", raw)
    e.run()
    reach = e.relation("Reach")
    np.savez_compressed(HERE / "c1_tc_rand.npz", edges=raw, reach=reach,
                        delta_history=np.asarray(e.delta_history("Reach"), dtype=np.uint64),
                        iterations=np.uint64(e.stats().iterations))
    # ---- corpora ----------------------------------------------------------
    out = {"reach": [], "sg": [], "cspa": []}
    for idx in range(200):
        g, _ = corpus(ref, 0, idx)
        r = ref.engine("reach")
        r.load_edb("Edge", g)
        r.run()
        rr = r.relation("Reach")
        out["reach"].append({"edges": g.tolist(), "Reach": [len(rr), sha(rr)],
                             "iterations": r.stats().iterations})
    for idx in range(100):
        g, _ = corpus(ref, 1, idx)
        r = ref.engine("sg")
        r.load_edb("Edge", g)
        r.run()
        rr = r.relation("SG")
        out["sg"].append({"edges": g.tolist(), "SG": [len(rr), sha(rr)], "iterations": r.stats().iterations})
    for idx in range(50):
        a, d = corpus(ref, 2, idx)
        r = ref.engine("cspa")
        r.load_edb("assign", a)
        r.load_edb("dereference", d)
        r.run()
        rec = {"assign": a.tolist(), "dereference": d.tolist(), "iterations": r.stats().iterations}
        for rel in ("ValueFlow", "ValueAlias", "MemoryAlias"):
            rr = r.relation(rel)
            rec[rel] = [len(rr), sha(rr)]
        out["cspa"].append(rec)
    (HERE / "corpora.json").write_text(json.dumps(out))
    # ---- known answers (reference gtest suites) ---------------------------
    ka = {
        "canonicalize": {"src": "tests/tuple_array_test.cpp:12-17", "arity": 2, "in": [2, 1, 1, 2, 2, 1],
                         "out": [1, 2, 2, 1]},
        "permute": {"src": "tests/tuple_array_test.cpp:60-65", "arity": 2, "in": [1, 2, 3, 1], "perm": [1, 0],
                    "out": [1, 3, 2, 1]},
        "group_starts": {"src": "tests/hash_index_test.cpp:59-67", "arity": 2,
                         "in": [35, 100, 11, 101, 46, 102, 97, 103],
                         "lookups": {"11": [0, 1], "35": [1, 1], "46": [2, 1], "97": [3, 1]}},
        "range_lookup": {"src": "tests/hash_index_test.cpp:75-79", "arity": 2, "in": [1, 2, 1, 5, 4, 9],
                         "lookups": {"1": [0, 2], "4": [2, 1]}},
        "join_count": {"src": "tests/ra_test.cpp:38-43", "outer": [1, 3], "inner": [1, 2, 1, 5, 4, 9], "count": 2},
        "star_self_join": {"src": "tests/ra_test.cpp:87-95", "rel": [0, 1, 0, 2, 0, 3], "count": 9},
        "inequality": {"src": "tests/ra_test.cpp:106-116", "rel": [0, 1, 0, 2], "out": [[1, 2], [2, 1]]},
        "merge": {"src": "tests/ra_test.cpp:190-197", "full": [1, 2, 3, 3], "delta": [2, 2, 3, 4], "arity": 2,
                  "out": [1, 2, 2, 2, 3, 3, 3, 4]},
        "difference": {"src": "tests/ra_test.cpp:240-244", "new": [1, 2, 3], "full": [1, 4], "arity": 1,
                       "out": [2, 3]},
        "reach_path5": {"src": "tests/engine_test.cpp:42-52", "count": 10, "iterations": 4,
                        "delta_history": [4, 3, 2, 1]},
        "reach_self_loop": {"src": "tests/engine_test.cpp:54-59", "out": [[1, 1]], "iterations": 1},
        "sg_binary_tree": {"src": "tests/engine_test.cpp:71-81", "edges": [1, 2, 1, 3, 2, 4, 2, 5, 3, 6, 3, 7],
                           "count": 14},
        "cspa_seed": {"src": "tests/engine_test.cpp:83-93", "assign": [[1, 2]],
                      "ValueFlow": [[1, 1], [1, 2], [2, 2]], "MemoryAlias": [[1, 1], [2, 2]],
                      "ValueAlias": [[1, 1], [1, 2], [2, 1], [2, 2]]},
        "buffer_manager": {"src": "tests/budget_test.cpp:53-93", "first_capacity": 150, "reuse_capacity": 150,
                           "shrunk_capacity": 120},
        "c1": {"src": "SURVEY.md §8d (probe of the reference engine)", "edges": 9999, "reach": 198733,
               "iterations": 46, "first_iterations": [[9999, 10018, 10017, 10008, 20007],
                                                      [10008, 9999, 9998, 9996, 30003],
                                                      [9996, 10013, 10012, 10004, 40007]]},
    }
    # re-verify the engine-level answers against the compiled reference
    chain5 = np.array([[i, i + 1] for i in range(1, 5)], dtype=np.uint64)
    r = ref.engine("reach")
    r.load_edb("Edge", chain5)
    r.run()
    assert len(r.relation("Reach")) == 10 and r.delta_history("Reach") == [4, 3, 2, 1]
    r = ref.engine("sg")
    r.load_edb("Edge", np.array(ka["sg_binary_tree"]["edges"], dtype=np.uint64).reshape(-1, 2))
    r.run()
    assert len(r.relation("SG")) == 14
    assert len(reach) == 198733 and e.stats().iterations == 46
    (HERE / "known_answers.json").write_text(json.dumps(ka, indent=1))
    print("golden fixtures written")


if __name__ == "__main__":
    main()
