"""GPU parity of the device fixpoint engine against the reference engine
(oracle/_ref): output relations byte-identical, Δ history and iteration
count identical, and the host bookkeeping (charge events, peaks, EBM
allocations, budget errors) identical — engine_test.cpp and
acceptance_test.cpp restated.
"""
import numpy as np
import pytest

from paper_2311_02206_b200 import abi as A
from paper_2311_02206_b200 import arraylog as al
from tests.helpers import U64MAX, chain_edges, program_from_ref, random_relation, rows

pytestmark = pytest.mark.gpu


def run_gpu(program, edbs, cfg=None):
    e = al.engine(program, cfg)
    for name, r in edbs.items():
        r = np.asarray(r, dtype=np.uint64)
        e.load_edb(name, al.tuple_array(r.shape[1] if r.ndim == 2 else 2, r))
    e.run()
    return e


def run_ref(ref, program_src, edbs, cfg=None):
    e = ref.engine(program_src, cfg.to_c() if cfg else None)
    for name, r in edbs.items():
        e.load_edb(name, np.asarray(r, dtype=np.uint64))
    e.run()
    return e


def assert_same(g, r, names, stats=True):
    for n in names:
        assert np.array_equal(g.relation(n).data, r.relation(n)), n
    gs, rs = g.raw_stats(), r.stats()
    assert gs.iterations == rs.iterations
    for n in names:
        if n in [h for h, _ in g.stats().delta_history]:
            assert g.delta_history(n) == r.delta_history(n), n
    if stats:
        assert gs.charge_events == rs.charge_events
        assert gs.peak_tracked_bytes == rs.peak_tracked_bytes
        assert gs.peak_temp_bytes == rs.peak_temp_bytes
        assert gs.buffer_allocations == rs.buffer_allocations


# ---- known answers (engine_test.cpp) ---------------------------------------

def test_reach_five_node_path(ref):
    g = run_gpu("reach", {"Edge": chain_edges(5)})
    assert g.relation("Reach").count() == 10
    s = g.stats()
    assert s.iterations == 4
    assert s.delta_history == [("Reach", [4, 3, 2, 1])]
    assert_same(g, run_ref(ref, "reach", {"Edge": chain_edges(5)}), ["Reach"])


def test_reach_self_loop():
    g = run_gpu("reach", {"Edge": rows([1, 1], 2)})
    assert g.relation("Reach").rows() == [(1, 1)]
    assert g.stats().iterations == 1


def test_sg_binary_tree(ref):
    edges = rows([1, 2, 1, 3, 2, 4, 2, 5, 3, 6, 3, 7], 2)
    g = run_gpu("sg", {"Edge": edges})
    assert g.relation("SG").count() == 14
    assert_same(g, run_ref(ref, "sg", {"Edge": edges}), ["SG"])
    assert g.stats().peak_temp_bytes > 0


def test_cspa_seed_copy_rules():
    g = run_gpu("cspa", {"assign": rows([1, 2], 2)})
    assert g.relation("ValueFlow").rows() == [(1, 1), (1, 2), (2, 2)]
    assert g.relation("MemoryAlias").rows() == [(1, 1), (2, 2)]
    assert g.relation("ValueAlias").rows() == [(1, 1), (1, 2), (2, 1), (2, 2)]


def test_empty_edb_gives_empty_idb():
    e = al.engine("cspa")
    e.run()
    for n in e.idb_relations():
        assert e.relation(n).count() == 0
    assert e.stats().iterations == 0


def test_cspa_toy(ref):
    db = {"assign": rows([1, 2, 2, 3, 4, 1], 2), "dereference": rows([1, 5, 3, 6, 2, 5], 2)}
    assert_same(run_gpu("cspa", db), run_ref(ref, "cspa", db), ["ValueFlow", "ValueAlias", "MemoryAlias"])


def test_delta_rows_counted_once():
    g = run_gpu("reach", {"Edge": chain_edges(12)})
    assert sum(g.delta_history("Reach")) == g.relation("Reach").count()


def test_ebm_saves_allocations(ref):
    on = run_gpu("reach", {"Edge": chain_edges(60)}, al.engine_config(ebm_enabled=True))
    off = run_gpu("reach", {"Edge": chain_edges(60)}, al.engine_config(ebm_enabled=False))
    assert np.array_equal(on.relation("Reach").data, off.relation("Reach").data)
    assert on.stats().buffer_allocations < off.stats().buffer_allocations
    cfg = al.engine_config(ebm_enabled=False)
    assert_same(off, run_ref(ref, "reach", {"Edge": chain_edges(60)}, cfg), ["Reach"])


LOOPS = {"resident": {}, "host": {"resident_loop": 0}}


@pytest.mark.parametrize("loop", list(LOOPS))
def test_budget_error_names_a_phase(ref, loop):
    """Finite budgets run on both loops: the resident device loop replays
    the reference's charges after the fixpoint and raises the same error."""
    cfg = al.engine_config(memory_budget_bytes=400)
    with pytest.raises(al.budget_error) as ei, al.default_context().configured(**LOOPS[loop]):
        run_gpu("reach", {"Edge": chain_edges(30)}, cfg)
    from oracle.bindings import OracleError
    with pytest.raises(OracleError) as er:
        run_ref(ref, "reach", {"Edge": chain_edges(30)}, cfg)
    assert ei.value.phase() == er.value.phase
    assert ei.value.phase() in A.PHASES


@pytest.mark.parametrize("loop", list(LOOPS))
@pytest.mark.parametrize("budget", [2000, 6000, 20000, 60000])
def test_budget_errors_match_reference_phase(ref, budget, loop):
    cfg = al.engine_config(memory_budget_bytes=budget)
    from oracle.bindings import OracleError
    edges = chain_edges(40)
    try:
        run_ref(ref, "reach", {"Edge": edges}, cfg)
        ref_phase = None
    except OracleError as e:
        ref_phase = e.phase
    try:
        with al.default_context().configured(**LOOPS[loop]):
            run_gpu("reach", {"Edge": edges}, cfg)
        gpu_phase = None
    except al.budget_error as e:
        gpu_phase = e.phase()
    assert gpu_phase == ref_phase


@pytest.mark.parametrize("loop", list(LOOPS))
@pytest.mark.parametrize("prog,budget", [("reach", 3 << 20), ("sg", 1 << 20), ("reach", 200_000)])
def test_finite_budget_runs_match_reference(ref, prog, budget, loop):
    """A finite budget that the run fits (EBM shrinks K to fit it): result,
    Δ history, iterations, peaks and buffer allocations equal the
    reference's on both loops (the resident loop under a budget)."""
    from oracle.bindings import OracleError
    rng = np.random.default_rng(budget)
    edges = random_relation(rng, 2, 3000, 1200) if prog == "reach" else random_relation(rng, 2, 900, 700)
    cfg = al.engine_config(memory_budget_bytes=budget)
    try:
        r = run_ref(ref, prog, {"Edge": edges}, cfg)
    except OracleError as e:
        with pytest.raises(al.budget_error) as ei, al.default_context().configured(**LOOPS[loop]):
            run_gpu(prog, {"Edge": edges}, cfg)
        assert ei.value.phase() == e.phase
        return
    with al.default_context().configured(**LOOPS[loop]):
        g = run_gpu(prog, {"Edge": edges}, cfg)
    assert_same(g, r, [{"reach": "Reach", "sg": "SG"}[prog]])


def test_load_errors_and_config_validation():
    e = al.engine("reach")
    with pytest.raises(al.load_error):
        e.load_edb("Nope", al.tuple_array(2, [1, 2]))
    with pytest.raises(al.load_error):
        e.load_edb("Edge", al.tuple_array(1, [1]))
    with pytest.raises(al.load_error):
        e.load_edb("Edge", al.tuple_array(2, [1, U64MAX]))
    with pytest.raises(al.usage_error):
        e.relation("Nope")
    with pytest.raises(al.config_error):
        al.engine("reach", al.engine_config(alpha=0))
    with pytest.raises(al.config_error):
        al.engine("reach", al.engine_config(load_factor=1.0))


def test_stats_tsv_shape():
    g = run_gpu("reach", {"Edge": chain_edges(5)})
    tsv = al.to_tsv(g.stats())
    assert tsv.startswith("phase\tseconds\nindex\t")
    assert "relation\tReach\niteration\tdelta_rows\n1\t4\n" in tsv


CUSTOM = {
    "dropping": (".decl EA(2)\n.decl EB(2)\nA(x, y) :- EA(x, y).\nA(x, y) :- A(x, z), EA(z, y).\n"
                 "B(x, y) :- EB(x, y).\nB(x, y) :- B(x, z), EB(z, y).\nP(x, y) :- A(x, z), B(z, y).\n",
                 {"EA": rows([1, 2, 2, 3], 2), "EB": rows([3, 10, 10, 11, 11, 12, 12, 13], 2)}),
    "constants": (".decl E(2)\n.decl A(1)\n.decl B(1)\nMarker(1) :- E(x, y).\nSelfish(x) :- E(x, x).\n"
                  "Pairs(x, y) :- A(x), B(y).\nLoopy(x, y) :- E(x, y), x != y.\n"
                  "Loopy(x, y) :- Loopy(x, z), E(z, y), x != y.\n",
                  {"E": rows([1, 1, 1, 2, 2, 3, 3, 1], 2), "A": rows([5, 6], 1), "B": rows([7], 1)}),
    "stratified": (".decl E(2)\nC(x, y) :- E(x, y).\nC(x, y) :- C(x, z), E(z, y).\nH(y, x) :- C(x, y).\n",
                   {"E": rows([1, 2, 2, 3, 3, 4], 2)}),
    "ternary": (".decl E(3)\nT(x, y, z) :- E(x, y, z).\nT(x, y, w) :- T(x, y, z), E(z, w, v).\n"
                "U(a, b) :- T(a, b, c), T(c, b, a).\n",
                {"E": rows([1, 2, 3, 3, 4, 5, 5, 6, 1, 2, 2, 2, 6, 1, 1], 3)}),
}


@pytest.mark.parametrize("case", sorted(CUSTOM))
def test_custom_programs_match_reference(ref, case):
    src, db = CUSTOM[case]
    r = run_ref(ref, src, db)
    prog = program_from_ref(r)
    g = run_gpu(prog, db)
    assert_same(g, r, prog.idbs)


def test_override_plans_drop_variant(ref):
    src, db = CUSTOM["dropping"]
    r = run_ref(ref, src, db)
    prog = program_from_ref(r)
    full = run_gpu(prog, db).relation("P").rows()
    from paper_2311_02206_b200.builtins import to_blob
    for drop in (0, 1):
        plans = to_blob(prog)
        for p in plans:
            if prog.relations[p.head_rel][0] == "P":
                assert p.nvariants == 2
                if drop == 0:
                    p.variants[0] = p.variants[1]
                p.nvariants = 1
        e = al.engine(prog)
        e.override_plans(plans)
        for n, rr in db.items():
            e.load_edb(n, al.tuple_array(2, rr))
        e.run()
        got = e.relation("P").rows()
        assert set(got) < set(full)


# ---- seeded corpora (acceptance_test.cpp criteria 1-3) ----------------------

def corpus(ref, kind, idx):
    import ctypes as C
    out = np.zeros((400, 2), dtype=np.uint64)
    counts = np.zeros(2, dtype=np.uint64)
    rc = ref.lib.ref_acceptance_corpus(C.c_int(kind), C.c_uint32(idx), out.ctypes.data_as(C.c_void_p),
                                       C.c_uint64(400), counts.ctypes.data_as(C.c_void_p))
    assert rc == 0
    a = int(counts[0])
    return out[:a], out[a: a + int(counts[1])]


@pytest.mark.parametrize("idx", list(range(0, 200, 13)))
def test_reach_corpus(ref, idx):
    g, _ = corpus(ref, 0, idx)
    assert_same(run_gpu("reach", {"Edge": g}), run_ref(ref, "reach", {"Edge": g}), ["Reach"])


@pytest.mark.parametrize("idx", list(range(0, 100, 9)))
def test_sg_corpus(ref, idx):
    g, _ = corpus(ref, 1, idx)
    assert_same(run_gpu("sg", {"Edge": g}), run_ref(ref, "sg", {"Edge": g}), ["SG"])


@pytest.mark.parametrize("idx", list(range(0, 50, 7)))
def test_cspa_corpus(ref, idx):
    a, d = corpus(ref, 2, idx)
    db = {"assign": a, "dereference": d}
    assert_same(run_gpu("cspa", db), run_ref(ref, "cspa", db), ["ValueFlow", "ValueAlias", "MemoryAlias"])


# ---- larger synthetic instances ----------------------------------------------

def test_c1_tc_rand_matches_reference_and_survey(ref):
    """n = m = 10^4, mt19937_64 seed 1 -> |Edge| 9,999,
    |Reach| 198,733, 46 iterations."""
    import ctypes as C
    raw = np.zeros((10000, 2), dtype=np.uint64)
    assert ref.lib.ref_gen_tc_rand(C.c_uint64(10000), C.c_uint64(10000), C.c_uint64(1),
                                   raw.ctypes.data_as(C.c_void_p)) == 0
    g = run_gpu("reach", {"Edge": raw})
    r = run_ref(ref, "reach", {"Edge": raw})
    assert g.relation("Reach").count() == 198733
    assert g.stats().iterations == 46
    assert_same(g, r, ["Reach"])
    log = g.iter_log("Reach")
    assert log[:3] == [(9999, 10018, 10017, 10008, 20007), (10008, 9999, 9998, 9996, 30003),
                       (9996, 10013, 10012, 10004, 40007)]


def test_wide_values_engine(ref):
    rng = np.random.default_rng(4)
    e = random_relation(rng, 2, 3000, 800, U64MAX - 2000)
    g = run_gpu("reach", {"Edge": e})
    assert g.encoding()["dictionary"]
    assert_same(g, run_ref(ref, "reach", {"Edge": e}), ["Reach"])


def test_cspa_random_medium(ref):
    rng = np.random.default_rng(8)
    db = {"assign": random_relation(rng, 2, 400, 120), "dereference": random_relation(rng, 2, 500, 120)}
    assert_same(run_gpu("cspa", db), run_ref(ref, "cspa", db), ["ValueFlow", "ValueAlias", "MemoryAlias"])


@pytest.mark.parametrize("chunk", [40, 700, 20000])
@pytest.mark.parametrize("prog", ["cspa", "sg", "reach"])
def test_chunked_final_steps_match_reference(ref, prog, chunk):
    """Host-driven loop with every final join step above `chunk` output rows
    run in row ranges of about that many outputs (chain_chunk_rows), the
    join sink hash-deduplicated between the ranges (engine.cu
    chunked_final_step): relations, Δ history, iterations and the
    reference's charge events, peaks and EBM allocations are unchanged
    (the charges follow the logical join rows)."""
    rng = np.random.default_rng(chunk + len(prog))
    if prog == "cspa":
        db = {"assign": random_relation(rng, 2, 400, 120), "dereference": random_relation(rng, 2, 500, 120)}
        names = ["ValueFlow", "ValueAlias", "MemoryAlias"]
    else:
        db = {"Edge": random_relation(rng, 2, 3000, 1200) if prog == "reach" else random_relation(rng, 2, 900, 700)}
        names = [{"reach": "Reach", "sg": "SG"}[prog]]
    with al.default_context().configured(resident_loop=0, chain_chunk_rows=chunk):
        g = run_gpu(prog, db)
    assert_same(g, run_ref(ref, prog, db), names)


def test_chunked_final_steps_under_budget(ref):
    """Chunked final steps under a finite budget: the reference's budget
    outcome (error phase or peaks) is unchanged."""
    from oracle.bindings import OracleError
    rng = np.random.default_rng(77)
    db = {"assign": random_relation(rng, 2, 300, 100), "dereference": random_relation(rng, 2, 400, 100)}
    for budget in (20_000, 200_000, 2_000_000):
        cfg = al.engine_config(memory_budget_bytes=budget)
        try:
            r = run_ref(ref, "cspa", db, cfg)
        except OracleError as e:
            with pytest.raises(al.budget_error) as ei, al.default_context().configured(chain_chunk_rows=64):
                run_gpu("cspa", db, cfg)
            assert ei.value.phase() == e.phase
            continue
        with al.default_context().configured(chain_chunk_rows=64):
            g = run_gpu("cspa", db, cfg)
        assert_same(g, r, ["ValueFlow", "ValueAlias", "MemoryAlias"])
