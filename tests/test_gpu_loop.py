"""The resident device loop (csrc/loop.cu) against the
host-driven loop and the reference engine: graph (device-side `while`),
eager and host-driven modes give byte-identical relations, identical Δ
histories, iteration records and accountant statistics; min_capacities
(gd_device_config) starts every capacity at its minimum so every overflow -> rollback ->
grow -> re-run path runs.
"""
import numpy as np
import pytest

from paper_2311_02206_b200 import arraylog as al
from tests.helpers import chain_edges, program_from_ref, rows
from tests.test_gpu_engine import CUSTOM, assert_same, corpus, run_gpu, run_ref

pytestmark = pytest.mark.gpu

MODES = {  # gd_device_config fields of each mode
    "graph": {},
    "eager": {"loop_mode": 1},
    "tiny": {"min_capacities": 1},
    "tiny_eager": {"min_capacities": 1, "loop_mode": 1},
    "host": {"resident_loop": 0},
    "hashindex": {"dense_inner": 0},
    "split": {"split_insert": 1},
    "tiny_split": {"min_capacities": 1, "split_insert": 1},
    "tiny_casrehash": {"min_capacities": 1, "rehash_cas_only": 1},
    # final steps over a dense inner: probe/scan/merge-path fused insert
    # instead of count + warp-expanded insert (the default), and the wide
    # expansion rounds (8 keys per lane)
    "noxp": {"warp_expand": 0},
    "xp8": {"warp_expand": 1, "expand_keys_per_lane": 8},
    "xp_split": {"warp_expand": 1, "split_insert": 1},
    # warp expansion with rows of more than 3 outputs queued as (row,
    # segment) items of 3 outputs (the heavy-row path on small inputs)
    "heavy": {"warp_expand": 1, "heavy_rows": 3},
    "tiny_heavy": {"min_capacities": 1, "warp_expand": 1, "heavy_rows": 2},
    # head-index insert variants: CAS first, batched probing, pipelined /
    # narrow materialized-key inserts
    "cas_first": {"insert_slots": 0},
    "batched": {"insert_slots": 2, "split_insert": 1, "insert_per_thread": 4},
    "pipe_insert": {"split_insert": 1, "insert_pipeline": 1},
    "precount": {"precount": 1},
    "tiny_precount": {"precount": 1, "min_capacities": 1, "heavy_rows": 2},
    # chain temps above 7 rows are materialized in windows of 7 (the
    # windowed iteration of SURVEY §8f rank 2), with and without the rest
    # of the capacities at their minimum
    "window": {"temp_limit_rows": 7},
    "tiny_window": {"min_capacities": 1, "temp_limit_rows": 5},
    "window_xp": {"temp_limit_rows": 16, "warp_expand": 1},
    # end-of-round insert variants: count ahead (no loop_count in the graph
    # iteration; eager counts after every rollback), the insert as a
    # programmatic dependent launch, the gate back in loop_count, 2x logs
    "count_ahead": {"count_ahead": 1},
    "tiny_count_ahead": {"count_ahead": 1, "min_capacities": 1},
    "pdl": {"pdl": 1},
    "gate_in_count": {"gate_in_insert": 0},
    "log2": {"log_growth": 2},
    "load35": {"index_load_pct": 35},
    "tiny_load80": {"index_load_pct": 80, "min_capacities": 1},
}


def configured(**fields):
    """The default context with these gd_device_config fields set."""
    return al.default_context().configured(**fields)


def run_mode(mode, program, db):
    with configured(**MODES[mode]):
        return run_gpu(program, db)


def c1_edges(ref):
    import ctypes as C
    raw = np.zeros((10000, 2), dtype=np.uint64)
    assert ref.lib.ref_gen_tc_rand(C.c_uint64(10000), C.c_uint64(10000), C.c_uint64(1),
                                   raw.ctypes.data_as(C.c_void_p)) == 0
    return raw


@pytest.mark.parametrize("mode", sorted(MODES))
def test_c1_all_modes(ref, mode):
    raw = c1_edges(ref)
    g = run_mode(mode, "reach", {"Edge": raw})
    assert g.relation("Reach").count() == 198733
    assert g.stats().iterations == 46
    assert g.iter_log("Reach")[:3] == [(9999, 10018, 10017, 10008, 20007), (10008, 9999, 9998, 9996, 30003),
                                       (9996, 10013, 10012, 10004, 40007)]
    assert_same(g, run_ref(ref, "reach", {"Edge": raw}), ["Reach"])
    assert g.raw_stats().join_tuples == 190496  # SURVEY §6 probe: ΣJ over 46 iterations


@pytest.mark.parametrize("mode", ["graph", "tiny", "eager", "hashindex", "split", "noxp", "xp8", "xp_split", "heavy",
                                  "tiny_heavy", "window", "tiny_window", "window_xp", "cas_first", "batched",
                                  "pipe_insert", "precount", "tiny_precount"])
@pytest.mark.parametrize("idx", [0, 17, 55])
def test_sg_corpus_modes(ref, mode, idx):
    g, _ = corpus(ref, 1, idx)
    assert_same(run_mode(mode, "sg", {"Edge": g}), run_ref(ref, "sg", {"Edge": g}), ["SG"])


@pytest.mark.parametrize("mode", ["graph", "tiny", "tiny_split", "heavy", "window", "tiny_window"])
@pytest.mark.parametrize("case", sorted(CUSTOM))
def test_custom_programs_modes(ref, mode, case):
    src, db = CUSTOM[case]
    r = run_ref(ref, src, db)
    prog = program_from_ref(r)
    assert_same(run_mode(mode, prog, db), r, prog.idbs)


@pytest.mark.parametrize("mode", ["graph", "tiny"])
def test_long_chain_many_iterations(ref, mode):
    """1200-node path: 1199 iterations (> the initial history capacity)."""
    e = chain_edges(1200)
    g = run_mode(mode, "reach", {"Edge": e})
    assert g.stats().iterations == 1199
    assert g.relation("Reach").count() == 1199 * 1200 // 2
    assert_same(g, run_ref(ref, "reach", {"Edge": e}), ["Reach"])


def test_modes_agree_on_power_law(ref):
    from paper_2311_02206_b200 import workloads as W
    e = W.tc_pl(20000, 20000, 100, 1.05, 3)
    outs = {m: run_mode(m, "reach", {"Edge": e}) for m in ("graph", "host", "tiny", "hashindex", "tiny_casrehash",
                                                            "eager", "noxp", "heavy", "tiny_heavy")}
    base = outs["host"]
    for m, g in outs.items():
        assert np.array_equal(g.relation("Reach").data, base.relation("Reach").data), m
        assert g.iter_log("Reach") == base.iter_log("Reach"), m
        assert g.raw_stats().charge_events == base.raw_stats().charge_events, m
        assert g.raw_stats().peak_tracked_bytes == base.raw_stats().peak_tracked_bytes, m
    assert_same(base, run_ref(ref, "reach", {"Edge": e}), ["Reach"])


def test_repeated_engines_reuse_context(ref):
    e = rows([1, 2, 2, 3, 3, 4, 4, 1], 2)
    for _ in range(3):
        g = run_gpu("reach", {"Edge": e})
        assert g.relation("Reach").count() == 16


def test_hash_predup_matches_sort_path():
    """Host-driven loop (CSPA, IDB inners): the hash pre-dedup of mostly
    duplicate join output (dedup.cu) gives the same relations, Δ histories,
    iteration records and accountant stats as sorting every join row."""
    from paper_2311_02206_b200 import workloads as W
    a, d = W.cspa_local(300_000, 72_000, 228_000, 256, 2)
    db = {"assign": a, "dereference": d}
    outs = {}
    for mode, kv in (("1", {"hash_dedup": 1}), ("0", {"hash_dedup": 0}),
                     ("split", {"hash_dedup": 1, "dedup_part_slots": 65536})):
        with configured(**kv):
            outs[mode] = run_gpu("cspa", db)
    g, h = outs["1"], outs["0"]
    for n in ("ValueFlow", "MemoryAlias", "ValueAlias"):
        assert np.array_equal(g.relation(n).data, h.relation(n).data), n
        assert g.iter_log(n) == h.iter_log(n), n
        assert np.array_equal(outs["split"].relation(n).data, h.relation(n).data), n
        assert outs["split"].iter_log(n) == h.iter_log(n), n
    assert max(r[1] for r in g.iter_log("ValueAlias")) >= (1 << 20)  # the hash path ran
    gs, hs = g.raw_stats(), h.raw_stats()
    assert (gs.charge_events, gs.peak_tracked_bytes, gs.join_tuples) == (hs.charge_events, hs.peak_tracked_bytes,
                                                                        hs.join_tuples)


@pytest.mark.parametrize("mode", ["graph", "tiny", "eager", "noxp", "heavy", "tiny_heavy", "precount", "tiny_precount",
                                  "count_ahead", "tiny_count_ahead", "pdl", "gate_in_count"])
def test_hub_rows(ref, mode):
    """Hubs (in-degree 700, out-degree 300) give Δ rows with long match
    ranges next to short ones: the load-balanced expansion must match the
    reference's results, histories and stats."""
    rng = np.random.default_rng(11)
    e = rng.integers(0, 3000, size=(6000, 2), dtype=np.uint64)
    hubs = np.stack([rng.integers(0, 3000, size=700, dtype=np.uint64), np.full(700, 17, dtype=np.uint64)], 1)
    hub2 = np.stack([np.full(300, 5, dtype=np.uint64), rng.integers(0, 3000, size=300, dtype=np.uint64)], 1)
    edges = np.vstack([e, hubs, hub2])
    g = run_mode(mode, "reach", {"Edge": edges})
    assert_same(g, run_ref(ref, "reach", {"Edge": edges}), ["Reach"])


@pytest.mark.parametrize("mode", ["graph", "eager", "tiny"])
def test_stamp_epoch_restart(ref, mode):
    """56-bit keys leave 8 stamp bits: a 599-iteration fixpoint restarts the
    stamp epoch twice (table restamp on the device); results, histories and
    iteration records must equal the reference."""
    n = 600
    ids = (np.arange(n, dtype=np.uint64) * np.uint64(400_000) + np.uint64(7))  # < 2^28: 28 bits per column
    edges = np.stack([ids[:-1], ids[1:]], 1)
    g = run_mode(mode, "reach", {"Edge": edges})
    assert g.encoding()["bits"] >= 28 and not g.encoding()["dictionary"]
    assert g.stats().iterations == n - 1
    assert_same(g, run_ref(ref, "reach", {"Edge": edges}), ["Reach"])
    # Δ_out of every iteration = 599 - i: no key counted twice across epochs
    assert [r[3] for r in g.iter_log("Reach")] == list(range(n - 2, -1, -1))


@pytest.mark.parametrize("mode", ["graph", "eager", "tiny", "tiny_casrehash"])
def test_wide_slots(ref, mode):
    # 31-bit identity-encoded columns: 62-bit keys leave < 8 stamp bits, so
    # the head index uses 16-byte HSlots (key + stamp word) — insertion,
    # zone growth (tiny: every capacity starts at its minimum) and the CAS
    # re-spread on that layout
    rng = np.random.default_rng(11)
    n = 3000
    ids = np.sort(rng.choice(np.uint64(2_000_000_000), n, replace=False).astype(np.uint64))
    src = rng.integers(0, n - 1, 6000)
    dst = np.minimum(src + 1 + rng.integers(0, 40, 6000), n - 1)
    edges = np.unique(np.stack([ids[src], ids[dst]], 1), axis=0)
    g = run_mode(mode, "reach", {"Edge": edges})
    enc = g.encoding()
    assert enc["bits"] == 31 and not enc["dictionary"]
    assert_same(g, run_ref(ref, "reach", {"Edge": edges}), ["Reach"])


@pytest.mark.parametrize("limit", [64, 1000, 20000])
def test_sg_windowed_chain_temps_vs_reference(ref, limit):
    """SG on a bushy random DAG whose step-1 temps reach tens of thousands of
    rows per iteration, with chain temps capped at `limit` rows: the
    iterations whose temp exceeds the cap run in windows; relation, Δ
    history, iteration records and accountant statistics (the reference's
    charges for the whole temp) equal the reference's."""
    rng = np.random.default_rng(limit)
    n = 3000
    child = np.arange(1, n, dtype=np.uint64)
    parent = (child - 1 - rng.integers(0, 40, size=n - 1).astype(np.uint64) % child).astype(np.uint64)
    edges = np.stack([parent, child], 1)
    r = run_ref(ref, "sg", {"Edge": edges})
    with configured(temp_limit_rows=limit):
        g = run_gpu("sg", {"Edge": edges})
    assert_same(g, r, ["SG"])
    with configured(resident_loop=0):
        h = run_gpu("sg", {"Edge": edges})
    assert g.iter_log("SG") == h.iter_log("SG")
    assert g.raw_stats().join_tuples == h.raw_stats().join_tuples
