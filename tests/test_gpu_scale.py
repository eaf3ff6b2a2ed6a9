"""Parity at the benchmark configurations (BASELINE configs C2-C5).

1. Bounded samples of the exact bench generators, byte-compared with the
   reference engine (oracle/_ref) through the resident device loop and the
   host-driven loop: relations, Δ history, iteration count, accountant
   statistics, ΣJ and the device digest.
     - C2 `tc_pl` at bench.py's CPU sample (n = m = 2·10^5, W = 200, α = 1.05)
     - C3 `sg_tree` (n = 3·10^4, W = 300)
     - C4 `cspa_local` (1/25 httpd scale) with the hash pre-dedup forced on
2. Every seeded acceptance corpus of the reference (200 REACH, 100 SG, 50
   CSPA; acceptance_test.cpp:58-89) on the device.
3. Full-scale C2 / C3 / C5, where the CPU engine cannot finish: structural
   invariants checked on the device — rows strictly increasing (canonical),
   Σ Δ-history = |F| (engine_test.cpp:137-145), ΣJ = Σ_{(m,t) ∈ Reach}
   indeg(m) for TC — the resident loop's digest equal to the host-driven
   loop's and to the sum of the shard digests of the native partitioned
   driver over P = 2/4/8 loopback ranks, and everything equal to the
   committed record in tests/golden/scale_digests.json
   (tests/golden/make_scale_golden.py wrote it after the same checks).
"""
import ctypes as C
import hashlib
import json
import threading
from pathlib import Path

import numpy as np
import pytest

from paper_2311_02206_b200 import arraylog as al
from paper_2311_02206_b200 import workloads as W
from tests.helpers import digest_rows
from tests.test_gpu_engine import assert_same, corpus, run_gpu, run_ref

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden" / "scale_digests.json"
MODES = {"graph": {}, "eager": {"loop_mode": 1}, "host": {"resident_loop": 0}}

# bounded samples (reference CPU engine ≈ 5-20 s each on the box's cores)
C2_SAMPLE = dict(n=200_000, m=200_000, window=200, alpha=1.05, seed=1)  # = bench.py CPU_SAMPLE
C3_SAMPLE = dict(n=30_000, window=300, seed=1)
C4_SAMPLE = dict(n=60_000, n_assign=14_480, n_deref=45_600, module=256, seed=1)

# full-scale configs (bench.py C2; workloads.CONFIGS)
SCALE = {
    "c2_tc_pl": dict(program="reach", head="Reach", gen=lambda: W.tc_pl(5_000_000, 5_000_000, 200, 1.05, 1),
                     parts=(2, 4, 8), host=True),
    "c3_sg_tree_w1000": dict(program="sg", head="SG", gen=lambda: W.sg_tree(1_000_001, 1000, 1),
                             parts=(2, 4), host=True),
    # C5 (|Reach| 2.5e9, 20 GB of keys) on one B200: the resident loop with
    # the invariants; two loopback shards of it do not fit one GPU's HBM
    "c5_tc_dag": dict(program="reach", head="Reach", gen=lambda: W.tc_dag(100_000_000, 100_000_000, 200, 1),
                      parts=(), host=False),
}


def configured(**kv):
    return al.default_context().configured(**kv)


def tc_join_tuples(edges: np.ndarray, reach: np.ndarray) -> int:
    """ΣJ of Reach(f,t) :- Edge(f,m), Reach(m,t): every Reach row enters Δ
    once and joins with indeg(m) distinct edges."""
    e = np.unique(edges, axis=0)
    indeg = np.bincount(e[:, 1].astype(np.int64), minlength=int(max(e.max(), reach.max())) + 1)
    return int(indeg[reach[:, 0].astype(np.int64)].sum())


def hist_sha(h) -> str:
    return hashlib.sha256(np.asarray(h, dtype=np.uint64).tobytes()).hexdigest()[:16]


# ---- 1. bounded samples of the bench generators vs the reference ----------

@pytest.fixture(scope="module")
def c2_sample(ref):
    s = C2_SAMPLE
    edges = W.tc_pl(s["n"], s["m"], s["window"], s["alpha"], s["seed"])
    return edges, run_ref(ref, "reach", {"Edge": edges})


@pytest.mark.parametrize("mode", sorted(MODES))
def test_c2_bench_sample_vs_reference(c2_sample, mode):
    edges, r = c2_sample
    with configured(**MODES[mode]):
        g = run_gpu("reach", {"Edge": edges})
    assert_same(g, r, ["Reach"])
    reach = r.relation("Reach")
    assert len(reach) == 7_178_880  # bench.py's reference arm prints the same count
    assert g.raw_stats().join_tuples == tc_join_tuples(edges, reach)
    assert g.relation_digest("Reach") == digest_rows(reach)
    log = g.iter_log("Reach")
    assert [x[0] for x in log] == r.delta_history("Reach")
    assert log[-1][3] == 0 and log[-1][4] == len(reach)
    g.close()


@pytest.fixture(scope="module")
def c3_sample(ref):
    s = C3_SAMPLE
    edges = W.sg_tree(s["n"], s["window"], s["seed"])
    return edges, run_ref(ref, "sg", {"Edge": edges})


@pytest.mark.parametrize("mode", sorted(MODES))
def test_c3_sg_tree_sample_vs_reference(c3_sample, mode):
    edges, r = c3_sample
    with configured(**MODES[mode]):
        g = run_gpu("sg", {"Edge": edges})
    assert_same(g, r, ["SG"])
    assert g.relation_digest("SG") == digest_rows(r.relation("SG"))
    assert g.relation("SG").count() > 4_000_000
    g.close()


@pytest.fixture(scope="module")
def c4_sample(ref):
    s = C4_SAMPLE
    a, d = W.cspa_local(s["n"], s["n_assign"], s["n_deref"], s["module"], s["seed"])
    db = {"assign": a, "dereference": d}
    return db, run_ref(ref, "cspa", db)


@pytest.mark.parametrize("mode", ["predup", "predup_split", "sort"])
def test_c4_cspa_sample_vs_reference(c4_sample, mode):
    """CSPA (IDB inners, host-driven loop) with the hash pre-dedup of
    duplicate-heavy join output forced on (every join output of ≥ 4096 rows;
    predup_split: L2 parts of 4096 slots), and with plain sort dedup."""
    db, r = c4_sample
    kv = {"predup": {"hash_dedup": 1, "hash_dedup_min_rows": 4096},
          "predup_split": {"hash_dedup": 1, "hash_dedup_min_rows": 4096, "dedup_part_slots": 4096},
          "sort": {"hash_dedup": 0}}[mode]
    names = ["ValueFlow", "ValueAlias", "MemoryAlias"]
    with configured(**kv):
        g = run_gpu("cspa", db)
    assert_same(g, r, names)
    for n in names:
        assert g.relation_digest(n) == digest_rows(r.relation(n)), n
    if mode != "sort":  # the pre-dedup path ran: many join outputs collapsed ≥ 4x
        log = g.iter_log("ValueAlias")
        assert any(j >= 4096 and 4 * u < j for _, j, u, _, _ in log)
    g.close()


# ---- 2. every acceptance corpus -------------------------------------------

@pytest.mark.parametrize("kind,prog,names,count", [
    (0, "reach", ["Reach"], 200), (1, "sg", ["SG"], 100),
    (2, "cspa", ["ValueFlow", "ValueAlias", "MemoryAlias"], 50)])
def test_all_acceptance_corpora(ref, kind, prog, names, count):
    """acceptance_test.cpp criteria 1-3 (seeds 20240601-20240603): all
    corpora, not a stride sample."""
    for idx in range(count):
        a, b = corpus(ref, kind, idx)
        db = {"Edge": a} if kind < 2 else {"assign": a, "dereference": b}
        g = run_gpu(prog, db)
        try:
            assert_same(g, run_ref(ref, prog, db), names)
        except AssertionError as ex:
            raise AssertionError(f"{prog} corpus {idx}: {ex}") from ex
        g.close()


# ---- 3. full scale: invariants, cross-mode and cross-partition digests ----

def device_rows(e, head):
    import torch
    n = e.relation_count(head)
    t = torch.empty((max(n, 1), 2), dtype=torch.int64, device="cuda")
    e.ctx.check(e.ctx.lib.gd_engine_relation_download_device(e.h, e._rid(head), C.c_void_p(t.data_ptr()), n))
    e.ctx.synchronize()
    return t[:n]


def check_invariants(e, head, program, edges):
    """Device-side checks of a full-size result (no CPU engine at this size)."""
    import torch
    e.ctx.trim()  # the fixpoint's cached device blocks back to the driver (torch allocates below)
    rows = device_rows(e, head)
    n = rows.shape[0]
    hist = e.delta_history(head)
    assert sum(hist) == n  # Σ Δ = |F| (engine_test.cpp:137-145)
    log = e.iter_log(head)
    assert [x[0] for x in log] == hist and log[-1][3] == 0 and log[-1][4] == n
    step = 1 << 27
    indeg = None
    if program == "reach":
        ed = torch.from_numpy(edges.view(np.int64)).cuda()
        key = torch.unique(ed[:, 0] << 32 | ed[:, 1])  # distinct edges (ids < 2^31)
        indeg = torch.bincount(key & 0xFFFFFFFF, minlength=int(rows[:, 0].max().item()) + 1 if n else 1)
        del ed, key
    jt = 0
    for i in range(0, n, step):  # strictly increasing, chunked (bounded temporaries)
        a = rows[i: min(n, i + step + 1)]
        b0, b1, a0, a1 = a[1:, 0], a[1:, 1], a[:-1, 0], a[:-1, 1]
        assert bool(((b0 > a0) | ((b0 == a0) & (b1 > a1))).all()), f"rows not canonical near {i}"
        if indeg is not None:
            jt += int(indeg[rows[i: i + step, 0]].sum().item())
    if indeg is not None:
        assert jt == e.raw_stats().join_tuples  # ΣJ = Σ_{(m,t) ∈ Reach} indeg(m)
    del rows
    torch.cuda.empty_cache()


def record_of(e, head):
    s = e.raw_stats()
    return {"count": e.relation_count(head), "digest": f"{e.relation_digest(head):016x}",
            "iterations": int(s.iterations), "join_tuples": int(s.join_tuples),
            "delta_history_sha": hist_sha(e.delta_history(head))}


def run_loopback(program, head, edges, P, name=None):
    """The native partitioned driver over P loopback ranks (threads, one
    context each); returns the union record (shard digests add up).  Up to
    3 ranks use the peer exchange, more the NCCL exchange (peer-exchange
    ranks sharing one GPU need a hardware queue each, test_gpu_partition)."""
    import gc
    gc.collect()
    from paper_2311_02206_b200.partition import LoopbackComms, run_partitioned_native
    ctxs = [al.Context(0, config={"partition_exchange": 0 if P <= 3 else 1}) for _ in range(P)]
    lb = LoopbackComms(ctxs[0], P)
    engines = []
    for r in range(P):
        e = al.engine(program, ctx=ctxs[r])
        e.set_partition(r, P)
        e.load_edb("Edge", al.tuple_array(2, edges))
        e.seed()
        engines.append(e)
    iters, errs = [None] * P, []

    def work(r):
        try:
            iters[r] = run_partitioned_native(engines[r], lb.comms[r])
        except Exception as ex:  # noqa: BLE001
            errs.append(ex)

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    assert all(not t.is_alive() for t in th)
    hists = [e.delta_history(head) for e in engines]
    hist = [sum(h[i] for h in hists) for i in range(iters[0])]
    rec = {"count": sum(e.relation_count(head) for e in engines),
           "digest": f"{sum(e.relation_digest(head) for e in engines) % (1 << 64):016x}",
           "iterations": int(iters[0]), "join_tuples": sum(int(e.raw_stats().join_tuples) for e in engines),
           "delta_history_sha": hist_sha(hist)}
    assert iters == [iters[0]] * P
    for e in engines:
        e.close()
    lb.close()
    for c in ctxs:
        c.close()
    return rec


def scale_records(name, check=True):
    """Every record of one full-scale config (resident loop, host loop,
    loopback partitions), after the invariant checks."""
    cfg = SCALE[name]
    edges = cfg["gen"]()
    out = {}
    g = run_gpu(cfg["program"], {"Edge": edges})
    if check:
        check_invariants(g, cfg["head"], cfg["program"], edges)
    out["resident"] = record_of(g, cfg["head"])
    g.close()
    al.default_context().trim()
    if cfg["host"]:
        with configured(resident_loop=0):
            h = run_gpu(cfg["program"], {"Edge": edges})
        out["host"] = record_of(h, cfg["head"])
        h.close()
        al.default_context().trim()
    for P in cfg["parts"]:
        out[f"loopback_p{P}"] = run_loopback(cfg["program"], cfg["head"], edges, P, name)
    return out


@pytest.mark.parametrize("name", sorted(SCALE))
def test_full_scale_digests(name):
    golden = json.loads(GOLD.read_text())
    assert name in golden, f"no golden record for {name}: run tests/golden/make_scale_golden.py on a B200"
    recs = scale_records(name)
    base = recs["resident"]
    for k, r in recs.items():
        assert r == base, (k, r, base)
    assert base == golden[name]["record"], (base, golden[name]["record"])
