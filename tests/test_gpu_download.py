"""Host download of large relations (engine.relation): packed keys cross
PCIe and host threads unpack them (engine.cu download_packed); the rows
must equal the device-unpack path and the numpy canonical form."""

import numpy as np
import pytest

from paper_2311_02206_b200 import arraylog as al
from tests.helpers import program_from_ref

pytestmark = pytest.mark.gpu

COPY2 = ".decl E(2)\nC(x, y) :- E(x, y).\n"
COPY3 = ".decl E(3)\nC(x, y, z) :- E(x, y, z).\n"


def canonical(a):
    return np.unique(a, axis=0)


@pytest.mark.parametrize("delta", [2, 1, 0])
@pytest.mark.parametrize("arity,n,hi", [(2, 3_000_000, 1 << 20), (3, 2_100_000, 1 << 14), (2, 40_000_000, 1 << 30)])
def test_host_unpack_matches(ref, arity, n, hi, delta):
    """Downloads of packed keys (delta-compressed or plain) unpacked by host
    threads equal the device-unpacked rows and the canonical input."""
    src = COPY2 if arity == 2 else COPY3
    r = ref.engine(src)
    prog = program_from_ref(r)
    rng = np.random.default_rng(arity * 7 + n)
    e = rng.integers(0, hi, size=(n, arity), dtype=np.uint64)
    outs = {}
    for mode in ("1", "0"):
        with al.default_context().configured(host_unpack=int(mode), download_delta=delta):
            g = al.engine(prog)
            g.load_edb("E", al.tuple_array(arity, e))
            g.run()
            outs[mode] = g.relation("C").data.copy()
    assert np.array_equal(outs["1"], outs["0"])
    assert np.array_equal(outs["1"].reshape(-1, arity), canonical(e))


@pytest.mark.parametrize("frac", ["0.25", "0.6"])
def test_pinned_destination_direct_tail(ref, frac):
    """(download_delta = 0: the transfer counter is checked against the
    plain packed-key formula; the delta path is covered below.)"""
    """Into a pinned destination the tail rows are unpacked on the device
    and DMA'd straight into the caller's rows on a second stream while the
    host unpacks the head (download_packed): same bytes as a pageable
    destination, and the transfer counter includes the direct rows."""
    import ctypes as C

    import torch

    r = ref.engine(COPY2)
    prog = program_from_ref(r)
    rng = np.random.default_rng(77)
    e = rng.integers(0, 1 << 22, size=(6_000_000, 2), dtype=np.uint64)
    g = al.engine(prog)
    g.load_edb("E", al.tuple_array(2, e))
    g.run()
    rid = g._rid("C")
    n = g.relation_count("C")
    want = canonical(e)
    assert n == len(want)
    pinned = torch.empty((n, 2), dtype=torch.int64).pin_memory().numpy().view(np.uint64)
    with g.ctx.configured(download_direct_frac=float(frac), download_delta=0):
        h0, d0 = g.ctx.transfer_bytes()
        g.ctx.check(g.ctx.lib.gd_engine_relation_download(g.h, rid, pinned.ctypes.data_as(C.c_void_p), n))
        h1, d1 = g.ctx.transfer_bytes()
    assert np.array_equal(pinned, want)
    nd = int(n * float(frac))
    assert d1 - d0 == (n - nd) * 8 + nd * 16  # packed head + unpacked direct tail


@pytest.mark.parametrize("case", ["dense", "sparse", "mixed", "wide3", "tail"])
def test_delta_download_gap_widths(ref, case):
    """Delta-compressed download across gap widths: runs of consecutive keys
    (1-bit gaps), sparse keys (wide gaps), blocks mixing both, arity-3 keys
    with 60-bit packed values (gaps up to 60 bits) and sizes that end in a
    partial block — rows equal the canonical input; the compressed transfer
    is smaller than 8 bytes per row for dense data."""
    rng = np.random.default_rng(hash(case) & 0xffff)
    if case == "dense":
        e = np.stack([np.repeat(np.arange(1500, dtype=np.uint64), 1000), np.tile(np.arange(1000, dtype=np.uint64), 1500)], 1)
        arity = 2
    elif case == "sparse":
        e = rng.integers(0, 1 << 31, size=(1_500_000, 2), dtype=np.uint64)
        arity = 2
    elif case == "mixed":
        a = np.stack([np.zeros(1_000_000, np.uint64), np.arange(1_000_000, dtype=np.uint64)], 1)
        b = rng.integers(1, 1 << 30, size=(600_000, 2), dtype=np.uint64)
        e = np.vstack([a, b])
        arity = 2
    elif case == "wide3":
        e = rng.integers(0, 1 << 20, size=(1_200_000, 3), dtype=np.uint64)
        arity = 3
    else:
        e = rng.integers(0, 1 << 22, size=(1_048_576 + 37, 2), dtype=np.uint64)
        arity = 2
    prog = program_from_ref(ref.engine(COPY2 if arity == 2 else COPY3))
    want = canonical(e)
    outs = {}
    for delta in (2, 1, 0):
        with al.default_context().configured(download_delta=delta):
            g = al.engine(prog)
            g.load_edb("E", al.tuple_array(arity, e))
            g.run()
            h0, d0 = g.ctx.transfer_bytes()
            outs[delta] = g.relation("C").data.copy()
            h1, d1 = g.ctx.transfer_bytes()
            outs[f"bytes{delta}"] = d1 - d0
    assert np.array_equal(outs[1].reshape(-1, arity), want)
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(outs[2], outs[1])
    if case == "dense":
        assert outs["bytes1"] < 2 * len(want)  # ~1.2 bits per gap + block headers
        # byte offsets: 1 byte per row + 9 bytes per 32-row block (+ unit offsets)
        assert outs["bytes2"] < 1.4 * len(want)


@pytest.mark.parametrize("delta", [2, 1])
@pytest.mark.parametrize("frac", ["0.0", "0.1", "0.5"])
def test_pinned_destination_delta(ref, frac, delta):
    """Delta-compressed head + device-unpacked direct tail into a pinned
    destination: same rows as the canonical input."""
    import ctypes as C

    import torch

    prog = program_from_ref(ref.engine(COPY2))
    rng = np.random.default_rng(78)
    e = rng.integers(0, 1 << 22, size=(3_000_000, 2), dtype=np.uint64)
    g = al.engine(prog)
    g.load_edb("E", al.tuple_array(2, e))
    g.run()
    rid = g._rid("C")
    n = g.relation_count("C")
    pinned = torch.empty((n, 2), dtype=torch.int64).pin_memory().numpy().view(np.uint64)
    with g.ctx.configured(download_direct_frac=float(frac), download_delta=delta):
        g.ctx.check(g.ctx.lib.gd_engine_relation_download(g.h, rid, pinned.ctypes.data_as(C.c_void_p), n))
    assert np.array_equal(pinned, canonical(e))


@pytest.mark.parametrize("arity", [2, 3])
@pytest.mark.parametrize("shift", [0, 1, 2, 3])
def test_byte_download_destination_alignment(ref, arity, shift):
    """Byte-offset download (download_delta = 2) into destinations at every
    16-byte shift of a 64-byte line (the vector rebuild needs 64-byte
    aligned rows; the others take the scalar rebuild) and into arity-3
    rows: same rows as the canonical input, and the bytes just past the
    destination are untouched."""
    import ctypes as C

    prog = program_from_ref(ref.engine(COPY2 if arity == 2 else COPY3))
    rng = np.random.default_rng(91 + shift)
    e = rng.integers(0, 1 << 17, size=(2_000_003, arity), dtype=np.uint64)
    g = al.engine(prog)
    g.load_edb("E", al.tuple_array(arity, e))
    g.run()
    rid = g._rid("C")
    n = g.relation_count("C")
    back = np.full(n * arity + 16, 0xABABABABABABABAB, dtype=np.uint64)
    base = (-(back.ctypes.data // 8)) % 8  # first 64-byte aligned word
    out = back[base + 2 * shift: base + 2 * shift + n * arity]
    with g.ctx.configured(download_delta=2):
        g.ctx.check(g.ctx.lib.gd_engine_relation_download(g.h, rid, out.ctypes.data_as(C.c_void_p), n))
    assert np.array_equal(out.reshape(-1, arity), canonical(e))
    rest = back[base + 2 * shift + n * arity:]
    assert (rest == 0xABABABABABABABAB).all()


def _reach_rows(edges, shift=None, **cfg):
    """Reach of `edges` downloaded through the C-ABI (optionally into a
    destination shifted by `shift` 16-byte rows from a 64-byte line)."""
    import ctypes as C

    from paper_2311_02206_b200.builtins import REACH

    with al.default_context().configured(**cfg):
        g = al.engine(REACH)
        g.load_edb("Edge", al.tuple_array(2, edges))
        g.run()
        rid = g._rid("Reach")
        n = g.relation_count("Reach")
        back = np.zeros(2 * n + 16, dtype=np.uint64)
        base = (-(back.ctypes.data // 8)) % 8
        s = 2 * (shift or 0)
        out = back[base + s: base + s + 2 * n]
        g.ctx.check(g.ctx.lib.gd_engine_relation_download(g.h, rid, out.ctypes.data_as(C.c_void_p), n))
        hist = g.delta_history("Reach")
        g.close()
    return out.reshape(-1, 2), hist


@pytest.mark.parametrize("shift", [0, 1, 3])
def test_segmented_final_sort_download(shift):
    """Segmented final sort + per-segment packed download (download_pipeline,
    PipedPack in engine.cu) on the C2 generator at the CPU-sample scale
    (7.2 M Reach rows, 64 top-digit segments): the rows equal the plain
    sort + byte-offset download and the numpy canonical order, into aligned
    and line-misaligned destinations."""
    from paper_2311_02206_b200 import workloads as W

    edges = W.tc_pl(200_000, 200_000, 200, 1.05, 1)
    got, h1 = _reach_rows(edges, shift, download_pipeline=1, download_pipeline_min_rows=1 << 20)
    want, h0 = _reach_rows(edges, 0, download_pipeline=0)
    assert len(got) > (1 << 20)
    assert h1 == h0
    assert np.array_equal(got, want)
    k = got[:, 0] << np.uint64(32) | got[:, 1]
    assert (np.diff(k.astype(np.uint64)) > 0).all()


def test_segmented_final_sort_small_relations():
    """The segmented sort on cyclic and chain graphs (host download of the
    segment packs) and below the host-unpack size (device unpack of the
    segment-sorted keys): rows and Δ history equal the plain sort's."""
    rng = np.random.default_rng(5)
    cases = [rng.integers(0, 2000, size=(6000, 2), dtype=np.uint64),  # Reach ~ 4 M rows
             np.stack([np.arange(2999), np.arange(1, 3000)], 1).astype(np.uint64),  # chain, 4.5 M rows
             rng.integers(0, 500, size=(1500, 2), dtype=np.uint64)]  # < 1 M rows
    for edges in cases:
        got, h1 = _reach_rows(edges, None, download_pipeline=1, download_pipeline_min_rows=1)
        want, h0 = _reach_rows(edges, None, download_pipeline=0)
        assert h1 == h0
        assert np.array_equal(got, want)


@pytest.mark.parametrize("arity,n,hi", [(2, 3_000_000, 1 << 20), (3, 2_100_000, 1 << 14), (2, 40_000_000, 1 << 30)])
def test_overlapped_pack_download(ref, arity, n, hi):
    """Byte-offset download with the packing overlapped (download_overlap_pack:
    4 M-row chunks packed with events, copies and rebuild starting on chunk
    0; 40 M rows = 10 chunks through a ring of 6 staging areas): rows equal
    the canonical input and the whole-array pack."""
    src = COPY2 if arity == 2 else COPY3
    prog = program_from_ref(ref.engine(src))
    rng = np.random.default_rng(arity * 13 + n)
    e = rng.integers(0, hi, size=(n, arity), dtype=np.uint64)
    outs = {}
    for ov in (1, 0):
        with al.default_context().configured(download_delta=2, download_overlap_pack=ov):
            g = al.engine(prog)
            g.load_edb("E", al.tuple_array(arity, e))
            g.run()
            outs[ov] = g.relation("C").data.copy()
    assert np.array_equal(outs[1], outs[0])
    assert np.array_equal(outs[1].reshape(-1, arity), canonical(e))
