"""GPU parity of the kernel-level entries against the reference functions
(oracle/_ref, the unmodified arraylog headers): bit-exact bytes.

Mirrors tests/tuple_array_test.cpp, hash_index_test.cpp and ra_test.cpp of
the reference, plus wide-value, empty, duplicate-heavy and larger cases.
"""
import numpy as np
import pytest

from paper_2311_02206_b200 import arraylog as al
from tests.helpers import F, I, K, O, U64MAX, random_relation, rows, spec

pytestmark = pytest.mark.gpu


def gd_canon(a, arity):
    return al.canonicalize(al.tuple_array(arity, a)).data


# ---- canonicalize (tuple_array_test.cpp:12-58) ----------------------------

def test_canonicalize_known_answer():
    # tuple_array_test.cpp:12-17: {2,1,1,2,2,1} -> {1,2,2,1}
    c = al.canonicalize(al.tuple_array(2, [2, 1, 1, 2, 2, 1]))
    assert c.canonical
    assert c.data.reshape(-1).tolist() == [1, 2, 2, 1]


def test_canonicalize_empty():
    c = al.canonicalize(al.tuple_array(1))
    assert c.count() == 0 and c.canonical


@pytest.mark.parametrize("arity,n,domain,high", [
    (2, 1000, 10, 0), (2, 5000, 1 << 20, 0), (3, 2000, 6, 0), (1, 3000, 50, 0),
    (2, 4000, 1000, U64MAX - 3000),           # values near 2^64-2: dictionary path
    (4, 3000, 1 << 40, 0),                    # 160 bits: dictionary / u128 path
    (2, 200000, 1 << 31, 0),                  # multi-tile sort
    (5, 1000, 3, (1 << 62)),                  # arity 5 with huge values
])
def test_canonicalize_matches_reference(ref, arity, n, domain, high):
    rng = np.random.default_rng(7 + arity + n)
    a = random_relation(rng, arity, n, domain, high)
    # duplicate-heavy: repeat a slice
    a = np.vstack([a, a[: n // 3]])
    got = gd_canon(a, arity)
    exp = ref.canonicalize(a, arity)
    assert got.dtype == np.uint64
    assert np.array_equal(got, exp)


def test_canonicalize_idempotent():
    rng = np.random.default_rng(11)
    for _ in range(5):
        a = random_relation(rng, 3, 200, 6)
        once = al.canonicalize(al.tuple_array(3, a))
        twice = al.canonicalize(al.tuple_array(3, once.data))
        assert np.array_equal(once.data, twice.data)


def test_canonicalize_large_portions(ref):
    # 2^26+ rows of 48-bit keys with duplicates (one look-back portion since
    # kPortion = 2^28; test_canonicalize_multi_portion crosses portions)
    rng = np.random.default_rng(5)
    n = (1 << 26) + 12345
    a = rng.integers(0, 1 << 24, size=(n, 2), dtype=np.uint64)
    got = gd_canon(a, 2)
    # property check at full size: strictly increasing rows + count of
    # distinct rows equals numpy's
    keys = (got[:, 0] << np.uint64(24)) | got[:, 1]
    assert np.all(keys[1:] > keys[:-1])
    ka = np.unique((a[:, 0] << np.uint64(24)) | a[:, 1])
    assert np.array_equal(ka, keys)


def test_canonicalize_multi_portion():
    # > 2^28 keys: several onesweep look-back portions per pass (radix_sort.cu
    # kPortion).  Distinct 40-bit keys in scrambled order (an odd multiplier
    # is a bijection mod 2^40); size-independent checks: length, strict
    # order and the wrap-around sum of the keys.
    n = (1 << 28) + 12345
    k = (np.arange(n, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)) & np.uint64((1 << 40) - 1)
    got = gd_canon(k.reshape(-1, 1), 1).reshape(-1)
    assert len(got) == n
    assert np.all(got[1:] > got[:-1])
    assert np.sum(got, dtype=np.uint64) == np.sum(k, dtype=np.uint64)


# ---- permute_columns (tuple_array_test.cpp:60-94) ---------------------------

def test_permute_known_answer():
    rel = al.canonicalize(al.tuple_array(2, [1, 2, 3, 1]))
    p = al.permute_columns(rel, [1, 0])
    assert p.data.reshape(-1).tolist() == [1, 3, 2, 1]
    assert np.array_equal(al.permute_columns(rel, [0, 1]).data, rel.data)


def test_permute_round_trip_and_errors(ref):
    rng = np.random.default_rng(3)
    a = ref.canonicalize(random_relation(rng, 3, 500, 9), 3)
    rel = al.tuple_array(3, a, canonical=True)
    for perm in ([1, 2, 0], [2, 0, 1], [0, 2, 1]):
        got = al.permute_columns(rel, perm).data
        assert np.array_equal(got, ref.permute_columns(a, 3, perm))
    with pytest.raises(al.config_error):
        al.permute_columns(rel, [0, 0, 1])
    with pytest.raises(al.config_error):
        al.permute_columns(rel, [0, 1])
    with pytest.raises(al.logic_error):
        al.permute_columns(al.tuple_array(3, a, canonical=False), [1, 2, 0])


# ---- prefix hash / index (hash_index_test.cpp) -----------------------------

def test_prefix_hash_bit_exact(ref):
    rng = np.random.default_rng(1)
    a = np.vstack([random_relation(rng, 3, 3000, 1 << 63),
                   np.array([[0, 0, 0], [U64MAX - 1, 1, 2]], dtype=np.uint64)])
    for ncols in (1, 2, 3):
        assert np.array_equal(al.prefix_hash(a, ncols), ref.prefix_hash(a, 3, ncols))


def test_index_known_answers():
    # hash_index_test.cpp:59-79
    c = al.make_container(al.canonicalize(al.tuple_array(2, [35, 100, 11, 101, 46, 102, 97, 103])), None, 1)
    assert [al.range_lookup(c, [k]) for k in (11, 35, 46, 97)] == [
        al.row_range(0, 1), al.row_range(1, 1), al.row_range(2, 1), al.row_range(3, 1)]
    c = al.make_container(al.canonicalize(al.tuple_array(2, [1, 2, 1, 5, 4, 9])), None, 1)
    assert al.range_lookup(c, [1]) == al.row_range(0, 2)
    assert al.range_lookup(c, [4]) == al.row_range(2, 1)
    assert al.range_lookup(c, [5]).empty()
    c1 = al.make_container(al.canonicalize(al.tuple_array(2, [7, 8])), None, 1)
    assert c1.index.occupied() == 1
    with pytest.raises(al.usage_error):
        al.range_lookup(al.make_container(al.canonicalize(al.tuple_array(2, [7, 8]))), [7])
    with pytest.raises(al.usage_error):
        al.range_lookup(c1, [7, 8])


def test_build_index_rejects_bad_params():
    # hash_index_test.cpp:81-89
    t = al.canonicalize(al.tuple_array(2, [1, 2]))
    for lf in (0.0, 1.0, -0.5, 1.5):
        with pytest.raises(al.config_error):
            al.build_index(t, 1, lf)
    for pl in (0, 3):
        with pytest.raises(al.config_error):
            al.build_index(t, pl, 0.8)
    with pytest.raises(al.logic_error):
        al.build_index(al.tuple_array(2, [1, 2]), 1, 0.8)


@pytest.mark.parametrize("arity,plen,n,domain,high,lf", [
    (2, 1, 200, 40, 0, 0.8), (2, 1, 20000, 3000, 0, 0.8), (3, 2, 5000, 20, 0, 0.5),
    (2, 2, 3000, 100, 0, 0.9), (2, 1, 4000, 500, U64MAX - 1000, 0.8), (4, 3, 3000, 7, 1 << 50, 0.8),
])
def test_range_lookup_matches_reference(ref, arity, plen, n, domain, high, lf):
    rng = np.random.default_rng(n + plen)
    a = ref.canonicalize(random_relation(rng, arity, n, domain, high), arity)
    keys = np.vstack([a[:, :plen], random_relation(rng, plen, 500, domain + 5, high)]).astype(np.uint64)
    c = al.make_container(al.tuple_array(arity, a, canonical=True), None, plen, lf)
    st, ct = al.range_lookup_batch(c, keys)
    est, ect, esc, eoc = ref.index_lookup(a, arity, plen, keys, lf)
    assert np.array_equal(ct, ect)
    assert np.array_equal(st[ct > 0], est[ect > 0])
    assert (c.index.slot_count(), c.index.occupied()) == (esc, eoc)
    assert c.index.occupied() <= lf * c.index.slot_count()


def test_group_starts_match_reference(ref):
    rng = np.random.default_rng(9)
    a = ref.canonicalize(random_relation(rng, 3, 3000, 8), 3)
    for plen in (1, 2, 3):
        got = al.group_starts(al.tuple_array(3, a, canonical=True), plen)
        assert np.array_equal(got, ref.group_starts(a, 3, plen))


# ---- joins (ra_test.cpp) ----------------------------------------------------

def cont(flat, arity, plen=None):
    return al.make_container(al.canonicalize(al.tuple_array(arity, flat)), None, plen)


def test_join_known_answers():
    both = al.column_map([al.operand.outer(1), al.operand.inner(1)])
    o, i = cont([1, 3], 2), cont([1, 2, 1, 5, 4, 9], 2, 1)
    assert al.join_count(al.join_spec(1, o, i, both)) == 2          # ra_test.cpp:38-43
    o, i = cont([7, 1, 8, 2], 2), cont([1, 2, 4, 9], 2, 1)
    assert al.join_count(al.join_spec(1, o, i, both)) == 0          # :45-50
    o, i = cont([0, 1, 0, 2, 0, 3], 2), cont([0, 1, 0, 2, 0, 3], 2, 1)
    s = al.join_spec(1, o, i, both)
    out = al.tuple_array(2, np.zeros((al.join_count(s), 2)))
    al.join_materialize(s, out)
    assert out.count() == 9                                          # :87-95
    o, i = cont([0, 1, 0, 2], 2), cont([0, 1, 0, 2], 2, 1)
    s = al.join_spec(1, o, i, both, [al.row_filter(al.operand.outer(1), al.operand.inner(1), False)])
    assert al.join_count(s) == 2                                     # :106-116
    out = al.tuple_array(2, np.zeros((2, 2)))
    al.join_materialize(s, out)
    assert sorted(map(tuple, al.canonicalize(out).data.tolist())) == [(1, 2), (2, 1)]


def test_join_capacity_mismatch_is_logic_error():
    both = al.column_map([al.operand.outer(1), al.operand.inner(1)])
    s = al.join_spec(1, cont([1, 3], 2), cont([1, 2, 1, 5], 2, 1), both)
    with pytest.raises(al.logic_error):
        al.join_materialize(s, al.tuple_array(2, np.zeros((1, 2))))


def test_join_validation_errors():
    # ra_test.cpp:309-326
    both = al.column_map([al.operand.outer(1), al.operand.inner(1)])
    o, i_noidx = cont([1, 2], 2), cont([1, 2], 2)
    with pytest.raises(al.usage_error):
        al.join_count(al.join_spec(1, o, i_noidx, both))
    with pytest.raises(al.config_error):
        al.join_count(al.join_spec(1, o, cont([1, 2], 2, 1), al.column_map([])))
    with pytest.raises(al.config_error):
        al.join_count(al.join_spec(3, o, cont([1, 2], 2, 1), both))
    with pytest.raises(al.config_error):
        al.join_count(al.join_spec(1, o, cont([1, 2], 2, 1), al.column_map([al.operand.inner(5)])))
    with pytest.raises(al.usage_error):
        al.join_count(al.join_spec(1, o, cont([1, 2], 2, 2), both))


JOIN_CASES = [
    # (outer n, domain, inner n, proj, filters, jcc, high)
    (200, 15, 200, [O(1), I(1)], [], 1, 0),
    (150, 12, 150, [O(1), I(1), K(7)], [], 1, 0),
    (300, 10, 300, [I(1), O(1)], [F(O(1), I(1), False)], 1, 0),
    (300, 10, 300, [O(0), I(1)], [F(O(1), K(3), True)], 1, 0),
    (40, 8, 30, [O(1), I(1)], [], 0, 0),                       # Cartesian (jcc 0)
    (5000, 800, 20000, [I(1), O(1)], [], 1, 0),
    (3000, 400, 3000, [O(1), I(1)], [], 2, 0),
    (2000, 300, 2000, [I(1), O(1)], [], 1, U64MAX - 400),      # dictionary path
    (100, 30, 4000, [O(1), I(1)], [F(O(1), K(1 << 63), True)], 1, 0),  # absent constant
]


@pytest.mark.parametrize("on,dom,inn,proj,filters,jcc,high", JOIN_CASES)
def test_join_raw_bytes_match_reference(ref, on, dom, inn, proj, filters, jcc, high):
    """Raw materialize bytes (outer-row then inner-range order) equal the
    reference's (ra_test.cpp:134-152 pins that order)."""
    rng = np.random.default_rng(on * 7 + inn)
    o = ref.canonicalize(random_relation(rng, 2, on, dom, high), 2)
    i = ref.canonicalize(random_relation(rng, 2, inn, dom, high), 2)
    # power-law hub: one key with many inner rows
    s = spec(jcc, proj, filters)
    exp = ref.join(o, 2, i, 2, s, index_prefix=jcc)
    oc = al.relation_container(al.tuple_array(2, o, canonical=True))
    ic = al.make_container(al.tuple_array(2, i, canonical=True), None, jcc or None)
    js = al.join_spec(jcc, oc, ic, al.column_map(list(proj)), list(filters))
    assert al.join_count(js) == len(exp)
    out = al.tuple_array(len(proj), np.zeros((len(exp), len(proj))))
    al.join_materialize(js, out)
    assert np.array_equal(out.data, exp)


def test_join_skewed_hub(ref):
    rng = np.random.default_rng(77)
    hub = np.column_stack([np.zeros(30000, dtype=np.uint64), np.arange(30000, dtype=np.uint64)])
    i = ref.canonicalize(np.vstack([hub, random_relation(rng, 2, 5000, 2000)]), 2)
    o = ref.canonicalize(np.vstack([[[0, 5], [0, 9]], random_relation(rng, 2, 3000, 2000)]), 2)
    s = spec(1, [I(1), O(1)])
    exp = ref.join(o, 2, i, 2, s)
    oc = al.relation_container(al.tuple_array(2, o, canonical=True))
    ic = al.make_container(al.tuple_array(2, i, canonical=True), None, 1)
    js = al.join_spec(1, oc, ic, al.column_map([al.operand.inner(1), al.operand.outer(1)]))
    out = al.tuple_array(2, np.zeros((len(exp), 2)))
    al.join_materialize(js, out)
    assert np.array_equal(out.data, exp)


def test_select_project_matches_reference(ref):
    rng = np.random.default_rng(21)
    a = random_relation(rng, 3, 2000, 6)
    proj = [O(2), O(0), K(42)]
    filt = [F(O(0), O(1), False), F(O(2), K(3), False)]
    got = al.select_project(al.relation_container(al.tuple_array(3, a)), al.column_map(proj), filt).data
    assert np.array_equal(got, ref.select_project(a, 3, proj, filt))
    with pytest.raises(al.logic_error):
        al.select_project(al.relation_container(al.tuple_array(3, a)), al.column_map([I(0)]))


# ---- merge_sorted / difference (ra_test.cpp:190-297) ------------------------

def test_merge_known_answers():
    f = al.tuple_array(1, [1, 3], canonical=True)
    d = al.tuple_array(1, [2, 4], canonical=True)
    assert al.merge_sorted(f, d).data.reshape(-1).tolist() == [1, 2, 3, 4]
    f2 = al.tuple_array(2, [1, 2, 3, 3], canonical=True)
    d2 = al.tuple_array(2, [2, 2, 3, 4], canonical=True)
    assert al.merge_sorted(f2, d2).data.reshape(-1).tolist() == [1, 2, 2, 2, 3, 3, 3, 4]
    assert al.merge_sorted(f, al.tuple_array(1, [], canonical=True)).data.reshape(-1).tolist() == [1, 3]
    with pytest.raises(al.logic_error):
        al.merge_sorted(f, d, buffer_rows=3)
    with pytest.raises(al.logic_error):
        al.merge_sorted(f, al.tuple_array(1, [3], canonical=True))
    with pytest.raises(al.logic_error):
        al.merge_sorted(f, al.tuple_array(1, [2], canonical=False))


def test_difference_known_answers():
    n = al.tuple_array(1, [1, 2, 3], canonical=True)
    f = al.tuple_array(1, [1, 4], canonical=True)
    assert al.difference(n, f).data.reshape(-1).tolist() == [2, 3]
    assert al.difference(n, n).count() == 0
    with pytest.raises(al.logic_error):
        al.difference(al.tuple_array(1, [1], canonical=False), f)


@pytest.mark.parametrize("nf,nd,domain,high", [
    (0, 100, 1000, 0), (100, 0, 1000, 0), (5000, 3000, 100000, 0), (300000, 70000, 1 << 40, 0),
    (2000, 1500, 1 << 62, U64MAX - (1 << 62) - 5),
])
def test_merge_and_difference_match_reference(ref, nf, nd, domain, high):
    rng = np.random.default_rng(nf + 3 * nd)
    pool = ref.canonicalize(random_relation(rng, 2, nf + nd + 100, domain, high), 2)
    rng.shuffle(pool)
    f = ref.canonicalize(pool[:nf], 2) if nf else pool[:0]
    d = ref.canonicalize(pool[nf: nf + nd], 2) if nd else pool[:0]
    got = al.merge_sorted(al.tuple_array(2, f, canonical=True), al.tuple_array(2, d, canonical=True)).data
    assert np.array_equal(got, ref.merge_sorted(f, d, 2))
    # difference of an overlapping new set
    new = ref.canonicalize(np.vstack([d, f[: nf // 2]]), 2) if nf + nd else pool[:0]
    gd = al.difference(al.tuple_array(2, new, canonical=True), al.tuple_array(2, f, canonical=True)).data
    assert np.array_equal(gd, ref.difference(new, f, 2))
