"""Fact ingestion and TSV output on the device (csrc/tsv.cu) against the
reference io.hpp (oracle/_ref): parsed rows, error statuses and messages,
and TSV bytes identical; io_test.cpp's cases restated plus messy random
files, 20-digit values, and engine-level load/write."""
import numpy as np
import pytest

from paper_2311_02206_b200 import arraylog as al
from tests.helpers import U64MAX

pytestmark = pytest.mark.gpu


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_bytes(text.encode() if isinstance(text, str) else text)
    return p


def dev_read(path, arity, **kw):
    try:
        return 0, al.read_facts(path, arity, **kw).data
    except al.load_error as e:
        return 4, str(e)


CASES = [
    ("1 2\n2 3\n1 2\n", 2), ("# header comment\n1\t2\n\n  3   4 \n\t5\t6\r\n", 2), ("1 2\n3 4 5\n", 2),
    ("99999999999999999999 1\n", 2), ("x 1\n", 2), ("1 18446744073709551615\n", 2), ("", 2), ("\n\n#c\n", 2),
    ("7 8", 2), ("1 2\r\n3 4\r\n", 2), ("1 2\r\r\n", 2), ("18446744073709551614 0\n", 2), ("00012 0004\n", 2),
    ("1\t\t2\t\n", 2), ("1 2 3\n4 5 6\n1 2 3\n", 3), ("5\n5\n3\n", 1), ("1 2\n1 -2\n", 2), ("1 2\n\n1\n", 2),
    ("12a 1\n", 2), ("1 2\n# 1 2 3\n 3 4\n", 2),
]


@pytest.mark.parametrize("i", range(len(CASES)))
def test_read_facts_cases(ref, tmp_path, i):
    text, arity = CASES[i]
    p = write(tmp_path, "f.tsv", text)
    got, exp = dev_read(p, arity), ref.read_facts(p, arity)
    assert got[0] == exp[0], (got, exp)
    if exp[0] == 0:
        assert np.array_equal(got[1].reshape(-1), exp[1].reshape(-1))
    else:
        assert got[1] == exp[1]


def test_missing_file_is_load_error(tmp_path):
    with pytest.raises(al.load_error):
        al.read_facts(tmp_path / "missing.tsv", 2)


@pytest.mark.parametrize("seed", [211, 5, 77])
def test_random_messy_files(ref, tmp_path, seed):
    """io_test.cpp:83-96 (10000 random lines) plus random separators,
    comments, blank and CR lines, and the odd bad line."""
    rng = np.random.default_rng(seed)
    lines = []
    for _ in range(10000):
        k = rng.integers(0, 20)
        a, b = rng.integers(0, 501, size=2)
        sep = ["\t", " ", "  ", " \t "][rng.integers(0, 4)]
        if k == 0:
            lines.append("# comment")
        elif k == 1:
            lines.append("  ")
        elif k == 2:
            lines.append(f"{a}{sep}{b}\r")
        else:
            lines.append(f"{' ' * (k % 3)}{a}{sep}{b}")
    text = "\n".join(lines) + ("\n" if seed != 5 else "")
    p = write(tmp_path, "big.tsv", text)
    got, exp = dev_read(p, 2), ref.read_facts(p, 2)
    assert got[0] == exp[0] == 0 and np.array_equal(got[1], exp[1])
    bad = lines[:]
    bad[7777] = "1 2 3"
    bad[9000] = "zz 1"
    p2 = write(tmp_path, "bad.tsv", "\n".join(bad) + "\n")
    got, exp = dev_read(p2, 2), ref.read_facts(p2, 2)
    assert got == exp and ":7778:" in got[1]


@pytest.mark.parametrize("arity,n,hi", [(1, 5000, 1 << 64), (2, 20000, 1 << 64), (3, 3000, 1000), (5, 2000, 50)])
def test_to_tsv_bytes(ref, arity, n, hi):
    rng = np.random.default_rng(arity)
    v = rng.integers(0, hi - 1, size=(n, arity), dtype=np.uint64) if hi < (1 << 64) else \
        rng.integers(0, U64MAX - 1, size=(n, arity), dtype=np.uint64, endpoint=True)
    v[0, :] = U64MAX - 1
    v[1, :] = 0
    t = al.canonicalize(al.tuple_array(arity, v))
    assert al.to_tsv(t).encode() == ref.to_tsv(v, arity)


def test_write_relation_and_round_trip(ref, tmp_path):  # io_test.cpp:98-128
    t = al.canonicalize(al.tuple_array(2, [1, 2]))
    p = tmp_path / "out.tsv"
    al.write_relation(t, p)
    assert p.read_bytes() == b"1\t2\n"
    e = al.tuple_array(2, canonical=True)
    al.write_relation(e, tmp_path / "empty.tsv")
    assert (tmp_path / "empty.tsv").stat().st_size == 0
    with pytest.raises(al.logic_error):
        al.write_relation(al.tuple_array(2, [2, 1, 1, 0]), tmp_path / "x.tsv")
    rng = np.random.default_rng(223)
    for _ in range(10):
        r = al.canonicalize(al.tuple_array(3, rng.integers(0, 50, size=(200, 3), dtype=np.uint64)))
        al.write_relation(r, tmp_path / "rt.tsv")
        assert al.read_facts(tmp_path / "rt.tsv", 3) == r


def test_dictionary_mode(ref, tmp_path):  # io_test.cpp:130-161
    d = al.dictionary()
    assert (d.intern("apple"), d.intern("pear"), d.intern("apple"), d.size()) == (0, 1, 0, 2)
    assert d.symbol(1) == "pear"
    with pytest.raises(al.logic_error):
        d.symbol(2)
    p = write(tmp_path, "f.tsv", "alice bob\nbob carol\nalice bob\n")
    d = al.dictionary()
    t = al.read_facts(p, 2, d)
    assert t.count() == 2 and d.size() == 3
    out = tmp_path / "out.tsv"
    al.write_relation(t, out, d)
    assert out.read_bytes() == ref.dict_roundtrip(p, 2)
    d3 = al.dictionary()
    assert al.read_facts(write(tmp_path, "g.tsv", "7 hello\n"), 2, d3).data.reshape(-1).tolist() == [0, 1]


@pytest.mark.parametrize("text", ["1 2\n# x\n3 4\n", "1 x\n", "18446744073709551615\n", "", "1 2 3\n4\n",
                                  "1\r\n2 2\r\n", "-1\n"])
def test_file_is_all_integers(ref, tmp_path, text):
    p = write(tmp_path, "s.tsv", text)
    assert al.file_is_all_integers(p) == ref.file_is_all_integers(p)


def test_engine_tsv_c1(ref, tmp_path):
    """Reach of C1 loaded from a TSV file on the device and written as TSV:
    bytes equal the reference's write_relation of its own run."""
    import ctypes as C
    raw = np.zeros((10000, 2), dtype=np.uint64)
    assert ref.lib.ref_gen_tc_rand(C.c_uint64(10000), C.c_uint64(10000), C.c_uint64(1),
                                   raw.ctypes.data_as(C.c_void_p)) == 0
    p = write(tmp_path, "edge.tsv", "".join(f"{a}\t{b}\n" for a, b in raw))
    g = al.engine("reach")
    g.load_edb_tsv("Edge", p)
    g.run()
    r = ref.engine("reach")
    r.load_edb("Edge", raw)
    r.run()
    assert g.relation_tsv("Reach") == ref.to_tsv(r.relation("Reach"), 2)
    assert g.relation("Reach").count() == 198733


def test_engine_tsv_errors(tmp_path):
    g = al.engine("reach")
    with pytest.raises(al.load_error) as ei:
        g.load_edb_tsv("Edge", write(tmp_path, "e.tsv", "1 2\n3\n"))
    assert ":2: expected 2 columns, got 1" in str(ei.value)
    with pytest.raises(al.load_error):
        g.load_edb_tsv("Reach", write(tmp_path, "r.tsv", "1 2\n"))
