"""CPU: the reference fact-file / TSV functions (oracle/_ref, io.hpp) pinned
to the known answers of the reference's own tests/io_test.cpp, before they
serve as the checker of the device TSV path (tests/test_gpu_tsv.py)."""
import pytest


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_bytes(text.encode() if isinstance(text, str) else text)
    return p


def test_collapses_duplicate_lines(ref, tmp_path):  # io_test.cpp:41-47
    rc, rows = ref.read_facts(write(tmp_path, "f.tsv", "1 2\n2 3\n1 2\n"), 2)
    assert rc == 0 and rows.reshape(-1).tolist() == [1, 2, 2, 3]


def test_tabs_spaces_comments_blanks(ref, tmp_path):  # io_test.cpp:49-59
    rc, rows = ref.read_facts(write(tmp_path, "f.tsv", "# header comment\n1\t2\n\n  3   4 \n\t5\t6\r\n"), 2)
    assert rc == 0 and len(rows) == 3


def test_wrong_column_count_names_the_line(ref, tmp_path):  # io_test.cpp:61-71
    rc, msg = ref.read_facts(write(tmp_path, "f.tsv", "1 2\n3 4 5\n"), 2)
    assert rc == 4 and ":2:" in msg and "got 3" in msg


@pytest.mark.parametrize("text", ["99999999999999999999 1\n", "x 1\n", "1 18446744073709551615\n"])
def test_overflow_and_garbage(ref, tmp_path, text):  # io_test.cpp:73-81
    rc, _ = ref.read_facts(write(tmp_path, "a", text), 2)
    assert rc == 4


def test_missing_file(ref, tmp_path):
    rc, msg = ref.read_facts(tmp_path / "missing.tsv", 2)
    assert rc == 4 and "cannot open" in msg


def test_single_row_bytes_and_dump(ref):  # io_test.cpp:98-107, 171-174
    assert ref.to_tsv([1, 2], 2) == b"1\t2\n"
    assert ref.to_tsv([3, 4, 1, 2], 2) == b"1\t2\n3\t4\n"
    assert ref.to_tsv([], 2) == b""


def test_dictionary_round_trip(ref, tmp_path):  # io_test.cpp:140-152
    assert ref.dict_roundtrip(write(tmp_path, "f.tsv", "alice bob\nbob carol\nalice bob\n"), 2) == \
        b"alice\tbob\nbob\tcarol\n"


def test_file_scan(ref, tmp_path):  # io_test.cpp:163-169
    assert ref.file_is_all_integers(write(tmp_path, "a", "1 2\n# x\n3 4\n"))
    assert not ref.file_is_all_integers(write(tmp_path, "b", "1 x\n"))
    assert not ref.file_is_all_integers(write(tmp_path, "c", "18446744073709551615\n"))
