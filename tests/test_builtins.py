"""CPU: the built-in programs' plans shipped in builtins.py equal, field by
field, what the reference planner (plan_program, plan.hpp:407-413)
produces — the data contract of the device engine."""
import ctypes as C

import pytest

from paper_2311_02206_b200.builtins import BUILTINS, to_blob


def blob_bytes(p):
    return bytes(C.string_at(C.addressof(p), C.sizeof(p)))


@pytest.mark.parametrize("name", sorted(BUILTINS))
def test_builtin_plans_equal_reference_planner(ref, name):
    prog = BUILTINS[name]
    e = ref.engine(name)
    assert e.names == [n for n, _, _ in prog.relations]
    assert e.arities == [a for _, a, _ in prog.relations]
    ours = to_blob(prog)
    theirs = e.plans()
    assert len(ours) == len(theirs)
    for a, b in zip(ours, theirs):
        assert blob_bytes(a) == blob_bytes(b), f"rule {a.rule_index}"
