"""Built-in programs (builtins.hpp:13-41) as compiled rule plans.

The planner is outside the hot path; its OUTPUT is the
data contract the device engine consumes.  These are the plans
plan_program() produces for the three built-in programs (SURVEY §3.2,
tests/plan_test.cpp:21-136); tests/test_builtins.py checks them field by
field against the reference planner compiled in oracle/_ref.

Notation: operands "o<c>" = outer column c, "i<c>" = inner column c,
"c<v>" = constant v; filters are (lhs, rhs, require_equal).
"""
from __future__ import annotations

from dataclasses import dataclass, field

from . import abi as A


@dataclass
class Step:
    inner: str
    inner_perm: list
    jcc: int
    proj: list
    filters: list = field(default_factory=list)


@dataclass
class Variant:
    source: str
    version: str  # "full" | "delta"
    perm: list
    steps: list = field(default_factory=list)
    sel: list = field(default_factory=list)
    sel_filters: list = field(default_factory=list)


@dataclass
class Rule:
    index: int
    head: str
    recursive: bool
    variants: list


@dataclass
class Program:
    """Relations in id order: EDB declarations first (program order), then
    IDB relations in program::idb_relations() order (program.hpp:79-86)."""

    name: str
    relations: list  # [(name, arity, is_edb)]
    rules: list

    def rid(self, name: str) -> int:
        for i, (n, _, _) in enumerate(self.relations):
            if n == name:
                return i
        raise KeyError(name)

    def arity(self, name: str) -> int:
        return self.relations[self.rid(name)][1]

    @property
    def edbs(self):
        return [n for n, _, e in self.relations if e]

    @property
    def idbs(self):
        return [n for n, _, e in self.relations if not e]


def _operand(s: str) -> A.gd_operand:
    kind = {"o": A.GD_OUTER_COL, "i": A.GD_INNER_COL, "c": A.GD_CONSTANT}[s[0]]
    v = int(s[1:])
    if kind == A.GD_CONSTANT:
        return A.gd_operand(kind, 0, v)
    return A.gd_operand(kind, v, 0)


def _filter(f) -> A.gd_filter:
    lhs, rhs, eq = f
    return A.gd_filter(_operand(lhs), _operand(rhs), int(bool(eq)), 0)


def to_blob(prog: Program) -> list:
    """Compiles the plan dataclasses into gd_rule_plan structs."""
    out = []
    for r in prog.rules:
        p = A.gd_rule_plan()
        p.rule_index = r.index
        p.head_rel = prog.rid(r.head)
        p.head_arity = prog.arity(r.head)
        p.recursive = int(r.recursive)
        p.nvariants = len(r.variants)
        for vi, v in enumerate(r.variants):
            gv = p.variants[vi]
            gv.src_rel = prog.rid(v.source)
            gv.src_version = A.GD_DELTA if v.version == "delta" else A.GD_FULL
            for c, x in enumerate(v.perm):
                gv.src_perm[c] = x
            gv.nsteps = len(v.steps)
            for si, s in enumerate(v.steps):
                gs = gv.steps[si]
                gs.inner_rel = prog.rid(s.inner)
                gs.join_column_count = s.jcc
                for c, x in enumerate(s.inner_perm):
                    gs.inner_perm[c] = x
                gs.proj_arity = len(s.proj)
                for c, o in enumerate(s.proj):
                    gs.proj[c] = _operand(o)
                gs.nfilters = len(s.filters)
                for c, f in enumerate(s.filters):
                    gs.filters[c] = _filter(f)
            gv.sel_arity = len(v.sel)
            for c, o in enumerate(v.sel):
                gv.sel_proj[c] = _operand(o)
            gv.nsel_filters = len(v.sel_filters)
            for c, f in enumerate(v.sel_filters):
                gv.sel_filters[c] = _filter(f)
        out.append(p)
    return out


ID = [0, 1]
SW = [1, 0]

# Reach(from, to) :- Edge(from, to).  Reach(from, to) :- Edge(from, mid), Reach(mid, to).
REACH = Program(
    "reach",
    [("Edge", 2, True), ("Reach", 2, False)],
    [
        Rule(0, "Reach", False, [Variant("Edge", "full", ID, sel=["o0", "o1"])]),
        Rule(1, "Reach", True, [Variant("Reach", "delta", ID, steps=[Step("Edge", SW, 1, ["i1", "o1"])])]),
    ],
)

# SG(x, y) :- Edge(p, x), Edge(p, y), x != y.
# SG(x, y) :- Edge(a, x), SG(a, b), Edge(b, y).
SG = Program(
    "sg",
    [("Edge", 2, True), ("SG", 2, False)],
    [
        Rule(0, "SG", False, [Variant("Edge", "full", ID, steps=[
            Step("Edge", ID, 1, ["o1", "i1"], [("o1", "i1", False)])])]),
        Rule(1, "SG", True, [Variant("SG", "delta", ID, steps=[
            Step("Edge", ID, 1, ["o1", "i1"]),
            Step("Edge", ID, 1, ["o1", "i1"])])]),
    ],
)

VF, MA, VA = "ValueFlow", "MemoryAlias", "ValueAlias"
CSPA = Program(
    "cspa",
    [("assign", 2, True), ("dereference", 2, True), (VF, 2, False), (MA, 2, False), (VA, 2, False)],
    [
        Rule(0, VF, False, [Variant("assign", "full", ID, sel=["o0", "o1"])]),
        Rule(1, VF, False, [Variant("assign", "full", ID, sel=["o0", "o0"])]),
        Rule(2, VF, False, [Variant("assign", "full", ID, sel=["o1", "o1"])]),
        Rule(3, MA, False, [Variant("assign", "full", ID, sel=["o1", "o1"])]),
        Rule(4, MA, False, [Variant("assign", "full", ID, sel=["o0", "o0"])]),
        Rule(5, VF, True, [
            Variant(VF, "delta", SW, steps=[Step(VF, ID, 1, ["o1", "i1"])]),
            Variant(VF, "delta", ID, steps=[Step(VF, SW, 1, ["i1", "o1"])]),
        ]),
        Rule(6, VA, True, [
            Variant(VF, "delta", ID, steps=[Step(VF, ID, 1, ["o1", "i1"])]),
            Variant(VF, "delta", ID, steps=[Step(VF, ID, 1, ["i1", "o1"])]),
        ]),
        Rule(7, VF, True, [Variant(MA, "delta", ID, steps=[Step("assign", SW, 1, ["i1", "o1"])])]),
        Rule(8, MA, True, [Variant(VA, "delta", ID, steps=[
            Step("dereference", ID, 1, ["o1", "i1"]),
            Step("dereference", ID, 1, ["o1", "i1"])])]),
        Rule(9, VA, True, [
            Variant(VF, "delta", ID, steps=[Step(MA, ID, 1, ["i1", "o1"]), Step(VF, ID, 1, ["o1", "i1"])]),
            Variant(MA, "delta", ID, steps=[Step(VF, ID, 1, ["o1", "i1"]), Step(VF, ID, 1, ["o1", "i1"])]),
            Variant(VF, "delta", ID, steps=[Step(MA, SW, 1, ["i1", "o1"]), Step(VF, ID, 1, ["i1", "o1"])]),
        ]),
    ],
)

BUILTINS = {"reach": REACH, "sg": SG, "cspa": CSPA}


def builtin_program(name: str) -> Program:
    """builtin_program (builtins.hpp:55-60)."""
    try:
        return BUILTINS[name]
    except KeyError:
        from .arraylog import usage_error

        raise usage_error(f"unknown builtin program '{name}' (expected reach, sg, or cspa)") from None
