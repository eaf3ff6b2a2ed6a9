"""oracle/bindings.py — TEST INFRASTRUCTURE ONLY.

ctypes loaders for the two checkers:
  * PortOracle  — oracle/_build/libgdlog_oracle.so, the plain-C restatement
                  (oracle/gdlog_oracle.c);
  * RefOracle   — oracle/_ref/libarraylog_ref.so, the UNMODIFIED reference
                  engine compiled from /root/reference (oracle/Makefile).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_2311_02206_b200 import abi as A

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "_build" / "libgdlog_oracle.so"
REF_LIB = HERE / "_ref" / "libarraylog_ref.so"

P = C.c_void_p
PU64 = C.POINTER(C.c_uint64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(P) if a.size else None


def _rows(a, arity):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint64).reshape(-1, arity))
    return a


class OracleError(RuntimeError):
    def __init__(self, code, msg, phase=""):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg
        self.phase = phase


class _Base:
    prefix = ""

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._err(), self._phase())

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    # --- kernel-level (same argument order as gd_*) ---------------------
    def prefix_hash(self, rows, arity, ncols):
        r = _rows(rows, arity)
        out = np.zeros(len(r), dtype=np.uint64)
        self._check(self._fn("prefix_hash")(_ptr(r), C.c_uint64(len(r)), C.c_uint32(arity), C.c_uint32(ncols),
                                            _ptr(out)))
        return out

    def merge_sorted(self, full, delta, arity, buffer_rows=None, full_canonical=True, delta_canonical=True):
        f, d = _rows(full, arity), _rows(delta, arity)
        buf = len(f) + len(d) if buffer_rows is None else buffer_rows
        out = np.zeros((len(f) + len(d), arity), dtype=np.uint64)
        args = [_ptr(f), C.c_uint64(len(f)), C.c_int(full_canonical), _ptr(d), C.c_uint64(len(d)),
                C.c_int(delta_canonical), C.c_uint32(arity), C.c_uint64(buf)]
        if self.prefix == "ref_":
            args.append(C.c_uint32(1))
        self._check(self._fn("merge_sorted")(*args, _ptr(out)))
        return out

    def difference(self, new, full, arity, new_canonical=True, full_canonical=True):
        n, f = _rows(new, arity), _rows(full, arity)
        out = np.zeros((len(n), arity), dtype=np.uint64)
        m = C.c_uint64(0)
        args = [_ptr(n), C.c_uint64(len(n)), C.c_int(new_canonical), _ptr(f), C.c_uint64(len(f)),
                C.c_int(full_canonical), C.c_uint32(arity)]
        if self.prefix == "ref_":
            args.append(C.c_uint32(1))
        self._check(self._fn("difference")(*args, _ptr(out), C.byref(m)))
        return out[: m.value]

    def permute_columns(self, rows, arity, perm, canonical=True):
        r = _rows(rows, arity)
        p = np.asarray(perm, dtype=np.uint32)
        out = np.zeros((len(r), arity), dtype=np.uint64)
        m = C.c_uint64(0)
        self._check(self._fn("permute_columns")(_ptr(r), C.c_uint64(len(r)), C.c_uint32(arity),
                                                C.c_int(canonical), _ptr(p), C.c_uint32(len(p)), _ptr(out),
                                                C.byref(m)))
        return out[: m.value]

    def group_starts(self, rows, arity, prefix_len, canonical=True):
        r = _rows(rows, arity)
        out = np.zeros(max(len(r), 1), dtype=np.uint64)
        m = C.c_uint64(0)
        self._check(self._fn("group_starts")(_ptr(r), C.c_uint64(len(r)), C.c_uint32(arity),
                                             C.c_int(canonical), C.c_uint32(prefix_len), _ptr(out), C.byref(m)))
        return out[: m.value]

    def index_lookup(self, rows, arity, prefix_len, keys, load_factor=0.8, canonical=True, key_len=None):
        r = _rows(rows, arity)
        kl = prefix_len if key_len is None else key_len
        k = _rows(keys, kl) if len(keys) else np.zeros((0, kl), dtype=np.uint64)
        st = np.zeros(max(len(k), 1), dtype=np.uint64)
        ct = np.zeros(max(len(k), 1), dtype=np.uint64)
        sc, oc = C.c_uint64(0), C.c_uint64(0)
        self._check(self._fn("index_lookup")(_ptr(r), C.c_uint64(len(r)), C.c_uint32(arity), C.c_int(canonical),
                                             C.c_uint32(prefix_len), C.c_double(load_factor), _ptr(k),
                                             C.c_uint64(len(k)), C.c_uint32(kl), _ptr(st), _ptr(ct),
                                             C.byref(sc), C.byref(oc)))
        return st[: len(k)], ct[: len(k)], sc.value, oc.value

    def select_project(self, rows, arity, proj, filters=()):
        r = _rows(rows, arity)
        pa = (A.gd_operand * max(len(proj), 1))(*proj)
        fa = (A.gd_filter * max(len(filters), 1))(*filters)
        out = np.zeros((max(len(r), 1), len(proj)), dtype=np.uint64)
        m = C.c_uint64(0)
        self._check(self._fn("select_project")(_ptr(r), C.c_uint64(len(r)), C.c_uint32(arity), pa,
                                               C.c_uint32(len(proj)), fa, C.c_uint32(len(filters)), _ptr(out),
                                               C.byref(m)))
        return out[: m.value]


class PortOracle(_Base):
    """The plain-C restatement (oracle/gdlog_oracle.c)."""

    prefix = "or_"

    def __init__(self, path: Path | str = PORT_LIB):
        if not Path(path).exists():
            raise RuntimeError(f"{path} missing: run `make -C oracle port`")
        self.lib = C.CDLL(str(path))
        self.lib.or_last_error.restype = C.c_char_p
        self.lib.or_engine_create.restype = P
        self.lib.or_engine_create.argtypes = [C.c_uint32, P, P]
        for n in ("set_plans", "load_edb", "run", "relation_count", "relation_download", "delta_history",
                  "iter_log", "seed", "iterate"):
            getattr(self.lib, "or_engine_" + n).restype = C.c_int
        self.lib.or_engine_destroy.argtypes = [P]
        self.lib.or_engine_iterations.restype = C.c_uint64
        self.lib.or_engine_iterations.argtypes = [P]

    def _err(self):
        return self.lib.or_last_error().decode()

    def _phase(self):
        return ""

    def canonicalize(self, rows, arity):
        r = _rows(rows, arity)
        out = np.zeros((len(r), arity), dtype=np.uint64)
        m = C.c_uint64(0)
        self._check(self.lib.or_canonicalize(_ptr(r), C.c_uint64(len(r)), C.c_uint32(arity), _ptr(out),
                                             C.byref(m)))
        return out[: m.value]

    def join(self, outer, oa, inner, ia, spec, outer_canonical=True, inner_canonical=True, index_prefix=None,
             materialize=True, capacity=None):
        return _join(self, outer, oa, inner, ia, spec, outer_canonical, inner_canonical, index_prefix,
                     materialize, capacity, extra=())

    def run_engine(self, arities, is_edb, plans, edbs):
        """Runs the restated engine; edbs: {rel_id: rows}.  Returns
        (relations {id: rows}, history {id: list}, log {id: records}, iterations)."""
        ar = np.asarray(arities, dtype=np.uint32)
        ed = np.asarray(is_edb, dtype=np.uint32)
        e = self.lib.or_engine_create(C.c_uint32(len(ar)), _ptr(ar), _ptr(ed))
        try:
            pl = (A.gd_rule_plan * max(len(plans), 1))(*plans)
            self._check(self.lib.or_engine_set_plans(P(e), pl, C.c_uint32(len(plans))))
            for rid, rows in edbs.items():
                r = _rows(rows, int(ar[rid]))
                self._check(self.lib.or_engine_load_edb(P(e), C.c_uint32(rid), _ptr(r), C.c_uint64(len(r)),
                                                        C.c_int(0)))
            self._check(self.lib.or_engine_run(P(e)))
            rels, hist, logs = {}, {}, {}
            for rid in range(len(ar)):
                n = C.c_uint64(0)
                self._check(self.lib.or_engine_relation_count(P(e), C.c_uint32(rid), C.byref(n)))
                out = np.zeros((n.value, int(ar[rid])), dtype=np.uint64)
                self._check(self.lib.or_engine_relation_download(P(e), C.c_uint32(rid), _ptr(out),
                                                                 C.c_uint64(n.value)))
                rels[rid] = out
                ln = C.c_uint64(0)
                self.lib.or_engine_delta_history(P(e), C.c_uint32(rid), None, C.c_uint64(0), C.byref(ln))
                h = np.zeros(max(ln.value, 1), dtype=np.uint64)
                self.lib.or_engine_delta_history(P(e), C.c_uint32(rid), _ptr(h), C.c_uint64(ln.value),
                                                 C.byref(ln))
                hist[rid] = [int(x) for x in h[: ln.value]]
                self.lib.or_engine_iter_log(P(e), C.c_uint32(rid), None, C.c_uint64(0), C.byref(ln))
                recs = (A.gd_iter_record * max(ln.value, 1))()
                self.lib.or_engine_iter_log(P(e), C.c_uint32(rid), recs, C.c_uint64(ln.value), C.byref(ln))
                logs[rid] = [(r.delta_in, r.join, r.new_unique, r.delta_out, r.full_after)
                             for r in recs[: ln.value]]
            iters = self.lib.or_engine_iterations(P(e))
            return rels, hist, logs, iters
        finally:
            self.lib.or_engine_destroy(P(e))


def _join(self, outer, oa, inner, ia, spec, outer_canonical, inner_canonical, index_prefix, materialize,
          capacity, extra):
    o, i = _rows(outer, oa), _rows(inner, ia)
    ov = A.gd_container_view(_ptr(o), len(o), oa, int(outer_canonical), 0, 0, 0.8)
    ip = spec.join_column_count if index_prefix is None else index_prefix
    iv = A.gd_container_view(_ptr(i), len(i), ia, int(inner_canonical), ip, 0, 0.8)
    total = C.c_uint64(0)
    self._check(self._fn("join_count")(C.byref(ov), C.byref(iv), C.byref(spec), *extra, C.byref(total)))
    if not materialize:
        return total.value
    cap = total.value if capacity is None else capacity
    out = np.zeros((max(cap, 1), spec.proj_arity), dtype=np.uint64)
    self._check(self._fn("join_materialize")(C.byref(ov), C.byref(iv), C.byref(spec), *extra, _ptr(out),
                                             C.c_uint64(cap)))
    return out[:cap]


class RefOracle(_Base):
    """The reference engine itself (oracle/_ref/libarraylog_ref.so)."""

    prefix = "ref_"

    def __init__(self, path: Path | str = REF_LIB):
        if not Path(path).exists():
            raise RuntimeError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_last_error_phase.restype = C.c_char_p
        L.ref_engine_create.restype = P
        L.ref_engine_create.argtypes = [C.c_char_p, C.POINTER(A.gd_engine_config)]
        L.ref_engine_destroy.argtypes = [P]
        L.ref_engine_relation_name.restype = C.c_char_p
        L.ref_engine_relation_name.argtypes = [P, C.c_uint32]
        for n in ("num_relations", "relation_arity", "load_edb", "run", "relation_count", "relation_download",
                  "stats", "delta_history", "plans", "stats_tsv"):
            getattr(L, "ref_engine_" + n).restype = C.c_int
        L.ref_engine_num_relations.argtypes = [P]
        L.ref_engine_relation_arity.argtypes = [P, C.c_uint32]

    def _err(self):
        return self.lib.ref_last_error().decode()

    # ---- fact files / TSV (io.hpp) ----
    def read_facts(self, path, arity, use_dict=False):
        """(status, rows or error message) of the reference read_facts."""
        import numpy as np
        cap = max(1, Path(path).stat().st_size // 2 + 1) if Path(path).exists() else 1
        out = np.zeros((cap, arity), dtype=np.uint64)
        n = C.c_uint64()
        rc = self.lib.ref_read_facts(str(path).encode(), C.c_uint32(arity), C.c_int(int(use_dict)),
                                     out.ctypes.data_as(C.c_void_p), C.c_uint64(cap), C.byref(n))
        return (rc, out[: n.value]) if rc == 0 else (rc, self._err())

    def to_tsv(self, rows, arity) -> bytes:
        import numpy as np
        rows = np.ascontiguousarray(rows, dtype=np.uint64).reshape(-1, arity)
        cap = max(1, rows.shape[0] * arity * 21 + 16)
        buf = C.create_string_buffer(cap)
        n = C.c_uint64()
        rc = self.lib.ref_to_tsv(rows.ctypes.data_as(C.c_void_p), C.c_uint64(rows.shape[0]), C.c_uint32(arity), buf,
                                 C.c_uint64(cap), C.byref(n))
        assert rc == 0, self._err()
        return buf.raw[: n.value]

    def dict_roundtrip(self, path, arity) -> bytes:
        cap = Path(path).stat().st_size * 2 + 16
        buf = C.create_string_buffer(cap)
        n = C.c_uint64()
        rc = self.lib.ref_dict_roundtrip(str(path).encode(), C.c_uint32(arity), buf, C.c_uint64(cap), C.byref(n))
        assert rc == 0, self._err()
        return buf.raw[: n.value]

    def file_is_all_integers(self, path) -> bool:
        r = C.c_int()
        rc = self.lib.ref_file_is_all_integers(str(path).encode(), C.byref(r))
        assert rc == 0, self._err()
        return bool(r.value)

    def _phase(self):
        return self.lib.ref_last_error_phase().decode()

    def canonicalize(self, rows, arity, workers=1):
        r = _rows(rows, arity)
        out = np.zeros((len(r), arity), dtype=np.uint64)
        m = C.c_uint64(0)
        self._check(self.lib.ref_canonicalize(_ptr(r), C.c_uint64(len(r)), C.c_uint32(arity),
                                              C.c_uint32(workers), _ptr(out), C.byref(m)))
        return out[: m.value]

    def join(self, outer, oa, inner, ia, spec, outer_canonical=True, inner_canonical=True, index_prefix=None,
             materialize=True, capacity=None, workers=1, stride=0):
        return _join(self, outer, oa, inner, ia, spec, outer_canonical, inner_canonical, index_prefix,
                     materialize, capacity, extra=(C.c_uint32(workers), C.c_uint64(stride)))

    # --- engine ---------------------------------------------------------
    def engine(self, program: str, config: A.gd_engine_config | None = None):
        h = self.lib.ref_engine_create(program.encode(), C.byref(config) if config else None)
        if not h:
            raise OracleError(-1, self._err())
        return RefEngine(self, h)


class RefEngine:
    def __init__(self, o: RefOracle, h):
        self.o, self.h, self.L = o, P(h), o.lib
        n = self.L.ref_engine_num_relations(self.h)
        self.names = [self.L.ref_engine_relation_name(self.h, i).decode() for i in range(n)]
        self.arities = [self.L.ref_engine_relation_arity(self.h, i) for i in range(n)]

    def __del__(self):
        try:
            self.L.ref_engine_destroy(self.h)
        except Exception:
            pass

    def rid(self, name):
        return self.names.index(name)

    def load_edb(self, name, rows, canonical=False):
        rid = self.rid(name)
        r = _rows(rows, self.arities[rid])
        self.o._check(self.L.ref_engine_load_edb(self.h, C.c_uint32(rid), _ptr(r), C.c_uint64(len(r)),
                                                 C.c_int(canonical)))

    def run(self):
        self.o._check(self.L.ref_engine_run(self.h))

    def relation(self, name):
        rid = self.rid(name)
        n = C.c_uint64(0)
        self.o._check(self.L.ref_engine_relation_count(self.h, C.c_uint32(rid), C.byref(n)))
        out = np.zeros((n.value, self.arities[rid]), dtype=np.uint64)
        self.o._check(self.L.ref_engine_relation_download(self.h, C.c_uint32(rid), _ptr(out),
                                                          C.c_uint64(n.value)))
        return out

    def stats(self) -> A.gd_run_stats:
        s = A.gd_run_stats()
        self.o._check(self.L.ref_engine_stats(self.h, C.byref(s)))
        return s

    def stats_tsv(self) -> str:
        buf = C.create_string_buffer(1 << 20)
        self.o._check(self.L.ref_engine_stats_tsv(self.h, buf, C.c_uint64(1 << 20)))
        return buf.value.decode()

    def delta_history(self, name):
        rid = self.rid(name)
        ln = C.c_uint64(0)
        self.o._check(self.L.ref_engine_delta_history(self.h, C.c_uint32(rid), None, C.c_uint64(0),
                                                      C.byref(ln)))
        h = np.zeros(max(ln.value, 1), dtype=np.uint64)
        self.o._check(self.L.ref_engine_delta_history(self.h, C.c_uint32(rid), _ptr(h), C.c_uint64(ln.value),
                                                      C.byref(ln)))
        return [int(x) for x in h[: ln.value]]

    def plans(self):
        cap = 64
        arr = (A.gd_rule_plan * cap)()
        n = C.c_uint32(0)
        self.o._check(self.L.ref_engine_plans(self.h, arr, C.c_uint32(cap), C.byref(n)))
        return list(arr[: n.value])
