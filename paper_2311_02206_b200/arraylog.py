"""Python mirror of the reference `arraylog` C++ API for the fixpoint hot path.

Names, argument meanings and error behaviour follow
/root/reference/proj/include/arraylog (cited per item); every call runs
the sm_100a kernels of libgdlog_b200.so through the C-ABI
(include/gdlog_b200.h).  There is no CPU fallback: without a B200 the
first device call raises cuda_error.

Rows are numpy uint64 arrays of shape (count, arity) inside `tuple_array`
(tuple_array.hpp:19-51).  `workers` / `stride_rows` arguments are accepted
for signature parity and ignored (results never depend on them).
"""
from __future__ import annotations

import contextlib
import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import abi as A
from .builtins import Program, builtin_program, to_blob

K_EMPTY_SLOT = (1 << 64) - 1  # kEmptySlot, types.hpp:16


# ---------------------------------------------------------------------------
# Exceptions (types.hpp:19-72)

class logic_error(RuntimeError):
    """std::logic_error: precondition violations / internal faults."""


class config_error(RuntimeError):
    pass


class usage_error(RuntimeError):
    pass


class load_error(RuntimeError):
    pass


class plan_error(RuntimeError):
    pass


class budget_error(RuntimeError):
    def __init__(self, phase: str, msg: str):
        super().__init__(msg)
        self._phase = phase

    def phase(self) -> str:
        return self._phase


class cuda_error(RuntimeError):
    """CUDA failure (no device, launch error).  No reference equivalent."""


class unsupported_error(RuntimeError):
    """A shape the device encoding cannot hold."""


_ERRORS = {
    A.GD_ERR_LOGIC: logic_error,
    A.GD_ERR_CONFIG: config_error,
    A.GD_ERR_USAGE: usage_error,
    A.GD_ERR_LOAD: load_error,
    A.GD_ERR_PLAN: plan_error,
    A.GD_ERR_CUDA: cuda_error,
    A.GD_ERR_UNSUPPORTED: unsupported_error,
    A.GD_ERR_INVALID_ARG: logic_error,
    A.GD_ERR_NCCL: cuda_error,
}


# ---------------------------------------------------------------------------
# Fact files and TSV output (io.hpp:17-170).  Numeric files are parsed and
# formatted on the device (tsv.cu); the dictionary mode interns tokens here,
# on the host, exactly as io.hpp's dictionary does (first-appearance ids).

class dictionary:
    """Symbol table, tokens -> dense ids in first-appearance order (io.hpp:19-41)."""

    def __init__(self):
        self._fwd: dict[str, int] = {}
        self._rev: list[str] = []

    def intern(self, token: str) -> int:
        i = self._fwd.get(token)
        if i is None:
            i = len(self._rev)
            self._fwd[token] = i
            self._rev.append(token)
        return i

    def symbol(self, i: int) -> str:
        if i < 0 or i >= len(self._rev):
            raise logic_error("dictionary: id out of range")
        return self._rev[i]

    def size(self) -> int:
        return len(self._rev)


def _read_bytes(path) -> bytes:
    try:
        with open(path, "rb") as f:
            return f.read()
    except OSError:
        raise load_error(f"cannot open fact file '{path}'") from None


def _dict_rows(text: bytes, arity: int, d: dictionary, name: str) -> np.ndarray:
    """read_facts with a dictionary (io.hpp:80-99): same line rules, tokens interned."""
    vals = []
    for ln, raw in enumerate(text.decode().split("\n") if text else [], 1):
        line = raw[:-1] if raw.endswith("\r") else raw
        stripped = line.strip(" \t")
        if not stripped or stripped[0] == "#":
            continue
        cols = [t for t in line.replace("\t", " ").split(" ") if t]
        if len(cols) != arity:
            raise load_error(f"{name}:{ln}: expected {arity} columns, got {len(cols)}")
        vals.extend(d.intern(t) for t in cols)
    return np.asarray(vals, dtype=np.uint64).reshape(-1, arity)


def read_facts(path, arity: int, dict_: dictionary | None = None, workers: int = 1,
               ctx: Context | None = None) -> tuple_array:
    """read_facts (io.hpp:64-114): canonical rows of a fact file.  Numeric
    files are parsed on the device; with a dictionary, tokens are interned on
    the host and the rows canonicalized on the device."""
    if arity <= 0:
        raise load_error("read_facts: arity must be positive")
    text = _read_bytes(path)
    ctx = ctx or default_context()
    if dict_ is not None:
        return canonicalize(tuple_array(arity, _dict_rows(text, arity, dict_, str(path))), ctx=ctx)
    cap = text.count(b"\n") + 1
    out = np.empty((cap, arity), dtype=np.uint64)
    n = A.u64()
    ctx.check(ctx.lib.gd_parse_facts(ctx.h, str(path).encode(), text, len(text), arity, _ptr(out), cap,
                                     C.byref(n)))
    return tuple_array(arity, out[: n.value], canonical=True)


def file_is_all_integers(path, ctx: Context | None = None) -> bool:
    """file_is_all_integers (io.hpp:145-170)."""
    text = _read_bytes(path)
    ctx = ctx or default_context()
    r = C.c_int()
    ctx.check(ctx.lib.gd_facts_all_integers(ctx.h, text, len(text), C.byref(r)))
    return bool(r.value)


def to_tsv(rel, dict_: dictionary | None = None, ctx: Context | None = None) -> str:
    """to_tsv: of a run_stats (stats.hpp:50-64), or of a relation (io.hpp:118-133):
    tab-separated rows, decimal or decoded tokens."""
    if not isinstance(rel, tuple_array):
        return _stats_to_tsv(rel)
    if dict_ is not None:
        return "".join("\t".join(dict_.symbol(int(v)) for v in r) + "\n" for r in rel.data)
    ctx = ctx or default_context()
    d = np.ascontiguousarray(rel.data)
    n = A.u64()
    ctx.check(ctx.lib.gd_rows_to_tsv(ctx.h, _ptr(d), rel.count(), rel.arity, None, 0, C.byref(n)))
    buf = C.create_string_buffer(max(n.value, 1))
    ctx.check(ctx.lib.gd_rows_to_tsv(ctx.h, _ptr(d), rel.count(), rel.arity, buf, n.value, C.byref(n)))
    return buf.raw[: n.value].decode()


def write_relation(rel: tuple_array, path, dict_: dictionary | None = None, ctx: Context | None = None):
    """write_relation (io.hpp:135-143): canonical relations only."""
    if not rel.canonical:
        raise logic_error("write_relation: relation must be canonical")
    text = to_tsv(rel, dict_, ctx)
    try:
        with open(path, "wb") as f:
            f.write(text.encode())
    except OSError:
        raise load_error(f"cannot open '{path}' for writing") from None


# ---------------------------------------------------------------------------
# Device context

# Diagnostics scripts (scripts/*.sh) select device knobs with these
# environment variables; the Python layer turns them into the context's
# gd_device_config at creation (the library itself reads no environment).
_ENV_KNOBS = {
    "GD_LOOP": ("resident_loop", int),
    "GD_LOOP_MODE": ("loop_mode", lambda v: {"graph": A.GD_LOOP_GRAPH, "eager": A.GD_LOOP_EAGER,
                                              "batch": A.GD_LOOP_BATCH}[v]),
    "GD_LOOP_BATCH": ("loop_batch", int),
    "GD_LOOP_TINY": ("min_capacities", int),
    "GD_LOOP_SPLIT": ("split_insert", int),
    "GD_DENSE": ("dense_inner", int),
    "GD_TAB_GROWTH": ("index_growth", int),
    "GD_INSERT_WAVES": ("insert_waves", int),
    "GD_REHASH_CAS": ("rehash_cas_only", int),
    "GD_ZONE_SLOTS": ("zone_slots", int),
    "GD_PART_LOOP": ("partition_loop", int),
    "GD_HASH_DEDUP": ("hash_dedup", int),
    "GD_DEDUP_L2_SLOTS": ("dedup_part_slots", int),
    "GD_DEDUP_SPLIT": ("dedup_split", int),
    "GD_HOST_UNPACK": ("host_unpack", int),
    "GD_DL_DIRECT_FRAC": ("download_direct_frac", float),
    "GD_DL_CHUNK_ROWS": ("download_chunk_rows", int),
    "GD_SORT_ITEMS": ("sort_items", int),
    "GD_WARP_EXPAND": ("warp_expand", int),
    "GD_HEAVY_ROWS": ("heavy_rows", int),
    "GD_SORT_DIGIT_BITS": ("sort_digit_bits", int),
    "GD_SORT_PIPE": ("sort_pipeline", int),
    "GD_SORT_PIPE_MIN": ("sort_pipeline_min_keys", int),
    "GD_TEMP_LIMIT_ROWS": ("temp_limit_rows", int),
    "GD_INSERT_SLOTS": ("insert_slots", int),
    "GD_L2_FETCH": ("l2_fetch_bytes", int),
    "GD_INSERT_PIPE": ("insert_pipeline", int),
    "GD_INSERT_PER": ("insert_per_thread", int),
    "GD_SORT_BALLOT": ("sort_ballot", int),
    "GD_SORT_MIN_CTAS": ("sort_min_ctas", int),
    "GD_DL_DELTA": ("download_delta", int),
    "GD_INDEX_LOAD_PCT": ("index_load_pct", int),
    "GD_DL_PIPELINE": ("download_pipeline", int),
    "GD_DL_PIPELINE_MIN": ("download_pipeline_min_rows", int),
    "GD_GATE_IN_INSERT": ("gate_in_insert", int),
    "GD_PDL": ("pdl", int),
    "GD_COUNT_AHEAD": ("count_ahead", int),
    "GD_CHAIN_CHUNK_ROWS": ("chain_chunk_rows", int),
    "GD_LOG_GROWTH": ("log_growth", int),
    "GD_DL_OVERLAP": ("download_overlap_pack", int),
    "GD_XP_PER": ("expand_keys_per_lane", int),
    "GD_WARP_APPEND": ("warp_append", int),
    "GD_PRECOUNT": ("precount", int),
    "GD_COUNT_CTAS": ("count_ctas_per_sm", int),
    "GD_PART_EXCHANGE": ("partition_exchange", lambda v: {"peer": 0, "nccl": 1}[v]),
}


def env_device_config() -> dict:
    """gd_device_config fields selected by GD_* environment variables."""
    out = {}
    for k, (field, conv) in _ENV_KNOBS.items():
        v = os.environ.get(k)
        if v is not None and v != "":
            out[field] = conv(v)
    tr = ((1 if os.environ.get("GD_LOOP_TRACE") == "1" else 0) | (2 if os.environ.get("GD_DL_TRACE") == "1" else 0)
          | (4 if os.environ.get("GD_SORT_TRACE") == "1" else 0))
    if tr:
        out["trace"] = tr
    return out


class Context:
    """Owns a gd_ctx (device + stream).  One host thread per context.

    `config` sets fields of the context's gd_device_config (defaults from
    gd_device_config_default, then GD_* diagnostics variables, then this)."""

    def __init__(self, device: int = 0, stream: int | None = None, config: dict | None = None):
        self.lib = A.load_library()
        h = C.c_void_p()
        rc = self.lib.gd_ctx_create(device, C.c_void_p(stream) if stream else None, C.byref(h))
        if rc != A.GD_OK:
            msg = self.lib.gd_last_error(None).decode()
            raise _ERRORS.get(rc, cuda_error)(msg)
        self.h = h
        kv = env_device_config()
        kv.update(config or {})
        if kv:
            self.set_config(**kv)

    @property
    def device_config(self) -> dict:
        c = A.gd_device_config()
        self.check(self.lib.gd_ctx_get_device_config(self.h, C.byref(c)))
        return {f: getattr(c, f) for f, _ in A.gd_device_config._fields_}

    def set_config(self, **fields):
        """Sets gd_device_config fields (GD_ERR_CONFIG -> config_error)."""
        c = A.gd_device_config()
        self.check(self.lib.gd_ctx_get_device_config(self.h, C.byref(c)))
        for f, v in fields.items():
            if f not in {n for n, _ in A.gd_device_config._fields_} or f == "size":
                raise config_error(f"unknown device config field '{f}'")
            setattr(c, f, v)
        self.check(self.lib.gd_ctx_set_device_config(self.h, C.byref(c)))

    @contextlib.contextmanager
    def configured(self, **fields):
        """Temporarily sets device config fields (tests select modes)."""
        old = self.device_config
        self.set_config(**fields)
        try:
            yield self
        finally:
            old.pop("size")
            self.set_config(**old)

    def check(self, rc: int):
        if rc == A.GD_OK:
            return
        msg = self.lib.gd_last_error(self.h).decode()
        if rc == A.GD_ERR_BUDGET:
            raise budget_error(self.lib.gd_last_error_phase(self.h).decode(), msg)
        raise _ERRORS.get(rc, logic_error)(msg)

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.gd_ctx_kernel_launches(self.h))

    def synchronize(self):
        self.check(self.lib.gd_ctx_synchronize(self.h))

    def trim(self):
        """Returns cached free device blocks to the driver (gd_ctx_trim)."""
        self.check(self.lib.gd_ctx_trim(self.h))

    def set_profiling(self, on: bool):
        self.check(self.lib.gd_ctx_set_profiling(self.h, int(on)))

    def profile(self) -> dict:
        """{kernel class: (ms, launches, algorithmic bytes)} since reset."""
        n = len(A.KCLASSES)
        ms = (C.c_double * n)()
        la = (A.u64 * n)()
        by = (A.u64 * n)()
        self.check(self.lib.gd_ctx_profile_read(self.h, ms, la, by))
        return {k: (ms[i], la[i], by[i]) for i, k in enumerate(A.KCLASSES)}

    def profile_reset(self):
        self.check(self.lib.gd_ctx_profile_reset(self.h))

    def transfer_bytes(self) -> tuple[int, int]:
        """(host->device, device->host) bytes copied by this context."""
        h, d = A.u64(), A.u64()
        self.check(self.lib.gd_ctx_transfer_bytes(self.h, C.byref(h), C.byref(d)))
        return int(h.value), int(d.value)

    def host_counters(self) -> dict:
        a, s = C.c_double(), C.c_double()
        na, ns = A.u64(), A.u64()
        self.check(self.lib.gd_ctx_host_counters(self.h, C.byref(a), C.byref(na), C.byref(s), C.byref(ns)))
        return {"alloc_s": a.value, "allocs": na.value, "sync_s": s.value, "syncs": ns.value}

    def close(self):
        if getattr(self, "h", None):
            self.lib.gd_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a.size else None


# ---------------------------------------------------------------------------
# tuple_array (tuple_array.hpp:19-51)

class tuple_array:
    def __init__(self, arity: int, data=None, canonical: bool = False):
        if arity <= 0:
            raise logic_error("tuple_array: arity must be positive")
        self.arity = int(arity)
        self.canonical = bool(canonical)
        if data is None:
            self.data = np.zeros((0, arity), dtype=np.uint64)
        else:
            flat = np.asarray(data, dtype=np.uint64).reshape(-1)
            if flat.size % arity:
                raise logic_error("tuple_array: data length must be count * arity")
            self.data = np.ascontiguousarray(flat.reshape(-1, arity))

    def count(self) -> int:
        return int(self.data.shape[0])

    def row(self, i: int):
        return self.data[i]

    def push_row(self, r):
        if len(r) != self.arity:
            raise logic_error("tuple_array: row width mismatch")
        self.data = np.vstack([self.data, np.asarray(r, dtype=np.uint64).reshape(1, -1)])
        self.canonical = False

    def byte_size(self) -> int:
        return self.data.size * 8

    def rows(self):
        return [tuple(int(x) for x in r) for r in self.data]

    def __eq__(self, o):
        return (isinstance(o, tuple_array) and self.arity == o.arity and self.canonical == o.canonical
                and np.array_equal(self.data, o.data))

    def __repr__(self):
        return f"tuple_array(arity={self.arity}, count={self.count()}, canonical={self.canonical})"


def canonicalize(raw: tuple_array, workers: int = 1, ctx: Context | None = None) -> tuple_array:
    """canonicalize (tuple_array.hpp:73-133): device radix sort + unique."""
    ctx = ctx or default_context()
    n = raw.count()
    if n == 0 or raw.canonical:
        return tuple_array(raw.arity, raw.data.copy(), canonical=True)
    out = np.zeros_like(raw.data)
    m = C.c_uint64(0)
    ctx.check(ctx.lib.gd_canonicalize(ctx.h, _ptr(raw.data), n, raw.arity, _ptr(out), C.byref(m)))
    return tuple_array(raw.arity, out[: m.value], canonical=True)


def permute_columns(rel: tuple_array, perm, workers: int = 1, ctx: Context | None = None) -> tuple_array:
    """permute_columns (ra.hpp:426-454)."""
    ctx = ctx or default_context()
    p = np.asarray(perm, dtype=np.uint32)
    out = np.zeros_like(rel.data)
    m = C.c_uint64(0)
    ctx.check(ctx.lib.gd_permute_columns(ctx.h, _ptr(rel.data), rel.count(), rel.arity, int(rel.canonical),
                                         _ptr(p), len(p), _ptr(out), C.byref(m)))
    return tuple_array(rel.arity, out[: m.value], canonical=True)


def prefix_hash(rows, ncols: int | None = None, ctx: Context | None = None) -> np.ndarray:
    """slot_key / prefix_hash of each row's first ncols columns (hash.hpp:28-60)."""
    ctx = ctx or default_context()
    r = np.ascontiguousarray(np.atleast_2d(np.asarray(rows, dtype=np.uint64)))
    arity = r.shape[1]
    ncols = arity if ncols is None else ncols
    out = np.zeros(r.shape[0], dtype=np.uint64)
    ctx.check(ctx.lib.gd_prefix_hash(ctx.h, _ptr(r), r.shape[0], arity, ncols, _ptr(out)))
    return out


def group_starts(tuples: tuple_array, prefix_len: int, workers: int = 1, ctx: Context | None = None):
    """detail::group_starts (index_map.hpp:46-66)."""
    ctx = ctx or default_context()
    out = np.zeros(max(tuples.count(), 1), dtype=np.uint64)
    m = C.c_uint64(0)
    ctx.check(ctx.lib.gd_group_starts(ctx.h, _ptr(tuples.data), tuples.count(), tuples.arity,
                                      int(tuples.canonical), prefix_len, _ptr(out), C.byref(m)))
    return out[: m.value]


# ---------------------------------------------------------------------------
# HISA index + container (index_map.hpp, container.hpp)

@dataclass
class index_map:
    """Device HISA index parameters; slot_count()/occupied() follow the
    reference sizing rule (index_map.hpp:87-94)."""

    prefix_len: int
    load_factor: float
    _slot_count: int
    _occupied: int

    def slot_count(self) -> int:
        return self._slot_count

    def occupied(self) -> int:
        return self._occupied


@dataclass
class row_range:
    start: int = 0
    count: int = 0

    def empty(self) -> bool:
        return self.count == 0


@dataclass
class relation_container:
    tuples: tuple_array
    index: index_map | None = None
    permutation: list = field(default_factory=list)

    def arity(self) -> int:
        return self.tuples.arity

    def row_count(self) -> int:
        return self.tuples.count()


def _index_call(tuples: tuple_array, prefix_len: int, load_factor: float, keys: np.ndarray, ctx: Context,
                key_len: int | None = None):
    kl = prefix_len if key_len is None else key_len
    k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64).reshape(-1, max(kl, 1)))
    st = np.zeros(max(len(k), 1), dtype=np.uint64)
    ct = np.zeros(max(len(k), 1), dtype=np.uint64)
    sc, oc = C.c_uint64(0), C.c_uint64(0)
    ctx.check(ctx.lib.gd_index_lookup(ctx.h, _ptr(tuples.data), tuples.count(), tuples.arity,
                                      int(tuples.canonical), prefix_len, load_factor, _ptr(k), len(k), kl,
                                      _ptr(st), _ptr(ct), C.byref(sc), C.byref(oc)))
    return st[: len(k)], ct[: len(k)], sc.value, oc.value


def build_index(tuples: tuple_array, prefix_len: int, load_factor: float = 0.8, workers: int = 1,
                ctx: Context | None = None) -> index_map:
    """build_index (index_map.hpp:74-124), built on the device."""
    ctx = ctx or default_context()
    _, _, sc, oc = _index_call(tuples, prefix_len, load_factor, np.zeros((0, max(prefix_len, 1))), ctx)
    return index_map(prefix_len, load_factor, sc, oc)


def make_container(canonical: tuple_array, permutation=None, index_prefix_len: int | None = None,
                   load_factor: float = 0.8, workers: int = 1, ctx: Context | None = None) -> relation_container:
    """make_container (container.hpp:99-114)."""
    if not canonical.canonical:
        raise logic_error("make_container: array must be canonical")
    c = relation_container(canonical, None,
                           list(permutation) if permutation else list(range(canonical.arity)))
    if index_prefix_len:
        c.index = build_index(canonical, index_prefix_len, load_factor, workers, ctx)
    return c


def range_lookup_batch(c: relation_container, prefixes, ctx: Context | None = None):
    """Batched range_lookup (container.hpp:52-89): one device index build,
    one probe per prefix row.  Returns (starts, counts)."""
    ctx = ctx or default_context()
    if c.index is None:
        raise usage_error("range_lookup: container has no index")
    p = np.asarray(prefixes, dtype=np.uint64)
    kl = p.shape[1] if p.ndim == 2 else (len(p) if p.ndim == 1 and len(p) else c.index.prefix_len)
    if kl != c.index.prefix_len:
        raise usage_error(f"range_lookup: prefix length {kl} does not match index prefix_len "
                          f"{c.index.prefix_len}")
    st, ct, _, _ = _index_call(c.tuples, c.index.prefix_len, c.index.load_factor, p.reshape(-1, kl), ctx)
    return st, ct


def range_lookup(c: relation_container, prefix, ctx: Context | None = None) -> row_range:
    """range_lookup (container.hpp:52-89) for one prefix."""
    prefix = list(prefix)
    if c.index is None:
        raise usage_error("range_lookup: container has no index")
    if len(prefix) != c.index.prefix_len:
        raise usage_error(f"range_lookup: prefix length {len(prefix)} does not match index prefix_len "
                          f"{c.index.prefix_len}")
    st, ct = range_lookup_batch(c, np.asarray([prefix], dtype=np.uint64), ctx)
    return row_range(int(st[0]), int(ct[0]))


# ---------------------------------------------------------------------------
# Join specs (ra.hpp:18-66) and RA functions

class operand:
    @staticmethod
    def outer(c: int) -> A.gd_operand:
        return A.gd_operand(A.GD_OUTER_COL, c, 0)

    @staticmethod
    def inner(c: int) -> A.gd_operand:
        return A.gd_operand(A.GD_INNER_COL, c, 0)

    @staticmethod
    def constant(v: int) -> A.gd_operand:
        return A.gd_operand(A.GD_CONSTANT, 0, v)


@dataclass
class column_map:
    sources: list = field(default_factory=list)

    def output_arity(self) -> int:
        return len(self.sources)


def row_filter(lhs: A.gd_operand, rhs: A.gd_operand, require_equal: bool = False) -> A.gd_filter:
    return A.gd_filter(lhs, rhs, int(require_equal), 0)


@dataclass
class join_spec:
    join_column_count: int = 0
    outer: relation_container | None = None
    inner: relation_container | None = None
    projection: column_map = field(default_factory=column_map)
    filters: list = field(default_factory=list)


def _view(c: relation_container) -> A.gd_container_view:
    t = c.tuples
    return A.gd_container_view(_ptr(t.data), t.count(), t.arity, int(t.canonical),
                               c.index.prefix_len if c.index else 0, 0,
                               c.index.load_factor if c.index else 0.8)


def _spec(s: join_spec) -> A.gd_join_spec:
    g = A.gd_join_spec()
    g.join_column_count = s.join_column_count
    g.proj_arity = len(s.projection.sources)
    for i, o in enumerate(s.projection.sources):
        g.proj[i] = o
    g.nfilters = len(s.filters)
    for i, f in enumerate(s.filters):
        g.filters[i] = f
    return g


def _check_spec(s: join_spec):
    if s.outer is None or s.inner is None:
        raise usage_error("join: outer and inner are required")


def join_count(spec: join_spec, workers: int = 1, stride_rows: int = 0, ctx: Context | None = None) -> int:
    """join_count (ra.hpp:141-182)."""
    ctx = ctx or default_context()
    _check_spec(spec)
    total = C.c_uint64(0)
    o, i, g = _view(spec.outer), _view(spec.inner), _spec(spec)
    ctx.check(ctx.lib.gd_join_count(ctx.h, C.byref(o), C.byref(i), C.byref(g), C.byref(total)))
    return total.value


def join_materialize(spec: join_spec, out: tuple_array, workers: int = 1, stride_rows: int = 0,
                     ctx: Context | None = None) -> None:
    """join_materialize (ra.hpp:189-263): `out` must be pre-sized to
    join_count rows of output_arity; rows land in outer-row, then
    inner-range order."""
    ctx = ctx or default_context()
    _check_spec(spec)
    arity = spec.projection.output_arity()
    cap = out.count() if out.arity == arity else out.data.size // max(arity, 1)
    buf = np.zeros((max(cap, 1), max(arity, 1)), dtype=np.uint64)
    o, i, g = _view(spec.outer), _view(spec.inner), _spec(spec)
    ctx.check(ctx.lib.gd_join_materialize(ctx.h, C.byref(o), C.byref(i), C.byref(g), _ptr(buf), cap))
    out.arity = arity
    out.canonical = False
    out.data = buf[:cap].copy()


def select_project(src: relation_container, projection: column_map, filters=(),
                   ctx: Context | None = None) -> tuple_array:
    """select_project (ra.hpp:267-293)."""
    ctx = ctx or default_context()
    t = src.tuples
    pa = (A.gd_operand * max(projection.output_arity(), 1))(*projection.sources)
    fa = (A.gd_filter * max(len(filters), 1))(*filters)
    out = np.zeros((max(t.count(), 1), max(projection.output_arity(), 1)), dtype=np.uint64)
    m = C.c_uint64(0)
    ctx.check(ctx.lib.gd_select_project(ctx.h, _ptr(t.data), t.count(), t.arity, pa, projection.output_arity(),
                                        fa, len(filters), _ptr(out), C.byref(m)))
    return tuple_array(projection.output_arity(), out[: m.value])


def merge_sorted(full: tuple_array, delta: tuple_array, buffer_rows: int | None = None, workers: int = 1,
                 ctx: Context | None = None) -> tuple_array:
    """merge_sorted (ra.hpp:299-381): canonical union of disjoint inputs
    through a merge buffer of `buffer_rows` rows (default: exactly enough)."""
    ctx = ctx or default_context()
    if full.arity != delta.arity:
        raise logic_error("merge_sorted: arity mismatch")
    nf, nd = full.count(), delta.count()
    buf = nf + nd if buffer_rows is None else buffer_rows
    out = np.zeros((nf + nd, full.arity), dtype=np.uint64)
    ctx.check(ctx.lib.gd_merge_sorted(ctx.h, _ptr(full.data), nf, int(full.canonical), _ptr(delta.data), nd,
                                      int(delta.canonical), full.arity, buf, _ptr(out)))
    return tuple_array(full.arity, out, canonical=True)


def difference(new_rel: tuple_array, full: tuple_array, workers: int = 1,
               ctx: Context | None = None) -> tuple_array:
    """difference (ra.hpp:386-422)."""
    ctx = ctx or default_context()
    if new_rel.arity != full.arity:
        raise logic_error("difference: arity mismatch")
    out = np.zeros_like(new_rel.data)
    m = C.c_uint64(0)
    ctx.check(ctx.lib.gd_difference(ctx.h, _ptr(new_rel.data), new_rel.count(), int(new_rel.canonical),
                                    _ptr(full.data), full.count(), int(full.canonical), new_rel.arity, _ptr(out),
                                    C.byref(m)))
    return tuple_array(new_rel.arity, out[: m.value], canonical=True)


# ---------------------------------------------------------------------------
# Engine (engine.hpp:25-277) and run_stats (stats.hpp:21-46)

@dataclass
class engine_config:
    memory_budget_bytes: int = (1 << 64) - 1
    ebm_enabled: bool = True
    alpha: int = 5
    load_factor: float = 0.8
    workers: int = 0
    stride_rows: int = 0

    def to_c(self) -> A.gd_engine_config:
        return A.gd_engine_config(self.memory_budget_bytes, int(self.ebm_enabled), self.alpha, self.load_factor,
                                  self.workers, 0, self.stride_rows)


@dataclass
class run_stats:
    phase_seconds: dict = field(default_factory=dict)
    total_seconds: float = 0.0
    iterations: int = 0
    delta_history: list = field(default_factory=list)  # [(relation, [rows...])], relation-name order
    buffer_allocations: int = 0
    charge_events: int = 0
    peak_tracked_bytes: int = 0
    peak_temp_bytes: int = 0
    # device extras
    join_tuples: int = 0
    device_bytes_peak: int = 0

    def phase(self, name: str) -> float:
        return self.phase_seconds.get(name, 0.0)

    def other_seconds(self) -> float:
        cat = sum(self.phase(p) for p in A.PHASES if p != "other")
        return max(self.total_seconds - cat, 0.0)


def _stats_to_tsv(s: run_stats) -> str:
    """to_tsv(run_stats) (stats.hpp:50-64)."""
    out = ["phase\tseconds"]
    for p in A.PHASES:
        v = s.other_seconds() if p == "other" else s.phase(p)
        out.append(f"{p}\t{v:g}")
    for rel, deltas in s.delta_history:
        out.append(f"relation\t{rel}")
        out.append("iteration\tdelta_rows")
        for i, d in enumerate(deltas):
            out.append(f"{i + 1}\t{d}")
    return "\n".join(out) + "\n"


class engine:
    """arraylog::engine on the B200 (engine.hpp:40-558)."""

    def __init__(self, program: Program | str, cfg: engine_config | None = None, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.prog = builtin_program(program) if isinstance(program, str) else program
        self.cfg = cfg or engine_config()
        lib = self.ctx.lib
        n = len(self.prog.relations)
        ar = (A.u32 * n)(*[a for _, a, _ in self.prog.relations])
        ed = (A.u32 * n)(*[int(e) for _, _, e in self.prog.relations])
        names = (C.c_char_p * n)(*[nm.encode() for nm, _, _ in self.prog.relations])
        h = C.c_void_p()
        c = self.cfg.to_c()
        self.ctx.check(lib.gd_engine_create(self.ctx.h, C.byref(c), n, ar, ed, names, C.byref(h)))
        self.h = h
        self._plans = to_blob(self.prog)
        self._set_plans(self._plans)
        self._seeded = False

    def _set_plans(self, plans):
        arr = (A.gd_rule_plan * max(len(plans), 1))(*plans)
        self.ctx.check(self.ctx.lib.gd_engine_set_plans(self.h, arr, len(plans)))

    def override_plans(self, plans):
        """override_plans (engine.hpp:97-101): gd_rule_plan list."""
        if self._seeded:
            raise logic_error("override_plans: engine already seeded")
        self._plans = list(plans)
        self._set_plans(self._plans)

    def plans(self):
        return self._plans

    def _rid(self, name: str, *, edb: bool | None = None) -> int:
        for i, (n, _, e) in enumerate(self.prog.relations):
            if n == name:
                return i
        if edb:
            raise load_error(f"load_edb: '{name}' is not a declared EDB relation")
        raise usage_error(f"unknown relation '{name}'")

    def load_edb(self, name: str, facts: tuple_array):
        """load_edb (engine.hpp:107-128)."""
        rid = self._rid(name, edb=True)
        if not self.prog.relations[rid][2]:
            raise load_error(f"load_edb: '{name}' is not a declared EDB relation")
        ar = self.prog.relations[rid][1]
        if facts.arity != ar:
            raise load_error(f"load_edb: '{name}' expects arity {ar}, got {facts.arity}")
        d = np.ascontiguousarray(facts.data)
        self.ctx.check(self.ctx.lib.gd_engine_load_edb(self.h, rid, _ptr(d), facts.count(), int(facts.canonical)))

    def load_edb_tsv(self, name: str, path):
        """load_edb(name, read_facts(path, arity)) with the file parsed on the
        device straight into the relation."""
        rid = self._rid(name, edb=True)
        text = _read_bytes(path)
        self.ctx.check(self.ctx.lib.gd_engine_load_edb_tsv(self.h, rid, str(path).encode(), text, len(text)))

    def relation_tsv(self, name: str) -> bytes:
        """to_tsv(relation(name)) (io.hpp:118-133), formatted on the device."""
        rid = self._rid(name)
        n = A.u64()
        self.ctx.check(self.ctx.lib.gd_engine_relation_tsv(self.h, rid, None, 0, C.byref(n)))
        buf = C.create_string_buffer(max(n.value, 1))
        self.ctx.check(self.ctx.lib.gd_engine_relation_tsv(self.h, rid, buf, n.value, C.byref(n)))
        return buf.raw[: n.value]

    def load_edb_device(self, name: str, d_ptr: int, count: int, canonical: bool = False):
        """load_edb from device-resident rows (count x arity uint64 at d_ptr)."""
        rid = self._rid(name, edb=True)
        self.ctx.check(self.ctx.lib.gd_engine_load_edb_device(self.h, rid, C.c_void_p(d_ptr), count,
                                                              int(canonical)))

    def run(self):
        self.seed()
        self.iterate_to_fixpoint()

    def seed(self):
        self.ctx.check(self.ctx.lib.gd_engine_seed(self.h))
        self._seeded = True

    def iterate_to_fixpoint(self):
        self.ctx.check(self.ctx.lib.gd_engine_iterate(self.h))
        self._seeded = True

    def relation_count(self, name: str) -> int:
        n = C.c_uint64(0)
        self.ctx.check(self.ctx.lib.gd_engine_relation_count(self.h, self._rid(name), C.byref(n)))
        return n.value

    def relation(self, name: str) -> tuple_array:
        """relation(name) (engine.hpp:259-264): canonical rows."""
        rid = self._rid(name)
        n = self.relation_count(name)
        ar = self.prog.relations[rid][1]
        out = np.zeros((n, ar), dtype=np.uint64)
        self.ctx.check(self.ctx.lib.gd_engine_relation_download(self.h, rid, _ptr(out), n))
        return tuple_array(ar, out, canonical=True)

    def relation_digest(self, name: str) -> int:
        d = C.c_uint64(0)
        self.ctx.check(self.ctx.lib.gd_engine_relation_digest(self.h, self._rid(name), C.byref(d)))
        return d.value

    def idb_relations(self):
        return self.prog.idbs

    def delta_history(self, name: str):
        rid = self._rid(name)
        ln = C.c_uint64(0)
        self.ctx.check(self.ctx.lib.gd_engine_delta_history(self.h, rid, None, 0, C.byref(ln)))
        h = np.zeros(max(ln.value, 1), dtype=np.uint64)
        self.ctx.check(self.ctx.lib.gd_engine_delta_history(self.h, rid, _ptr(h), ln.value, C.byref(ln)))
        return [int(x) for x in h[: ln.value]]

    def iter_log(self, name: str):
        rid = self._rid(name)
        ln = C.c_uint64(0)
        self.ctx.check(self.ctx.lib.gd_engine_iter_log(self.h, rid, None, 0, C.byref(ln)))
        recs = (A.gd_iter_record * max(ln.value, 1))()
        self.ctx.check(self.ctx.lib.gd_engine_iter_log(self.h, rid, recs, ln.value, C.byref(ln)))
        return [(r.delta_in, r.join, r.new_unique, r.delta_out, r.full_after) for r in recs[: ln.value]]

    def encoding(self):
        b, k, d = A.u32(), A.u32(), A.u32()
        self.ctx.check(self.ctx.lib.gd_engine_encoding(self.h, C.byref(b), C.byref(k), C.byref(d)))
        return {"bits": b.value, "key_words": k.value, "dictionary": bool(d.value)}

    def raw_stats(self) -> A.gd_run_stats:
        s = A.gd_run_stats()
        self.ctx.check(self.ctx.lib.gd_engine_stats(self.h, C.byref(s)))
        return s

    def stats(self) -> run_stats:
        """stats() (engine.hpp:270-277)."""
        s = self.raw_stats()
        hist = []
        rec = sorted({self.prog.relations[p.head_rel][0] for p in self._plans if p.recursive})
        for name in rec:  # std::map order (engine.hpp:192, 254-255)
            hist.append((name, self.delta_history(name)))
        return run_stats(
            phase_seconds={p: s.phase_seconds[i] for i, p in enumerate(A.PHASES) if p != "other"},
            total_seconds=s.total_seconds, iterations=s.iterations, delta_history=hist,
            buffer_allocations=s.buffer_allocations, charge_events=s.charge_events,
            peak_tracked_bytes=s.peak_tracked_bytes, peak_temp_bytes=s.peak_temp_bytes,
            join_tuples=s.join_tuples, device_bytes_peak=s.device_bytes_peak)

    # --- hash-partitioned multi-GPU mode ----------------------
    def set_partition(self, rank: int, nranks: int):
        self.ctx.check(self.ctx.lib.gd_engine_set_partition(self.h, rank, nranks))

    def exchange_words(self) -> int:
        w = A.u32()
        self.ctx.check(self.ctx.lib.gd_engine_exchange_words(self.h, C.byref(w)))
        return w.value

    def partition_begin(self, nranks: int):
        counts = np.zeros(nranks, dtype=np.uint64)
        ptr = C.c_void_p()
        self.ctx.check(self.ctx.lib.gd_engine_partition_begin(self.h, _ptr(counts), C.byref(ptr)))
        return counts, (ptr.value or 0)

    def partition_end(self, d_recv: int, recv_rows: int) -> int:
        d = C.c_uint64(0)
        self.ctx.check(self.ctx.lib.gd_engine_partition_end(self.h, C.c_void_p(d_recv), recv_rows, C.byref(d)))
        return d.value

    def run_partitioned(self, comm, max_iters: int = 0) -> int:
        """gd_engine_run_partitioned: the native multi-GPU driver (NCCL
        exchanges issued by the library on the context stream); collective
        over the ranks of `comm` (partition.NcclComm).  Returns iterations."""
        it = C.c_uint64(0)
        self.ctx.check(self.ctx.lib.gd_engine_run_partitioned(self.h, comm.h, max_iters, C.byref(it)))
        return it.value

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.gd_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
