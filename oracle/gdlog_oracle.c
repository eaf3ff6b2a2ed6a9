/*
 * oracle/gdlog_oracle.c — TEST INFRASTRUCTURE ONLY (the "port" oracle).
 *
 * A plain-C, single-threaded restatement of the reference CPU engine's hot
 * path (arraylog, /root/reference/proj/include/arraylog/*.hpp).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * it, and only as a checker; the product (paper_2311_02206_b200/) never
 * links or calls it.  Every function cites the reference lines it follows.
 *
 * Pinning: tests/test_oracle.py checks this restatement against (a) the
 * known-answer vectors of the reference's own gtest suites (committed in
 * tests/golden/known_answers.json with file:line provenance) and (b) the
 * reference engine itself, compiled from /root/reference into
 * oracle/_ref/libarraylog_ref.so (oracle/Makefile), on seeded corpora and
 * on the committed golden fixtures of tests/golden/.
 *
 * Arguments mirror include/gdlog_b200.h (without the context).  Errors are
 * returned as gd_status codes with a message in or_last_error().
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "gdlog_b200.h"

#define EMPTY_SLOT UINT64_MAX /* kEmptySlot, types.hpp:16 */

static char g_err[512];

const char* or_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

/* ---------------------------------------------------------------------
 * hash.hpp:13-60 — fmix64, prefix_hash (Murmur3 x64-128 mix, seed 0,
 * returns h1 + h2), slot_key (sentinel remap). */

static uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

static uint64_t fmix64(uint64_t k) { /* hash.hpp:13-20 */
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdULL;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ULL;
    k ^= k >> 33;
    return k;
}

static uint64_t prefix_hash(const uint64_t* cols, uint32_t n) { /* hash.hpp:28-53 */
    const uint64_t c1 = 0x87c37b91114253d5ULL, c2 = 0x4cf5ad432745937fULL;
    uint64_t h1 = 0, h2 = 0;
    for (uint32_t i = 0; i + 1 < n; i += 2) {
        uint64_t k1 = cols[i], k2 = cols[i + 1];
        k1 *= c1; k1 = rotl64(k1, 31); k1 *= c2; h1 ^= k1;
        h1 = rotl64(h1, 27); h1 += h2; h1 = h1 * 5 + 0x52dce729;
        k2 *= c2; k2 = rotl64(k2, 33); k2 *= c1; h2 ^= k2;
        h2 = rotl64(h2, 31); h2 += h1; h2 = h2 * 5 + 0x38495ab5;
    }
    if (n % 2) {
        uint64_t k1 = cols[n - 1];
        k1 *= c1; k1 = rotl64(k1, 31); k1 *= c2; h1 ^= k1;
    }
    const uint64_t len = (uint64_t)n * 8u;
    h1 ^= len; h2 ^= len;
    h1 += h2; h2 += h1;
    h1 = fmix64(h1);
    h2 = fmix64(h2);
    return h1 + h2;
}

static uint64_t slot_key(const uint64_t* cols, uint32_t n) { /* hash.hpp:57-60 */
    uint64_t h = prefix_hash(cols, n);
    return h == EMPTY_SLOT ? EMPTY_SLOT - 1 : h;
}

int or_prefix_hash(const uint64_t* rows, uint64_t n, uint32_t arity,
                   uint32_t ncols, uint64_t* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = slot_key(rows + i * arity, ncols);
    return GD_OK;
}

/* ---------------------------------------------------------------------
 * tuple_array.hpp:55-61 — lexicographic row compare. */
static int cmp_rows(const uint64_t* a, const uint64_t* b, uint32_t k) {
    for (uint32_t c = 0; c < k; ++c)
        if (a[c] != b[c]) return a[c] < b[c] ? -1 : 1;
    return 0;
}

/* Stable merge sort of row indices (the reference sorts an index vector,
 * tuple_array.hpp:92-122; any correct sort yields the same canonical
 * bytes because equal rows are identical). */
static void sort_indices(const uint64_t* rows, uint32_t k, uint64_t* idx,
                         uint64_t n) {
    if (n < 2) return;
    uint64_t* tmp = (uint64_t*)malloc(n * sizeof(uint64_t));
    for (uint64_t w = 1; w < n; w *= 2) {
        for (uint64_t lo = 0; lo < n; lo += 2 * w) {
            uint64_t mid = lo + w < n ? lo + w : n;
            uint64_t hi = lo + 2 * w < n ? lo + 2 * w : n;
            uint64_t i = lo, j = mid, o = lo;
            while (i < mid && j < hi)
                tmp[o++] = cmp_rows(rows + idx[j] * k, rows + idx[i] * k, k) < 0
                               ? idx[j++]
                               : idx[i++];
            while (i < mid) tmp[o++] = idx[i++];
            while (j < hi) tmp[o++] = idx[j++];
        }
        memcpy(idx, tmp, n * sizeof(uint64_t));
    }
    free(tmp);
}

/* canonicalize, tuple_array.hpp:73-133: index sort + adjacent dedup gather.
 * `out` may alias nothing; returns distinct count. */
static uint64_t canon(const uint64_t* rows, uint64_t n, uint32_t k,
                      uint64_t* out) {
    if (n == 0) return 0;
    uint64_t* idx = (uint64_t*)malloc(n * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) idx[i] = i;
    sort_indices(rows, k, idx, n);
    uint64_t m = 0;
    const uint64_t* prev = NULL;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t* r = rows + idx[i] * k;
        if (prev && cmp_rows(prev, r, k) == 0) continue;
        memcpy(out + m * k, r, k * sizeof(uint64_t));
        prev = out + m * k;
        ++m;
    }
    free(idx);
    return m;
}

int or_canonicalize(const uint64_t* rows, uint64_t n, uint32_t arity,
                    uint64_t* out, uint64_t* out_n) {
    if (arity == 0) return fail(GD_ERR_LOGIC, "canonicalize: arity must be positive");
    *out_n = canon(rows, n, arity, out);
    return GD_OK;
}

/* permute_columns, ra.hpp:426-454. */
int or_permute_columns(const uint64_t* rows, uint64_t n, uint32_t arity,
                       int canonical, const uint32_t* perm, uint32_t perm_len,
                       uint64_t* out, uint64_t* out_n) {
    if (!canonical) return fail(GD_ERR_LOGIC, "permute_columns: input must be canonical");
    if (perm_len != arity) return fail(GD_ERR_CONFIG, "permute_columns: permutation size mismatch");
    int seen[GD_MAX_ARITY] = {0};
    int ident = 1;
    for (uint32_t c = 0; c < arity; ++c) {
        if (perm[c] >= arity || seen[perm[c]])
            return fail(GD_ERR_CONFIG, "permute_columns: not a bijection");
        seen[perm[c]] = 1;
        if (perm[c] != c) ident = 0;
    }
    if (ident) {
        memcpy(out, rows, n * arity * sizeof(uint64_t));
        *out_n = n;
        return GD_OK;
    }
    uint64_t* raw = (uint64_t*)malloc((n ? n : 1) * arity * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i)
        for (uint32_t c = 0; c < arity; ++c) raw[i * arity + c] = rows[i * arity + perm[c]];
    *out_n = canon(raw, n, arity, out);
    free(raw);
    return GD_OK;
}

/* ---------------------------------------------------------------------
 * index_map.hpp:18-124 and container.hpp:52-89: the HISA index. */

typedef struct {
    uint64_t key_hash;
    uint64_t offset;
} or_slot;

typedef struct {
    or_slot* slots;
    uint64_t slot_count;
    uint64_t occupied;
    uint32_t prefix_len;
} or_index;

/* group_starts, index_map.hpp:46-66. Returns count; starts has room n. */
static uint64_t group_starts(const uint64_t* rows, uint64_t n, uint32_t k,
                             uint32_t plen, uint64_t* starts) {
    uint64_t m = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (i == 0 || cmp_rows(rows + (i - 1) * k, rows + i * k, plen) != 0)
            starts[m++] = i;
    return m;
}

int or_group_starts(const uint64_t* rows, uint64_t n, uint32_t arity,
                    int canonical, uint32_t prefix_len, uint64_t* out_starts,
                    uint64_t* out_count) {
    (void)canonical;
    *out_count = group_starts(rows, n, arity, prefix_len, out_starts);
    return GD_OK;
}

/* build_index, index_map.hpp:74-124: sequential linear probing in group
 * order, min offset on an equal prefix; byte-identical to the reference. */
static int index_build(const uint64_t* rows, uint64_t n, uint32_t k,
                       int canonical, uint32_t plen, double lf, or_index* ix) {
    if (!canonical) return fail(GD_ERR_LOGIC, "build_index: tuples must be canonical");
    if (plen == 0 || plen > k) return fail(GD_ERR_CONFIG, "build_index: prefix_len must be in [1, arity]");
    if (!(lf > 0.0) || lf >= 1.0) return fail(GD_ERR_CONFIG, "build_index: load factor must be in (0, 1)");
    uint64_t* starts = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    uint64_t distinct = group_starts(rows, n, k, plen, starts);
    uint64_t sc = distinct == 0 ? 1 : (uint64_t)ceil((double)distinct / lf);
    while ((double)distinct > lf * (double)sc) ++sc;
    ix->slot_count = sc;
    ix->prefix_len = plen;
    ix->occupied = distinct;
    ix->slots = (or_slot*)malloc(sc * sizeof(or_slot));
    for (uint64_t i = 0; i < sc; ++i) {
        ix->slots[i].key_hash = EMPTY_SLOT;
        ix->slots[i].offset = 0;
    }
    for (uint64_t g = 0; g < distinct; ++g) {
        uint64_t off = starts[g];
        uint64_t h = slot_key(rows + off * k, plen);
        uint64_t i = h % sc;
        for (;;) {
            or_slot* s = &ix->slots[i];
            if (s->key_hash == EMPTY_SLOT) {
                s->key_hash = h;
                s->offset = off;
                break;
            }
            if (s->key_hash == h && cmp_rows(rows + s->offset * k, rows + off * k, plen) == 0) {
                if (off < s->offset) s->offset = off;
                break;
            }
            i = (i + 1) % sc;
        }
    }
    free(starts);
    return GD_OK;
}

/* range_lookup, container.hpp:52-89: probe, verify prefix, forward scan. */
static void index_lookup(const or_index* ix, const uint64_t* rows, uint64_t n,
                         uint32_t k, const uint64_t* key, uint64_t* start,
                         uint64_t* count) {
    const uint32_t plen = ix->prefix_len;
    const uint64_t h = slot_key(key, plen);
    uint64_t i = h % ix->slot_count;
    *start = 0;
    *count = 0;
    for (uint64_t probes = 0; probes < ix->slot_count; ++probes) {
        const or_slot* s = &ix->slots[i];
        if (s->key_hash == EMPTY_SLOT) return;
        if (s->key_hash == h && cmp_rows(rows + s->offset * k, key, plen) == 0) {
            uint64_t end = s->offset + 1;
            while (end < n && cmp_rows(rows + end * k, key, plen) == 0) ++end;
            *start = s->offset;
            *count = end - s->offset;
            return;
        }
        i = (i + 1) % ix->slot_count;
    }
}

int or_index_lookup(const uint64_t* rows, uint64_t n, uint32_t arity,
                    int canonical, uint32_t prefix_len, double load_factor,
                    const uint64_t* keys, uint64_t nkeys, uint32_t key_len,
                    uint64_t* out_start, uint64_t* out_count,
                    uint64_t* out_slot_count, uint64_t* out_occupied) {
    or_index ix;
    int rc = index_build(rows, n, arity, canonical, prefix_len, load_factor, &ix);
    if (rc) return rc;
    if (key_len != prefix_len) {
        free(ix.slots);
        return fail(GD_ERR_USAGE, "range_lookup: prefix length does not match index prefix_len");
    }
    for (uint64_t i = 0; i < nkeys; ++i)
        index_lookup(&ix, rows, n, arity, keys + i * key_len, out_start + i, out_count + i);
    *out_slot_count = ix.slot_count;
    *out_occupied = ix.occupied;
    free(ix.slots);
    return GD_OK;
}

/* ---------------------------------------------------------------------
 * ra.hpp:18-263 — join_count / join_materialize / select_project. */

typedef struct {
    const uint64_t* rows;
    uint64_t n;
    uint32_t arity;
    const or_index* index; /* NULL = none */
} or_container;

static uint64_t eval_operand(const gd_operand* op, const uint64_t* o,
                             const uint64_t* i) { /* ra.hpp:70-77 */
    switch (op->kind) {
        case GD_OUTER_COL: return o[op->column];
        case GD_INNER_COL: return i[op->column];
        default: return op->value;
    }
}

static int passes(const gd_filter* f, uint32_t nf, const uint64_t* o,
                  const uint64_t* i) { /* ra.hpp:79-88 */
    for (uint32_t k = 0; k < nf; ++k) {
        uint64_t a = eval_operand(&f[k].lhs, o, i), b = eval_operand(&f[k].rhs, o, i);
        if ((a == b) != (f[k].require_equal != 0)) return 0;
    }
    return 1;
}

static int validate_operand(const gd_operand* op, uint32_t oa, uint32_t ia) { /* ra.hpp:90-96 */
    if (op->kind == GD_OUTER_COL && op->column >= oa) return fail(GD_ERR_CONFIG, "join: outer column out of range");
    if (op->kind == GD_INNER_COL && op->column >= ia) return fail(GD_ERR_CONFIG, "join: inner column out of range");
    return GD_OK;
}

static int validate_spec(const or_container* o, const or_container* in,
                         const gd_join_spec* s) { /* ra.hpp:98-120 */
    if (s->proj_arity == 0) return fail(GD_ERR_CONFIG, "join: projection must produce at least one column");
    if (s->join_column_count > 0) {
        if (s->join_column_count > o->arity || s->join_column_count > in->arity)
            return fail(GD_ERR_CONFIG, "join: join_column_count exceeds arity");
        if (!in->index) return fail(GD_ERR_USAGE, "join: inner relation has no index");
        if (in->index->prefix_len != s->join_column_count)
            return fail(GD_ERR_USAGE, "join: inner index prefix_len does not match join columns");
    }
    for (uint32_t c = 0; c < s->proj_arity; ++c) {
        int rc = validate_operand(&s->proj[c], o->arity, in->arity);
        if (rc) return rc;
    }
    for (uint32_t f = 0; f < s->nfilters; ++f) {
        int rc = validate_operand(&s->filters[f].lhs, o->arity, in->arity);
        if (!rc) rc = validate_operand(&s->filters[f].rhs, o->arity, in->arity);
        if (rc) return rc;
    }
    return GD_OK;
}

static void match_range(const or_container* in, uint32_t jcc,
                        const uint64_t* orow, uint64_t* start,
                        uint64_t* count) { /* ra.hpp:122-127 */
    if (jcc == 0) {
        *start = 0;
        *count = in->n;
        return;
    }
    index_lookup(in->index, in->rows, in->n, in->arity, orow, start, count);
}

/* Count pass (join_count, ra.hpp:141-182) when out == NULL; otherwise the
 * write pass of join_materialize (ra.hpp:189-263): outer-row order, then
 * inner-range order.  Returns rows produced (or that would be). */
static uint64_t join_run(const or_container* o, const or_container* in,
                         const gd_join_spec* s, uint64_t* out) {
    if (o->n == 0 || in->n == 0) return 0;
    uint64_t total = 0;
    for (uint64_t r = 0; r < o->n; ++r) {
        const uint64_t* orow = o->rows + r * o->arity;
        uint64_t st, cnt;
        match_range(in, s->join_column_count, orow, &st, &cnt);
        for (uint64_t m = 0; m < cnt; ++m) {
            const uint64_t* irow = in->rows + (st + m) * in->arity;
            if (!passes(s->filters, s->nfilters, orow, irow)) continue;
            if (out)
                for (uint32_t c = 0; c < s->proj_arity; ++c)
                    out[total * s->proj_arity + c] = eval_operand(&s->proj[c], orow, irow);
            ++total;
        }
    }
    return total;
}

static int open_view(const gd_container_view* v, or_container* c, or_index* ix) {
    c->rows = v->rows;
    c->n = v->n;
    c->arity = v->arity;
    c->index = NULL;
    if (v->index_prefix_len) {
        int rc = index_build(v->rows, v->n, v->arity, v->canonical, v->index_prefix_len,
                             v->load_factor, ix);
        if (rc) return rc;
        c->index = ix;
    }
    return GD_OK;
}

int or_join_count(const gd_container_view* outer, const gd_container_view* inner,
                  const gd_join_spec* spec, uint64_t* out_total) {
    or_container o, in;
    or_index oi = {0}, ii = {0};
    int rc = open_view(outer, &o, &oi);
    if (!rc) rc = open_view(inner, &in, &ii);
    if (!rc) rc = validate_spec(&o, &in, spec);
    if (!rc) *out_total = join_run(&o, &in, spec, NULL);
    free(oi.slots);
    free(ii.slots);
    return rc;
}

int or_join_materialize(const gd_container_view* outer,
                        const gd_container_view* inner,
                        const gd_join_spec* spec, uint64_t* out,
                        uint64_t out_capacity_rows) {
    or_container o, in;
    or_index oi = {0}, ii = {0};
    int rc = open_view(outer, &o, &oi);
    if (!rc) rc = open_view(inner, &in, &ii);
    if (!rc) rc = validate_spec(&o, &in, spec);
    if (!rc) {
        uint64_t total = join_run(&o, &in, spec, NULL);
        if (total != out_capacity_rows)
            rc = fail(GD_ERR_LOGIC, "join_materialize: output capacity mismatch");
        else
            join_run(&o, &in, spec, out);
    }
    free(oi.slots);
    free(ii.slots);
    return rc;
}

/* select_project, ra.hpp:267-293. */
int or_select_project(const uint64_t* rows, uint64_t n, uint32_t arity,
                      const gd_operand* proj, uint32_t proj_arity,
                      const gd_filter* filters, uint32_t nfilters,
                      uint64_t* out, uint64_t* out_n) {
    for (uint32_t c = 0; c < proj_arity; ++c) {
        if (proj[c].kind == GD_INNER_COL) return fail(GD_ERR_LOGIC, "select_project: inner operand");
        int rc = validate_operand(&proj[c], arity, 0);
        if (rc) return rc;
    }
    for (uint32_t f = 0; f < nfilters; ++f)
        if (filters[f].lhs.kind == GD_INNER_COL || filters[f].rhs.kind == GD_INNER_COL)
            return fail(GD_ERR_LOGIC, "select_project: inner operand");
    uint64_t m = 0;
    for (uint64_t r = 0; r < n; ++r) {
        const uint64_t* row = rows + r * arity;
        if (!passes(filters, nfilters, row, NULL)) continue;
        for (uint32_t c = 0; c < proj_arity; ++c)
            out[m * proj_arity + c] = eval_operand(&proj[c], row, NULL);
        ++m;
    }
    *out_n = m;
    return GD_OK;
}

/* merge_sorted, ra.hpp:299-381 (one tile: the tiling does not change the
 * bytes). Rejects overlap and an undersized buffer. */
int or_merge_sorted(const uint64_t* full, uint64_t nf, int full_canonical,
                    const uint64_t* delta, uint64_t nd, int delta_canonical,
                    uint32_t arity, uint64_t buffer_rows, uint64_t* out) {
    if (!full_canonical || !delta_canonical) return fail(GD_ERR_LOGIC, "merge_sorted: inputs must be canonical");
    if (buffer_rows < nf + nd) return fail(GD_ERR_LOGIC, "merge_sorted: buffer too small");
    uint64_t i = 0, j = 0, w = 0;
    const uint32_t k = arity;
    while (i < nf && j < nd) {
        int c = cmp_rows(full + i * k, delta + j * k, k);
        if (c == 0) return fail(GD_ERR_LOGIC, "merge_sorted: inputs are not disjoint");
        const uint64_t* src = c < 0 ? full + (i++) * k : delta + (j++) * k;
        memcpy(out + (w++) * k, src, k * sizeof(uint64_t));
    }
    for (; i < nf; ++i) memcpy(out + (w++) * k, full + i * k, k * sizeof(uint64_t));
    for (; j < nd; ++j) memcpy(out + (w++) * k, delta + j * k, k * sizeof(uint64_t));
    return GD_OK;
}

/* difference, ra.hpp:386-422: binary search per row, order-preserving. */
static uint64_t diff_rows(const uint64_t* nrows, uint64_t n, const uint64_t* frows,
                          uint64_t nf, uint32_t k, uint64_t* out) {
    uint64_t m = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t* key = nrows + i * k;
        uint64_t a = 0, b = nf;
        while (a < b) {
            uint64_t mid = a + (b - a) / 2;
            if (cmp_rows(frows + mid * k, key, k) < 0) a = mid + 1;
            else b = mid;
        }
        if (a == nf || cmp_rows(frows + a * k, key, k) != 0) {
            memcpy(out + m * k, key, k * sizeof(uint64_t));
            ++m;
        }
    }
    return m;
}

int or_difference(const uint64_t* new_rows, uint64_t nn, int new_canonical,
                  const uint64_t* full, uint64_t nf, int full_canonical,
                  uint32_t arity, uint64_t* out, uint64_t* out_n) {
    if (!new_canonical || !full_canonical) return fail(GD_ERR_LOGIC, "difference: inputs must be canonical");
    *out_n = diff_rows(new_rows, nn, full, nf, arity, out);
    return GD_OK;
}

/* ---------------------------------------------------------------------
 * engine.hpp:40-558 — the semi-naive fixpoint driver, restated over the
 * gd_rule_plan blobs (the data the reference planner produces). */

typedef struct {
    uint64_t* data;
    uint64_t n;
    uint32_t arity;
} arr;

static void arr_free(arr* a) {
    free(a->data);
    a->data = NULL;
    a->n = 0;
}

typedef struct {
    uint32_t perm[GD_MAX_ARITY];
    uint32_t prefix_len;
    arr tuples; /* permuted, canonical */
    or_index index;
    int has_index;
} or_copy;

typedef struct {
    uint32_t arity;
    int is_edb;
    arr full, delta, new_acc;
    or_copy* copies;
    uint32_t ncopies;
    int dirty;
    uint64_t* history;
    uint64_t nhist, caphist;
    gd_iter_record* log;
    uint64_t nlog, caplog;
} or_rel;

typedef struct or_engine {
    uint32_t nrels;
    or_rel* rels;
    gd_rule_plan* plans;
    uint32_t nplans;
    int seeded;
    uint64_t iterations;
} or_engine;

static int is_identity(const uint32_t* p, uint32_t k) {
    for (uint32_t i = 0; i < k; ++i)
        if (p[i] != i) return 0;
    return 1;
}

or_engine* or_engine_create(uint32_t nrels, const uint32_t* arities,
                            const uint32_t* is_edb) {
    or_engine* e = (or_engine*)calloc(1, sizeof(or_engine));
    e->nrels = nrels;
    e->rels = (or_rel*)calloc(nrels, sizeof(or_rel));
    for (uint32_t r = 0; r < nrels; ++r) {
        e->rels[r].arity = arities[r];
        e->rels[r].is_edb = is_edb[r] != 0;
        e->rels[r].full.arity = e->rels[r].delta.arity = e->rels[r].new_acc.arity = arities[r];
    }
    return e;
}

void or_engine_destroy(or_engine* e) {
    if (!e) return;
    for (uint32_t r = 0; r < e->nrels; ++r) {
        or_rel* st = &e->rels[r];
        arr_free(&st->full);
        arr_free(&st->delta);
        arr_free(&st->new_acc);
        for (uint32_t c = 0; c < st->ncopies; ++c) {
            arr_free(&st->copies[c].tuples);
            free(st->copies[c].index.slots);
        }
        free(st->copies);
        free(st->history);
        free(st->log);
    }
    free(e->rels);
    free(e->plans);
    free(e);
}

static or_copy* find_copy(or_rel* st, const uint32_t* perm, uint32_t plen) {
    for (uint32_t c = 0; c < st->ncopies; ++c)
        if (st->copies[c].prefix_len == plen &&
            memcmp(st->copies[c].perm, perm, st->arity * sizeof(uint32_t)) == 0)
            return &st->copies[c];
    return NULL;
}

/* set_plans, engine.hpp:300-310: register every (perm, prefix) copy. */
int or_engine_set_plans(or_engine* e, const gd_rule_plan* plans, uint32_t n) {
    if (e->seeded) return fail(GD_ERR_LOGIC, "override_plans: engine already seeded");
    free(e->plans);
    e->plans = (gd_rule_plan*)malloc((n ? n : 1) * sizeof(gd_rule_plan));
    memcpy(e->plans, plans, n * sizeof(gd_rule_plan));
    e->nplans = n;
    for (uint32_t p = 0; p < n; ++p)
        for (uint32_t v = 0; v < plans[p].nvariants; ++v)
            for (uint32_t s = 0; s < plans[p].variants[v].nsteps; ++s) {
                const gd_join_step* js = &plans[p].variants[v].steps[s];
                or_rel* st = &e->rels[js->inner_rel];
                if (!find_copy(st, js->inner_perm, js->join_column_count)) {
                    st->copies = (or_copy*)realloc(st->copies, (st->ncopies + 1) * sizeof(or_copy));
                    or_copy* c = &st->copies[st->ncopies++];
                    memset(c, 0, sizeof(*c));
                    memcpy(c->perm, js->inner_perm, sizeof(c->perm));
                    c->prefix_len = js->join_column_count;
                    c->tuples.arity = st->arity;
                }
                st->dirty = 1;
            }
    return GD_OK;
}

/* load_edb, engine.hpp:107-128. */
int or_engine_load_edb(or_engine* e, uint32_t rel, const uint64_t* rows,
                       uint64_t n, int canonical) {
    if (e->seeded) return fail(GD_ERR_LOGIC, "load_edb: engine already running");
    if (rel >= e->nrels || !e->rels[rel].is_edb) return fail(GD_ERR_LOAD, "load_edb: not a declared EDB relation");
    or_rel* st = &e->rels[rel];
    for (uint64_t i = 0; i < n * st->arity; ++i)
        if (rows[i] == EMPTY_SLOT) return fail(GD_ERR_LOAD, "load_edb: contains the reserved sentinel value");
    arr_free(&st->full);
    st->full.data = (uint64_t*)malloc((n ? n : 1) * st->arity * sizeof(uint64_t));
    if (canonical) {
        memcpy(st->full.data, rows, n * st->arity * sizeof(uint64_t));
        st->full.n = n;
    } else {
        st->full.n = canon(rows, n, st->arity, st->full.data);
    }
    st->dirty = 1;
    return GD_OK;
}

/* refresh_copies, engine.hpp:365-395: permute -> canonicalize -> index. */
static void refresh_copies(or_engine* e, or_rel* st) {
    (void)e;
    for (uint32_t c = 0; c < st->ncopies; ++c) {
        or_copy* cp = &st->copies[c];
        arr_free(&cp->tuples);
        free(cp->index.slots);
        cp->index.slots = NULL;
        cp->tuples.arity = st->arity;
        cp->tuples.data = (uint64_t*)malloc((st->full.n ? st->full.n : 1) * st->arity * sizeof(uint64_t));
        uint64_t m;
        or_permute_columns(st->full.data, st->full.n, st->arity, 1, cp->perm, st->arity,
                           cp->tuples.data, &m);
        cp->tuples.n = m;
        cp->has_index = cp->prefix_len > 0;
        if (cp->has_index)
            index_build(cp->tuples.data, m, st->arity, 1, cp->prefix_len, 0.8, &cp->index);
    }
    st->dirty = 0;
}

/* execute_chain, engine.hpp:401-484. Returns head-shaped rows (caller frees). */
static arr execute_chain(or_engine* e, const gd_variant* v) {
    or_rel* src = &e->rels[v->src_rel];
    const arr* base = v->src_version == GD_DELTA ? &src->delta : &src->full;
    arr permuted = {0};
    arr cur = *base;
    if (!is_identity(v->src_perm, src->arity)) {
        permuted.arity = src->arity;
        permuted.data = (uint64_t*)malloc((base->n ? base->n : 1) * src->arity * sizeof(uint64_t));
        or_permute_columns(base->data, base->n, src->arity, 1, v->src_perm, src->arity,
                           permuted.data, &permuted.n);
        cur = permuted;
    }
    arr result = {0};
    if (v->nsteps == 0) {
        result.arity = v->sel_arity;
        result.data = (uint64_t*)malloc((cur.n ? cur.n : 1) * v->sel_arity * sizeof(uint64_t));
        or_select_project(cur.data, cur.n, cur.arity, v->sel_proj, v->sel_arity,
                          v->sel_filters, v->nsel_filters, result.data, &result.n);
        arr_free(&permuted);
        return result;
    }
    arr chained = {0};
    for (uint32_t s = 0; s < v->nsteps; ++s) {
        const gd_join_step* js = &v->steps[s];
        or_rel* ist = &e->rels[js->inner_rel];
        or_copy* cp = find_copy(ist, js->inner_perm, js->join_column_count);
        or_container o = {cur.data, cur.n, cur.arity, NULL};
        or_container in = {cp->tuples.data, cp->tuples.n, ist->arity,
                           cp->has_index ? &cp->index : NULL};
        gd_join_spec spec;
        memset(&spec, 0, sizeof spec);
        spec.join_column_count = js->join_column_count;
        spec.proj_arity = js->proj_arity;
        spec.nfilters = js->nfilters;
        memcpy(spec.proj, js->proj, sizeof spec.proj);
        memcpy(spec.filters, js->filters, sizeof spec.filters);
        uint64_t total = join_run(&o, &in, &spec, NULL);
        arr out = {0};
        out.arity = js->proj_arity;
        out.data = (uint64_t*)malloc((total ? total : 1) * js->proj_arity * sizeof(uint64_t));
        out.n = join_run(&o, &in, &spec, out.data);
        arr_free(&chained);
        if (s + 1 == v->nsteps) {
            result = out;
            break;
        }
        chained = out;
        cur = chained;
    }
    arr_free(&permuted);
    return result;
}

static void append(arr* dst, const arr* rows) {
    if (rows->n == 0) return;
    dst->data = (uint64_t*)realloc(dst->data, (dst->n + rows->n) * dst->arity * sizeof(uint64_t));
    memcpy(dst->data + dst->n * dst->arity, rows->data, rows->n * rows->arity * sizeof(uint64_t));
    dst->n += rows->n;
}

/* merge_into_full, engine.hpp:520-533. */
static void merge_into_full(or_rel* st, const arr* gained) {
    uint64_t total = st->full.n + gained->n;
    uint64_t* buf = (uint64_t*)malloc((total ? total : 1) * st->arity * sizeof(uint64_t));
    or_merge_sorted(st->full.data, st->full.n, 1, gained->data, gained->n, 1, st->arity, total, buf);
    free(st->full.data);
    st->full.data = buf;
    st->full.n = total;
    st->dirty = 1;
}

static int plan_reads(const gd_rule_plan* p, uint32_t rel) {
    const gd_variant* v = &p->variants[0];
    if (v->src_rel == rel) return 1;
    for (uint32_t s = 0; s < v->nsteps; ++s)
        if (v->steps[s].inner_rel == rel) return 1;
    return 0;
}

/* seed, engine.hpp:137-179 (topological order: engine.hpp:322-353). */
int or_engine_seed(or_engine* e) {
    if (e->seeded) return fail(GD_ERR_LOGIC, "seed: called twice");
    uint32_t* nonrec = (uint32_t*)malloc((e->nplans + 1) * sizeof(uint32_t));
    uint32_t nn = 0;
    for (uint32_t i = 0; i < e->nplans; ++i)
        if (!e->plans[i].recursive) nonrec[nn++] = i;
    int* done = (int*)calloc(nn + 1, sizeof(int));
    uint32_t ndone = 0;
    while (ndone < nn) {
        int progressed = 0;
        for (uint32_t i = 0; i < nn; ++i) {
            if (done[i]) continue;
            int ready = 1;
            for (uint32_t j = 0; j < nn; ++j) {
                uint32_t h = e->plans[nonrec[j]].head_rel;
                if (!done[j] && j != i && !e->rels[h].is_edb && plan_reads(&e->plans[nonrec[i]], h))
                    ready = 0;
            }
            if (!ready) continue;
            done[i] = 1;
            ++ndone;
            progressed = 1;
            const gd_rule_plan* plan = &e->plans[nonrec[i]];
            const gd_variant* v = &plan->variants[0];
            for (uint32_t s = 0; s < v->nsteps; ++s)
                if (e->rels[v->steps[s].inner_rel].dirty) refresh_copies(e, &e->rels[v->steps[s].inner_rel]);
            arr rows = execute_chain(e, v);
            if (rows.n) {
                or_rel* head = &e->rels[plan->head_rel];
                arr fresh = {0};
                fresh.arity = head->arity;
                fresh.data = (uint64_t*)malloc(rows.n * head->arity * sizeof(uint64_t));
                fresh.n = canon(rows.data, rows.n, head->arity, fresh.data);
                arr gained = {0};
                gained.arity = head->arity;
                gained.data = (uint64_t*)malloc(fresh.n * head->arity * sizeof(uint64_t));
                gained.n = diff_rows(fresh.data, fresh.n, head->full.data, head->full.n, head->arity, gained.data);
                if (gained.n) merge_into_full(head, &gained);
                arr_free(&fresh);
                arr_free(&gained);
            }
            arr_free(&rows);
        }
        if (!progressed) {
            free(nonrec);
            free(done);
            return fail(GD_ERR_LOGIC, "nonrecursive rules form a dependency cycle");
        }
    }
    free(nonrec);
    free(done);
    for (uint32_t r = 0; r < e->nrels; ++r) {
        or_rel* st = &e->rels[r];
        if (st->is_edb) continue;
        arr_free(&st->delta);
        st->delta.data = (uint64_t*)malloc((st->full.n ? st->full.n : 1) * st->arity * sizeof(uint64_t));
        memcpy(st->delta.data, st->full.data, st->full.n * st->arity * sizeof(uint64_t));
        st->delta.n = st->full.n;
    }
    e->seeded = 1;
    return GD_OK;
}

static void push_hist(or_rel* st, uint64_t v) {
    if (st->nhist == st->caphist) {
        st->caphist = st->caphist ? 2 * st->caphist : 64;
        st->history = (uint64_t*)realloc(st->history, st->caphist * sizeof(uint64_t));
    }
    st->history[st->nhist++] = v;
}

static void push_log(or_rel* st, gd_iter_record rec) {
    if (st->nlog == st->caplog) {
        st->caplog = st->caplog ? 2 * st->caplog : 64;
        st->log = (gd_iter_record*)realloc(st->log, st->caplog * sizeof(gd_iter_record));
    }
    st->log[st->nlog++] = rec;
}

/* iterate_to_fixpoint, engine.hpp:181-257. */
int or_engine_iterate(or_engine* e) {
    if (!e->seeded) {
        int rc = or_engine_seed(e);
        if (rc) return rc;
    }
    uint32_t rec[64];
    uint32_t nrec = 0;
    for (uint32_t p = 0; p < e->nplans; ++p) {
        if (!e->plans[p].recursive) continue;
        uint32_t h = e->plans[p].head_rel, found = 0;
        for (uint32_t i = 0; i < nrec; ++i) found |= rec[i] == h;
        if (!found) rec[nrec++] = h;
    }
    for (;;) {
        int active = 0;
        for (uint32_t i = 0; i < nrec; ++i) active |= e->rels[rec[i]].delta.n > 0;
        if (!active) break;
        ++e->iterations;
        uint64_t delta_in[64];
        for (uint32_t i = 0; i < nrec; ++i) {
            delta_in[i] = e->rels[rec[i]].delta.n;
            push_hist(&e->rels[rec[i]], delta_in[i]);
        }
        for (uint32_t r = 0; r < e->nrels; ++r)
            if (e->rels[r].dirty) refresh_copies(e, &e->rels[r]);
        for (uint32_t p = 0; p < e->nplans; ++p) {
            const gd_rule_plan* plan = &e->plans[p];
            if (!plan->recursive) continue;
            or_rel* head = &e->rels[plan->head_rel];
            for (uint32_t v = 0; v < plan->nvariants; ++v) {
                const gd_variant* var = &plan->variants[v];
                if (var->src_version == GD_DELTA && e->rels[var->src_rel].delta.n == 0) continue;
                arr rows = execute_chain(e, var);
                append(&head->new_acc, &rows);
                arr_free(&rows);
            }
        }
        for (uint32_t i = 0; i < nrec; ++i) {
            or_rel* st = &e->rels[rec[i]];
            gd_iter_record log = {delta_in[i], st->new_acc.n, 0, 0, 0};
            arr fresh = {0};
            fresh.arity = st->arity;
            fresh.data = (uint64_t*)malloc((st->new_acc.n ? st->new_acc.n : 1) * st->arity * sizeof(uint64_t));
            fresh.n = canon(st->new_acc.data, st->new_acc.n, st->arity, fresh.data);
            arr_free(&st->new_acc);
            log.new_unique = fresh.n;
            arr_free(&st->delta);
            st->delta.arity = st->arity;
            st->delta.data = (uint64_t*)malloc((fresh.n ? fresh.n : 1) * st->arity * sizeof(uint64_t));
            st->delta.n = diff_rows(fresh.data, fresh.n, st->full.data, st->full.n, st->arity, st->delta.data);
            arr_free(&fresh);
            if (st->delta.n > 0) merge_into_full(st, &st->delta);
            log.delta_out = st->delta.n;
            log.full_after = st->full.n;
            push_log(st, log);
        }
    }
    return GD_OK;
}

int or_engine_run(or_engine* e) {
    int rc = or_engine_seed(e);
    return rc ? rc : or_engine_iterate(e);
}

uint64_t or_engine_iterations(const or_engine* e) { return e->iterations; }

int or_engine_relation_count(or_engine* e, uint32_t rel, uint64_t* n) {
    if (rel >= e->nrels) return fail(GD_ERR_USAGE, "unknown relation");
    *n = e->rels[rel].full.n;
    return GD_OK;
}

int or_engine_relation_download(or_engine* e, uint32_t rel, uint64_t* out,
                                uint64_t capacity_rows) {
    if (rel >= e->nrels) return fail(GD_ERR_USAGE, "unknown relation");
    const or_rel* st = &e->rels[rel];
    if (st->full.n > capacity_rows) return fail(GD_ERR_LOGIC, "capacity");
    memcpy(out, st->full.data, st->full.n * st->arity * sizeof(uint64_t));
    return GD_OK;
}

int or_engine_delta_history(or_engine* e, uint32_t rel, uint64_t* out,
                            uint64_t capacity, uint64_t* len) {
    const or_rel* st = &e->rels[rel];
    *len = st->nhist;
    for (uint64_t i = 0; i < st->nhist && i < capacity; ++i) out[i] = st->history[i];
    return GD_OK;
}

int or_engine_iter_log(or_engine* e, uint32_t rel, gd_iter_record* out,
                       uint64_t capacity, uint64_t* len) {
    const or_rel* st = &e->rels[rel];
    *len = st->nlog;
    for (uint64_t i = 0; i < st->nlog && i < capacity; ++i) out[i] = st->log[i];
    return GD_OK;
}
