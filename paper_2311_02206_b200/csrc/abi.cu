// abi.cu — the extern "C" boundary (include/gdlog_b200.h).  Exceptions from
// the device engine are mapped to gd_status codes here; nothing throws
// across the boundary.  The kernel-level entries reproduce the validation
// and error behaviour of the reference functions they replace (cited per
// entry) and run the same sm_100a kernels the engine uses.
#include "comm.h"
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "engine.h"
#include "tsv.h"
#include "gdlog_b200.h"
#include "ops.h"

using namespace gd;

struct gd_ctx {
    std::unique_ptr<Ctx> c;
    std::string err, phase;
};

struct gd_engine {
    gd_ctx* ctx;
    std::unique_ptr<Engine> e;
};

namespace {

thread_local std::string g_create_err;

template <typename F>
gd_status guard(gd_ctx* ctx, F&& f) {
    if (!ctx) return GD_ERR_INVALID_ARG;
    try {
        f();
        ctx->err.clear();
        ctx->phase.clear();
        return GD_OK;
    } catch (const Error& e) {
        ctx->err = e.what();
        ctx->phase = e.phase;
        if (e.code == GD_ERR_CUDA) cudaGetLastError();
        return e.code;
    } catch (const std::bad_alloc&) {
        ctx->err = "host allocation failed";
        ctx->phase = "other";
        return GD_ERR_BUDGET;
    } catch (const std::exception& e) {
        ctx->err = e.what();
        return GD_ERR_LOGIC;
    }
}

template <typename T>
DevBuf<T> upload(Ctx& c, const T* h, u64 count) {
    DevBuf<T> d(c, std::max<u64>(count, 1));
    c.h2d(d.p, h, count * sizeof(T));
    return d;
}

template <typename T>
void download(Ctx& c, T* h, const T* d, u64 count) {
    c.d2h(h, d, count * sizeof(T));
    c.sync();
}

template <typename F>
auto with_key(const Encoding& e, F&& f) {
    return e.key_words == 1 ? f(u64{}) : f(u128{});
}

void check_perm(const uint32_t* perm, uint32_t len, uint32_t arity, const char* who) {
    if (len != arity) throw_config(std::string(who) + ": permutation size mismatch");
    bool seen[GD_MAX_ARITY] = {false};
    for (uint32_t i = 0; i < len; ++i) {
        if (perm[i] >= arity || seen[perm[i]]) throw_config(std::string(who) + ": not a bijection");
        seen[perm[i]] = true;
    }
}

void validate_operand(const gd_operand& op, uint32_t oa, uint32_t ia) {  // ra.hpp:90-96
    if (op.kind == GD_OUTER_COL && op.column >= oa) throw_config("join: outer column out of range");
    if (op.kind == GD_INNER_COL && op.column >= ia) throw_config("join: inner column out of range");
}

void collect_constants(const gd_operand* ops, uint32_t n, std::vector<u64>& out) {
    for (uint32_t i = 0; i < n; ++i)
        if (ops[i].kind == GD_CONSTANT) out.push_back(ops[i].value);
}
void collect_constants(const gd_filter* f, uint32_t n, std::vector<u64>& out) {
    for (uint32_t i = 0; i < n; ++i) {
        collect_constants(&f[i].lhs, 1, out);
        collect_constants(&f[i].rhs, 1, out);
    }
}

DevJoin make_desc(Ctx& c, const Encoding& e, uint32_t jcc, uint32_t oa, uint32_t ia, uint32_t proj_arity,
                  const gd_operand* proj, uint32_t nfilters, const gd_filter* filters) {
    DevJoin jd;
    std::memset(&jd, 0, sizeof(jd));
    jd.jcc = jcc;
    jd.proj_arity = proj_arity;
    jd.nfilters = nfilters;
    jd.bits = e.bits;
    jd.outer_arity = oa;
    jd.outer_identity = 1;
    jd.inner_arity = ia;
    for (uint32_t i = 0; i < GD_MAX_ARITY; ++i) jd.outer_perm[i] = i;
    auto enc = [&](const gd_operand& o, bool* never) {
        DevOperand d{o.kind, o.column, 0};
        if (o.kind == GD_CONSTANT) {
            u64 v = 0;
            const bool ok = encode_value(c, e, o.value, &v);
            if (!ok && never) *never = true;
            d.value = v;
        }
        return d;
    };
    for (uint32_t k = 0; k < proj_arity; ++k) jd.proj[k] = enc(proj[k], nullptr);
    for (uint32_t f = 0; f < nfilters; ++f) {
        bool never = false;
        jd.filters[f].lhs = enc(filters[f].lhs, &never);
        jd.filters[f].rhs = enc(filters[f].rhs, &never);
        jd.filters[f].require_equal = filters[f].require_equal;
        jd.filters[f].never = never ? 1 : 0;
    }
    return jd;
}

// join_count / join_materialize shared body (ra.hpp:98-263).  Returns the
// total; when `out` is non-null writes exactly `cap` rows (checked).
u64 run_join(Ctx& c, const gd_container_view* outer, const gd_container_view* inner, const gd_join_spec* s,
             uint64_t* out, bool check_cap, uint64_t cap) {
    if (!outer || !inner || !s) throw Error(GD_ERR_INVALID_ARG, "join: null argument");
    const uint32_t oa = outer->arity, ia = inner->arity;
    auto check_view = [](const gd_container_view* v) {  // make_container / build_index
        if (v->index_prefix_len == 0) return;
        if (!v->canonical) throw_logic("make_container: array must be canonical");
        if (v->index_prefix_len > v->arity) throw_config("build_index: prefix_len must be in [1, arity]");
        if (!(v->load_factor > 0.0) || v->load_factor >= 1.0)
            throw_config("build_index: load factor must be in (0, 1)");
    };
    check_view(outer);
    check_view(inner);
    // validate_spec, ra.hpp:98-120
    if (s->proj_arity == 0) throw_config("join: projection must produce at least one column");
    if (s->proj_arity > GD_MAX_ARITY || s->nfilters > GD_MAX_FILTERS) throw_unsupported("join spec too wide");
    if (s->join_column_count > 0) {
        if (s->join_column_count > oa || s->join_column_count > ia)
            throw_config("join: join_column_count exceeds arity");
        if (inner->index_prefix_len == 0) throw_usage("join: inner relation has no index");
        if (inner->index_prefix_len != s->join_column_count)
            throw_usage("join: inner index prefix_len does not match join columns");
    }
    for (uint32_t k = 0; k < s->proj_arity; ++k) validate_operand(s->proj[k], oa, ia);
    for (uint32_t f = 0; f < s->nfilters; ++f) {
        validate_operand(s->filters[f].lhs, oa, ia);
        validate_operand(s->filters[f].rhs, oa, ia);
    }
    if (outer->n == 0 || inner->n == 0) {
        if (check_cap && cap != 0) throw_logic("join_materialize: output capacity mismatch");
        return 0;
    }
    DevBuf<u64> d_outer = upload(c, (const u64*)outer->rows, outer->n * oa);
    DevBuf<u64> d_inner = upload(c, (const u64*)inner->rows, inner->n * ia);
    std::vector<u64> consts;
    collect_constants(s->proj, s->proj_arity, consts);
    collect_constants(s->filters, s->nfilters, consts);
    EncodingOwner eo;
    choose_encoding(c, {{d_outer.p, outer->n * oa}, {d_inner.p, inner->n * ia}}, consts,
                    std::max(std::max(oa, ia), s->proj_arity), eo);
    const DevJoin jd = make_desc(c, eo.e, s->join_column_count, oa, ia, s->proj_arity, s->proj, s->nfilters,
                                 s->filters);
    return with_key(eo.e, [&](auto tag) -> u64 {
        using K = decltype(tag);
        const u32 bits = eo.e.bits;
        DevBuf<K> po(c, outer->n), pi(c, inner->n);
        pack_rows<K>(c, d_outer.p, outer->n, oa, eo.e, po.p);
        pack_rows<K>(c, d_inner.p, inner->n, ia, eo.e, pi.p);
        DevIndex<K> idx;
        IndexView<K> iv{};
        if (s->join_column_count > 0) {
            build_index<K>(c, pi.p, inner->n, ia, bits, s->join_column_count, inner->load_factor, idx);
            iv = IndexView<K>{idx.slots.p, idx.slot_count, pi.p, inner->n, ia, bits, s->join_column_count};
        }
        DevBuf<u64> row_start(c, outer->n), row_off(c, outer->n + 1);
        const u64 ncand = join_probe<K>(c, po.p, outer->n, jd, s->join_column_count ? &iv : nullptr, inner->n,
                                        row_start.p, row_off.p);
        DevBuf<K> res(c, std::max<u64>(ncand, 1));
        u64 total = ncand;
        if (s->nfilters) {
            DevBuf<K> raw(c, std::max<u64>(ncand, 1));
            DevBuf<uint8_t> flags(c, std::max<u64>(ncand, 1));
            join_materialize<K>(c, po.p, outer->n, pi.p, jd, row_start.p, row_off.p, ncand, raw.p, flags.p);
            total = compact_flagged<K>(c, raw.p, flags.p, ncand, res.p);
        } else if (out) {
            join_materialize<K>(c, po.p, outer->n, pi.p, jd, row_start.p, row_off.p, ncand, res.p, nullptr);
        }
        if (check_cap && cap != total) throw_logic("join_materialize: output capacity mismatch");
        if (out && total) {
            DevBuf<u64> un(c, total * s->proj_arity);
            unpack_rows<K>(c, res.p, total, s->proj_arity, eo.e, un.p);
            download(c, (u64*)out, un.p, total * s->proj_arity);
        }
        c.sync();
        return total;
    });
}

}  // namespace

extern "C" {

int gd_abi_version(void) { return GD_ABI_VERSION; }

gd_status gd_ctx_create(int device, void* stream, gd_ctx** out) {
    if (!out) return GD_ERR_INVALID_ARG;
    *out = nullptr;
    try {
        auto ctx = std::make_unique<gd_ctx>();
        ctx->c = std::make_unique<Ctx>(device, stream);
        *out = ctx.release();
        g_create_err.clear();
        return GD_OK;
    } catch (const Error& e) {
        g_create_err = e.what();
        cudaGetLastError();
        return e.code;
    } catch (const std::exception& e) {
        g_create_err = e.what();
        return GD_ERR_LOGIC;
    }
}

gd_status gd_ctx_destroy(gd_ctx* ctx) {
    if (!ctx) return GD_ERR_INVALID_ARG;
    try {
        if (ctx->c) ctx->c->sync();
    } catch (...) {
    }
    delete ctx;
    return GD_OK;
}

const char* gd_last_error(const gd_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }
const char* gd_last_error_phase(const gd_ctx* ctx) { return ctx ? ctx->phase.c_str() : ""; }
uint64_t gd_ctx_kernel_launches(const gd_ctx* ctx) { return ctx && ctx->c ? ctx->c->launches : 0; }
gd_status gd_ctx_synchronize(gd_ctx* ctx) {
    return guard(ctx, [&] { ctx->c->sync(); });
}
gd_status gd_ctx_trim(gd_ctx* ctx) {
    return guard(ctx, [&] { ctx->c->flush_cache(); });
}

void gd_device_config_default(gd_device_config* cfg) {
    if (cfg) *cfg = default_device_config();
}

gd_status gd_ctx_set_device_config(gd_ctx* ctx, const gd_device_config* cfg) {
    return guard(ctx, [&] {
        if (!cfg) throw Error(GD_ERR_INVALID_ARG, "null device config");
        if (cfg->size != sizeof(gd_device_config))
            throw_config("gd_device_config: size " + std::to_string(cfg->size) + " != " +
                         std::to_string(sizeof(gd_device_config)) + " (header/library mismatch)");
        if (cfg->loop_mode < GD_LOOP_GRAPH || cfg->loop_mode > GD_LOOP_BATCH) throw_config("loop_mode out of range");
        if (cfg->loop_batch == 0) throw_config("loop_batch must be positive");
        if (cfg->index_growth < 3) throw_config("index_growth must be at least 3");
        if (cfg->zone_slots < 1024 || cfg->zone_slots > 8192) throw_config("zone_slots must be in [1024, 8192]");
        if (cfg->dedup_part_slots < 1024 || (cfg->dedup_part_slots & (cfg->dedup_part_slots - 1)))
            throw_config("dedup_part_slots must be a power of two >= 1024");
        if (!(cfg->download_direct_frac >= 0.0 && cfg->download_direct_frac <= 1.0))
            throw_config("download_direct_frac must be in [0, 1]");
        if (cfg->download_chunk_rows < (1u << 16)) throw_config("download_chunk_rows must be at least 65536");
        if (cfg->download_delta > 2) throw_config("download_delta must be 0, 1 or 2");
        if (cfg->index_load_pct > 90) throw_config("index_load_pct must be at most 90");
        if (cfg->log_growth == 1 || cfg->log_growth > 64) throw_config("log_growth must be 0 or 2..64");
        if (cfg->sort_items != 4 && cfg->sort_items != 8 && cfg->sort_items != 16)
            throw_config("sort_items must be 4, 8 or 16");
        if (cfg->heavy_rows == 0) throw_config("heavy_rows must be positive");
        if (cfg->sort_digit_bits < 8 || cfg->sort_digit_bits > 10) throw_config("sort_digit_bits must be in [8, 10]");
        if (cfg->partition_exchange > GD_EXCHANGE_NCCL) throw_config("partition_exchange out of range");
        if (cfg->sort_pipeline < 0 || cfg->sort_pipeline > 4) throw_config("sort_pipeline must be in [0, 4]");
        if (cfg->peer_timeout_ms == 0) throw_config("peer_timeout_ms must be positive");
        if (cfg->insert_slots > 2) throw_config("insert_slots must be 0 (CAS first), 1 (load first) or 2 (batched)");
        if (cfg->l2_fetch_bytes && cfg->l2_fetch_bytes != 32 && cfg->l2_fetch_bytes != 64 &&
            cfg->l2_fetch_bytes != 128)
            throw_config("l2_fetch_bytes must be 0, 32, 64 or 128");
        if (cfg->l2_fetch_bytes && cfg->l2_fetch_bytes != ctx->c->cfg.l2_fetch_bytes) {
            GD_CUDA(cudaSetDevice(ctx->c->device));
            GD_CUDA(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, cfg->l2_fetch_bytes));
        }
        ctx->c->cfg = *cfg;
    });
}

gd_status gd_ctx_get_device_config(const gd_ctx* ctx, gd_device_config* cfg) {
    if (!ctx || !ctx->c || !cfg) return GD_ERR_INVALID_ARG;
    *cfg = ctx->c->cfg;
    return GD_OK;
}

gd_status gd_ctx_set_profiling(gd_ctx* ctx, int enable) {
    return guard(ctx, [&] { ctx->c->prof.on = enable != 0; });
}

gd_status gd_ctx_profile_read(gd_ctx* ctx, double* ms, uint64_t* launches, uint64_t* bytes) {
    return guard(ctx, [&] {
        ctx->c->sync();
        ctx->c->prof.resolve();
        for (int k = 0; k < KC_COUNT; ++k) {
            if (ms) ms[k] = ctx->c->prof.ms[k];
            if (launches) launches[k] = ctx->c->prof.launches[k];
            if (bytes) bytes[k] = ctx->c->prof.bytes[k];
        }
    });
}

gd_status gd_parse_facts(gd_ctx* ctx, const char* name, const char* text, uint64_t len, uint32_t arity,
                         uint64_t* out, uint64_t capacity_rows, uint64_t* count) {
    return guard(ctx, [&] {
        if ((!text && len) || !count) throw Error(GD_ERR_INVALID_ARG, "null argument");
        Ctx& c = *ctx->c;
        DevBuf<u64> rows;
        const u64 n = parse_facts_device(c, text, len, arity, name ? name : "<facts>", rows);
        *count = n;
        if (n > capacity_rows || (n && !out)) throw Error(GD_ERR_INVALID_ARG, "read_facts: output buffer too small");
        c.d2h(out, rows.p, n * arity * sizeof(u64));
        c.sync();
    });
}

gd_status gd_facts_all_integers(gd_ctx* ctx, const char* text, uint64_t len, int* result) {
    return guard(ctx, [&] {
        if ((!text && len) || !result) throw Error(GD_ERR_INVALID_ARG, "null argument");
        *result = facts_all_integers_device(*ctx->c, text, len) ? 1 : 0;
    });
}

gd_status gd_rows_to_tsv(gd_ctx* ctx, const uint64_t* rows, uint64_t n, uint32_t arity, char* out, uint64_t capacity,
                         uint64_t* len) {
    return guard(ctx, [&] {
        if ((!rows && n) || !len || arity == 0) throw Error(GD_ERR_INVALID_ARG, "bad argument");
        Ctx& c = *ctx->c;
        DevBuf<u64> d(c, std::max<u64>(n * arity, 1));
        c.h2d(d.p, rows, n * arity * sizeof(u64));
        *len = rows_to_tsv_device(c, d.p, n, arity, out, capacity);
    });
}

gd_status gd_ctx_transfer_bytes(gd_ctx* ctx, uint64_t* h2d, uint64_t* d2h) {
    return guard(ctx, [&] {
        if (h2d) *h2d = ctx->c->h2d_bytes;
        if (d2h) *d2h = ctx->c->d2h_bytes;
    });
}

gd_status gd_ctx_host_counters(gd_ctx* ctx, double* alloc_seconds, uint64_t* allocs, double* sync_seconds,
                               uint64_t* syncs) {
    return guard(ctx, [&] {
        if (alloc_seconds) *alloc_seconds = ctx->c->alloc_seconds;
        if (allocs) *allocs = ctx->c->alloc_count;
        if (sync_seconds) *sync_seconds = ctx->c->sync_seconds;
        if (syncs) *syncs = ctx->c->sync_count;
    });
}

gd_status gd_ctx_profile_reset(gd_ctx* ctx) {
    return guard(ctx, [&] {
        ctx->c->sync();
        ctx->c->prof.resolve();
        ctx->c->prof.reset();
    });
}

// ---- kernel-level entries -------------------------------------------

gd_status gd_prefix_hash(gd_ctx* ctx, const uint64_t* rows, uint64_t n, uint32_t arity, uint32_t ncols,
                         uint64_t* out) {
    return guard(ctx, [&] {
        Ctx& c = *ctx->c;
        if (ncols > arity || arity > GD_MAX_ARITY) throw_config("prefix_hash: column count out of range");
        if (n == 0) return;
        DevBuf<u64> d = upload(c, (const u64*)rows, n * arity);
        DevBuf<u64> h(c, n);
        prefix_hash_rows(c, d.p, n, arity, ncols, h.p);
        download(c, (u64*)out, h.p, n);
    });
}

gd_status gd_canonicalize(gd_ctx* ctx, const uint64_t* rows, uint64_t n, uint32_t arity, uint64_t* out,
                          uint64_t* out_n) {
    return guard(ctx, [&] {  // tuple_array.hpp:73-133
        Ctx& c = *ctx->c;
        if (arity == 0) throw_logic("canonicalize: arity must be positive");
        if (arity > GD_MAX_ARITY) throw_unsupported("arity above 8");
        *out_n = 0;
        if (n == 0) return;
        DevBuf<u64> d = upload(c, (const u64*)rows, n * arity);
        DevBuf<u64> res;
        const u64 m = canonicalize_rows(c, d.p, n, arity, res);
        download(c, (u64*)out, res.p, m * arity);
        *out_n = m;
    });
}

gd_status gd_sort_keys_device(gd_ctx* ctx, uint64_t* d_keys, uint64_t* d_tmp, uint64_t n, uint32_t nbits,
                              int* in_tmp) {
    return guard(ctx, [&] {
        if (!d_keys || !d_tmp || !in_tmp) throw Error(GD_ERR_INVALID_ARG, "sort_keys_device: null pointer");
        if (nbits > 64) throw_config("sort_keys_device: nbits above 64");
        u64* r = radix_sort<u64>(*ctx->c, (u64*)d_keys, (u64*)d_tmp, n, nbits);
        *in_tmp = r == (u64*)d_tmp && r != (u64*)d_keys;
    });
}

gd_status gd_permute_columns(gd_ctx* ctx, const uint64_t* rows, uint64_t n, uint32_t arity, int canonical,
                             const uint32_t* perm, uint32_t perm_len, uint64_t* out, uint64_t* out_n) {
    return guard(ctx, [&] {  // ra.hpp:426-454
        Ctx& c = *ctx->c;
        if (!canonical) throw_logic("permute_columns: input must be canonical");
        check_perm(perm, perm_len, arity, "permute_columns");
        *out_n = 0;
        if (n == 0) return;
        DevBuf<u64> d = upload(c, (const u64*)rows, n * arity);
        bool ident = true;
        for (uint32_t i = 0; i < arity; ++i) ident &= perm[i] == i;
        if (ident) {
            download(c, (u64*)out, d.p, n * arity);
            *out_n = n;
            return;
        }
        DevBuf<u64> p(c, n * arity);
        permute_raw_rows(c, d.p, n, arity, perm, p.p);
        DevBuf<u64> res;
        const u64 m = canonicalize_rows(c, p.p, n, arity, res);
        download(c, (u64*)out, res.p, m * arity);
        *out_n = m;
    });
}

gd_status gd_group_starts(gd_ctx* ctx, const uint64_t* rows, uint64_t n, uint32_t arity, int canonical,
                          uint32_t prefix_len, uint64_t* out_starts, uint64_t* out_count) {
    return guard(ctx, [&] {  // index_map.hpp:46-66
        (void)canonical;
        Ctx& c = *ctx->c;
        if (prefix_len == 0 || prefix_len > arity) throw_config("group_starts: prefix_len must be in [1, arity]");
        *out_count = 0;
        if (n == 0) return;
        DevBuf<u64> d = upload(c, (const u64*)rows, n * arity);
        EncodingOwner eo;
        choose_encoding(c, {{d.p, n * arity}}, {}, arity, eo);
        with_key(eo.e, [&](auto tag) {
            using K = decltype(tag);
            DevBuf<K> pk(c, n);
            pack_rows<K>(c, d.p, n, arity, eo.e, pk.p);
            DevBuf<u64> gs;
            const u64 g = group_starts<K>(c, pk.p, n, arity, eo.e.bits, prefix_len, gs);
            download(c, (u64*)out_starts, gs.p, g);
            *out_count = g;
            return 0;
        });
    });
}

gd_status gd_index_lookup(gd_ctx* ctx, const uint64_t* rows, uint64_t n, uint32_t arity, int canonical,
                          uint32_t prefix_len, double load_factor, const uint64_t* keys, uint64_t nkeys,
                          uint32_t key_len, uint64_t* out_start, uint64_t* out_count, uint64_t* out_slot_count,
                          uint64_t* out_occupied) {
    return guard(ctx, [&] {  // index_map.hpp:74-124 + container.hpp:52-89
        Ctx& c = *ctx->c;
        if (!canonical) throw_logic("build_index: tuples must be canonical");
        if (prefix_len == 0 || prefix_len > arity) throw_config("build_index: prefix_len must be in [1, arity]");
        if (!(load_factor > 0.0) || load_factor >= 1.0) throw_config("build_index: load factor must be in (0, 1)");
        if (key_len != prefix_len)
            throw_usage("range_lookup: prefix length " + std::to_string(key_len) +
                        " does not match index prefix_len " + std::to_string(prefix_len));
        DevBuf<u64> d = upload(c, (const u64*)rows, n * arity);
        DevBuf<u64> dk = upload(c, (const u64*)keys, nkeys * key_len);
        EncodingOwner eo;
        choose_encoding(c, {{d.p, n * arity}}, {}, arity, eo);
        with_key(eo.e, [&](auto tag) {
            using K = decltype(tag);
            DevBuf<K> pk(c, std::max<u64>(n, 1));
            pack_rows<K>(c, d.p, n, arity, eo.e, pk.p);
            DevIndex<K> idx;
            build_index<K>(c, pk.p, n, arity, eo.e.bits, prefix_len, load_factor, idx);
            *out_slot_count = idx.logical_slots;
            *out_occupied = idx.groups;
            if (nkeys) {
                DevBuf<K> pkeys(c, nkeys);
                DevBuf<uint8_t> valid(c, nkeys);
                pack_keys_checked<K>(c, dk.p, nkeys, key_len, eo.e, pkeys.p, valid.p);
                DevBuf<u64> st(c, nkeys), ct(c, nkeys);
                IndexView<K> iv{idx.slots.p, idx.slot_count, pk.p, n, arity, eo.e.bits, prefix_len};
                index_lookup<K>(c, iv, pkeys.p, valid.p, nkeys, st.p, ct.p);
                download(c, (u64*)out_start, st.p, nkeys);
                download(c, (u64*)out_count, ct.p, nkeys);
            }
            c.sync();
            return 0;
        });
    });
}

gd_status gd_join_count(gd_ctx* ctx, const gd_container_view* outer, const gd_container_view* inner,
                        const gd_join_spec* spec, uint64_t* out_total) {
    return guard(ctx, [&] { *out_total = run_join(*ctx->c, outer, inner, spec, nullptr, false, 0); });
}

gd_status gd_join_materialize(gd_ctx* ctx, const gd_container_view* outer, const gd_container_view* inner,
                              const gd_join_spec* spec, uint64_t* out, uint64_t out_capacity_rows) {
    return guard(ctx, [&] { run_join(*ctx->c, outer, inner, spec, out, true, out_capacity_rows); });
}

gd_status gd_select_project(gd_ctx* ctx, const uint64_t* rows, uint64_t n, uint32_t arity, const gd_operand* proj,
                            uint32_t proj_arity, const gd_filter* filters, uint32_t nfilters, uint64_t* out,
                            uint64_t* out_n) {
    return guard(ctx, [&] {  // ra.hpp:267-293
        Ctx& c = *ctx->c;
        for (uint32_t k = 0; k < proj_arity; ++k)
            if (proj[k].kind == GD_INNER_COL) throw_logic("select_project: inner operand");
        for (uint32_t f = 0; f < nfilters; ++f)
            if (filters[f].lhs.kind == GD_INNER_COL || filters[f].rhs.kind == GD_INNER_COL)
                throw_logic("select_project: inner operand");
        for (uint32_t k = 0; k < proj_arity; ++k) validate_operand(proj[k], arity, 0);
        if (proj_arity == 0 || proj_arity > GD_MAX_ARITY) throw_unsupported("select_project: projection arity");
        *out_n = 0;
        if (n == 0) return;
        DevBuf<u64> d = upload(c, (const u64*)rows, n * arity);
        std::vector<u64> consts;
        collect_constants(proj, proj_arity, consts);
        collect_constants(filters, nfilters, consts);
        EncodingOwner eo;
        choose_encoding(c, {{d.p, n * arity}}, consts, std::max(arity, proj_arity), eo);
        const DevJoin jd = make_desc(c, eo.e, 0, arity, 0, proj_arity, proj, nfilters, filters);
        with_key(eo.e, [&](auto tag) {
            using K = decltype(tag);
            DevBuf<K> pk(c, n), res(c, n);
            pack_rows<K>(c, d.p, n, arity, eo.e, pk.p);
            const u64 m = select_project<K>(c, pk.p, n, jd, res.p);
            DevBuf<u64> un(c, std::max<u64>(m * proj_arity, 1));
            unpack_rows<K>(c, res.p, m, proj_arity, eo.e, un.p);
            download(c, (u64*)out, un.p, m * proj_arity);
            *out_n = m;
            return 0;
        });
    });
}

gd_status gd_merge_sorted(gd_ctx* ctx, const uint64_t* full, uint64_t nf, int full_canonical, const uint64_t* delta,
                          uint64_t nd, int delta_canonical, uint32_t arity, uint64_t buffer_rows, uint64_t* out) {
    return guard(ctx, [&] {  // ra.hpp:299-381
        Ctx& c = *ctx->c;
        if (!full_canonical || !delta_canonical) throw_logic("merge_sorted: inputs must be canonical");
        if (buffer_rows < nf + nd) throw_logic("merge_sorted: buffer too small");
        if (nf + nd == 0) return;
        DevBuf<u64> df = upload(c, (const u64*)full, nf * arity);
        DevBuf<u64> dd = upload(c, (const u64*)delta, nd * arity);
        EncodingOwner eo;
        choose_encoding(c, {{df.p, nf * arity}, {dd.p, nd * arity}}, {}, arity, eo);
        with_key(eo.e, [&](auto tag) {
            using K = decltype(tag);
            DevBuf<K> pf(c, std::max<u64>(nf, 1)), pd(c, std::max<u64>(nd, 1)), res(c, nf + nd);
            pack_rows<K>(c, df.p, nf, arity, eo.e, pf.p);
            pack_rows<K>(c, dd.p, nd, arity, eo.e, pd.p);
            if (merge_disjoint<K>(c, pf.p, nf, pd.p, nd, res.p, true))
                throw_logic("merge_sorted: inputs are not disjoint");
            DevBuf<u64> un(c, (nf + nd) * arity);
            unpack_rows<K>(c, res.p, nf + nd, arity, eo.e, un.p);
            download(c, (u64*)out, un.p, (nf + nd) * arity);
            return 0;
        });
    });
}

gd_status gd_difference(gd_ctx* ctx, const uint64_t* new_rows, uint64_t nn, int new_canonical,
                        const uint64_t* full, uint64_t nf, int full_canonical, uint32_t arity, uint64_t* out,
                        uint64_t* out_n) {
    return guard(ctx, [&] {  // ra.hpp:386-422
        Ctx& c = *ctx->c;
        if (!new_canonical || !full_canonical) throw_logic("difference: inputs must be canonical");
        *out_n = 0;
        if (nn == 0) return;
        DevBuf<u64> dn = upload(c, (const u64*)new_rows, nn * arity);
        DevBuf<u64> df = upload(c, (const u64*)full, nf * arity);
        EncodingOwner eo;
        choose_encoding(c, {{dn.p, nn * arity}, {df.p, nf * arity}}, {}, arity, eo);
        with_key(eo.e, [&](auto tag) {
            using K = decltype(tag);
            DevBuf<K> pn(c, nn), pf(c, std::max<u64>(nf, 1)), res(c, nn);
            pack_rows<K>(c, dn.p, nn, arity, eo.e, pn.p);
            pack_rows<K>(c, df.p, nf, arity, eo.e, pf.p);
            const MergeResult mr = difference_sorted<K>(c, pf.p, nf, pn.p, nn, res.p);
            DevBuf<u64> un(c, std::max<u64>(mr.delta_n * arity, 1));
            unpack_rows<K>(c, res.p, mr.delta_n, arity, eo.e, un.p);
            download(c, (u64*)out, un.p, mr.delta_n * arity);
            *out_n = mr.delta_n;
            return 0;
        });
    });
}

// ---- engine ----------------------------------------------------------

gd_status gd_engine_create(gd_ctx* ctx, const gd_engine_config* cfg, uint32_t nrels, const uint32_t* arities,
                           const uint32_t* is_edb, const char* const* names, gd_engine** out) {
    return guard(ctx, [&] {
        // an empty program (no relations) may pass null arrays
        if (!out || (nrels && (!arities || !is_edb))) throw Error(GD_ERR_INVALID_ARG, "gd_engine_create: null argument");
        gd_engine_config def{UINT64_MAX, 1, 5, 0.8, 0, 0, 0};
        auto e = std::make_unique<gd_engine>();
        e->ctx = ctx;
        e->e = std::make_unique<Engine>(*ctx->c, cfg ? *cfg : def, nrels, arities, is_edb, names);
        *out = e.release();
    });
}

gd_status gd_engine_destroy(gd_engine* eng) {
    if (!eng) return GD_ERR_INVALID_ARG;
    try {
        eng->ctx->c->sync();
    } catch (...) {
    }
    delete eng;
    return GD_OK;
}

#define ENG_GUARD(body)                             \
    if (!eng) return GD_ERR_INVALID_ARG;            \
    return guard(eng->ctx, [&] { body; })

gd_status gd_engine_set_plans(gd_engine* eng, const gd_rule_plan* plans, uint32_t nplans) {
    ENG_GUARD(eng->e->set_plans(plans, nplans));
}
gd_status gd_engine_load_edb(gd_engine* eng, uint32_t rel, const uint64_t* rows, uint64_t n, int canonical) {
    ENG_GUARD(eng->e->load_edb(rel, (const u64*)rows, n, canonical != 0, false));
}
gd_status gd_engine_load_edb_device(gd_engine* eng, uint32_t rel, const uint64_t* d_rows, uint64_t n,
                                    int canonical) {
    ENG_GUARD(eng->e->load_edb(rel, (const u64*)d_rows, n, canonical != 0, true));
}
gd_status gd_engine_load_edb_tsv(gd_engine* eng, uint32_t rel, const char* name, const char* text, uint64_t len) {
    ENG_GUARD({
        if (!text && len) throw Error(GD_ERR_INVALID_ARG, "null text");
        Engine& E = *eng->e;
        E.check_rel(rel);
        if (!E.info_[rel].is_edb)
            throw_load("load_edb: '" + E.info_[rel].name + "' is not a declared EDB relation");
        DevBuf<u64> rows;
        const u64 n = parse_facts_device(E.c, text, len, E.info_[rel].arity, name ? name : E.info_[rel].name, rows);
        E.load_edb(rel, rows.p, n, true, true);
    });
}
gd_status gd_engine_relation_tsv(gd_engine* eng, uint32_t rel, char* out, uint64_t capacity, uint64_t* len) {
    ENG_GUARD({
        Engine& E = *eng->e;
        const u64 n = E.relation_count(rel);
        const u32 ar = E.rel(rel).arity;
        DevBuf<u64> rows(E.c, std::max<u64>(n * ar, 1));
        if (n) E.relation_download(rel, rows.p, n, true);
        *len = rows_to_tsv_device(E.c, rows.p, n, ar, out, capacity);
    });
}
gd_status gd_engine_seed(gd_engine* eng) { ENG_GUARD(eng->e->seed()); }
gd_status gd_engine_iterate(gd_engine* eng) { ENG_GUARD(eng->e->iterate()); }
gd_status gd_engine_run(gd_engine* eng) { ENG_GUARD(eng->e->run()); }
gd_status gd_engine_relation_count(gd_engine* eng, uint32_t rel, uint64_t* n) {
    ENG_GUARD(*n = eng->e->relation_count(rel));
}
gd_status gd_engine_relation_download(gd_engine* eng, uint32_t rel, uint64_t* out, uint64_t capacity_rows) {
    ENG_GUARD(eng->e->relation_download(rel, (u64*)out, capacity_rows, false));
}
gd_status gd_engine_relation_download_device(gd_engine* eng, uint32_t rel, uint64_t* d_out,
                                             uint64_t capacity_rows) {
    ENG_GUARD(eng->e->relation_download(rel, (u64*)d_out, capacity_rows, true));
}
gd_status gd_engine_relation_digest(gd_engine* eng, uint32_t rel, uint64_t* digest) {
    ENG_GUARD(*digest = eng->e->relation_digest(rel));
}
gd_status gd_engine_stats(gd_engine* eng, gd_run_stats* out) { ENG_GUARD(eng->e->fill_stats(out)); }
gd_status gd_engine_accountant(gd_engine* eng, uint64_t current[3], uint64_t* peak, uint64_t* peak_temp,
                               uint64_t* events, uint64_t* budget) {
    ENG_GUARD({
        const Accountant& a = eng->e->acct;
        if (current)
            for (int k = 0; k < 3; ++k) current[k] = a.current(static_cast<Accountant::Cat>(k));
        if (peak) *peak = a.peak();
        if (peak_temp) *peak_temp = a.peak_temp();
        if (events) *events = a.events();
        if (budget) *budget = a.budget();
    });
}
gd_status gd_engine_delta_history(gd_engine* eng, uint32_t rel, uint64_t* out, uint64_t capacity, uint64_t* len) {
    ENG_GUARD({
        const auto& h = eng->e->rel(rel).history;
        *len = h.size();
        for (size_t i = 0; i < h.size() && i < capacity; ++i) out[i] = h[i];
    });
}
gd_status gd_engine_iter_log(gd_engine* eng, uint32_t rel, gd_iter_record* out, uint64_t capacity, uint64_t* len) {
    ENG_GUARD({
        const auto& h = eng->e->rel(rel).log;
        *len = h.size();
        for (size_t i = 0; i < h.size() && i < capacity; ++i) out[i] = h[i];
    });
}
gd_status gd_engine_encoding(gd_engine* eng, uint32_t* bits, uint32_t* key_words, uint32_t* dictionary) {
    ENG_GUARD(eng->e->encoding(bits, key_words, dictionary));
}
gd_status gd_engine_set_partition(gd_engine* eng, uint32_t rank, uint32_t nranks) {
    ENG_GUARD(eng->e->set_partition(rank, nranks));
}
gd_status gd_engine_exchange_words(gd_engine* eng, uint32_t* words) { ENG_GUARD(*words = eng->e->exchange_words()); }
gd_status gd_engine_partition_begin(gd_engine* eng, uint64_t* send_counts, const void** d_send) {
    ENG_GUARD(eng->e->partition_begin((u64*)send_counts, d_send));
}
gd_status gd_engine_partition_end(gd_engine* eng, const void* d_recv, uint64_t recv_rows, uint64_t* local_delta) {
    ENG_GUARD(eng->e->partition_end(d_recv, recv_rows, (u64*)local_delta));
}
gd_status gd_engine_partition_finish(gd_engine* eng) { ENG_GUARD(eng->e->partition_finish()); }

struct gd_comm {
    gd::Comm c;
    std::unique_ptr<gd::Transport> t;
};

struct gd_loopback_hub {
    gd::LoopbackHub hub;
    explicit gd_loopback_hub(uint32_t p) : hub(p) {}
};

gd_status gd_nccl_unique_id(uint8_t id[128]) {
    if (!id) return GD_ERR_INVALID_ARG;
    ncclUniqueId u;
    try {
        if (gd::nccl().get_unique_id(&u) != ncclSuccess) return GD_ERR_NCCL;
    } catch (const gd::Error&) {
        return GD_ERR_NCCL;
    }
    static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, &u, sizeof(u));
    return GD_OK;
}

gd_status gd_nccl_comm_create(gd_ctx* ctx, const uint8_t id[128], uint32_t nranks, uint32_t rank, gd_comm** out) {
    if (!ctx || !id || !out || nranks == 0 || rank >= nranks) return GD_ERR_INVALID_ARG;
    return guard(ctx, [&] {
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        GD_CUDA(cudaSetDevice(ctx->c->device));
        auto t = std::make_unique<gd::NcclTransport>();
        t->nranks = nranks;
        t->rank = rank;
        gd::nccl_check(gd::nccl().comm_init_rank(&t->comm, (int)nranks, u, (int)rank), "ncclCommInitRank");
        auto* cm = new gd_comm;
        cm->c = gd::Comm{t.get(), nranks, rank};
        cm->t = std::move(t);
        *out = cm;
    });
}

gd_status gd_loopback_hub_create(uint32_t nranks, gd_loopback_hub** out) {
    if (!out || nranks == 0) return GD_ERR_INVALID_ARG;
    *out = new gd_loopback_hub(nranks);
    return GD_OK;
}

gd_status gd_loopback_hub_destroy(gd_loopback_hub* hub) {
    if (!hub) return GD_ERR_INVALID_ARG;
    delete hub;
    return GD_OK;
}

gd_status gd_loopback_comm_create(gd_loopback_hub* hub, uint32_t rank, gd_comm** out) {
    if (!hub || !out || rank >= hub->hub.P) return GD_ERR_INVALID_ARG;
    auto t = std::make_unique<gd::LoopbackTransport>();
    t->hub = &hub->hub;
    t->nranks = hub->hub.P;
    t->rank = rank;
    auto* cm = new gd_comm;
    cm->c = gd::Comm{t.get(), hub->hub.P, rank};
    cm->t = std::move(t);
    *out = cm;
    return GD_OK;
}

gd_status gd_nccl_comm_destroy(gd_comm* comm) {
    if (!comm) return GD_ERR_INVALID_ARG;
    delete comm;
    return GD_OK;
}

gd_status gd_engine_run_partitioned(gd_engine* eng, gd_comm* comm, uint64_t max_iters, uint64_t* iterations) {
    if (!comm) return GD_ERR_INVALID_ARG;
    if (!eng) return GD_ERR_INVALID_ARG;
    const gd_status st = guard(eng->ctx, [&] {
        const u64 it = eng->e->partition_run(comm->c, max_iters ? max_iters : ~0ull);
        if (iterations) *iterations = it;
    });
    // a failed rank must not leave its peers waiting in a host-side
    // collective of the transport (loopback ranks share one process)
    if (st != GD_OK) comm->t->abort();
    return st;
}

}  // extern "C"
