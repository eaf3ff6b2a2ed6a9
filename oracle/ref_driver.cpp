// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin C-ABI shim around the UNMODIFIED reference engine (the header-only
// C++20 `arraylog` library under /root/reference/proj/include).  It is
// compiled by oracle/Makefile straight from the reference headers into
// oracle/_ref/libarraylog_ref.so and is used only by tests/, by
// __graft_entry__.smoke() and by bench.py's CPU-baseline / `--impl reference`
// legs — never by the product path (paper_2311_02206_b200/).
//
// Every entry mirrors the gd_* entry of include/gdlog_b200.h with the same
// arguments, so parity tests can call both sides with one argument list.
// Nothing here re-implements the algorithm: each function forwards to the
// reference function it is named after.

#include <cstdint>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include <random>

#include "arraylog/arraylog.hpp"
#include "gdlog_b200.h"
#include "oracles.hpp"  // reference tests/oracles.hpp: seeded corpus generators

using namespace arraylog;

namespace {

thread_local std::string g_err;
thread_local std::string g_phase;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

template <typename F>
int guard(F&& f) {
    try {
        f();
        g_err.clear();
        g_phase.clear();
        return GD_OK;
    } catch (const budget_error& e) {
        g_phase = e.phase();
        return fail(GD_ERR_BUDGET, e.what());
    } catch (const config_error& e) {
        return fail(GD_ERR_CONFIG, e.what());
    } catch (const usage_error& e) {
        return fail(GD_ERR_USAGE, e.what());
    } catch (const load_error& e) {
        return fail(GD_ERR_LOAD, e.what());
    } catch (const plan_error& e) {
        return fail(GD_ERR_PLAN, e.what());
    } catch (const std::logic_error& e) {
        return fail(GD_ERR_LOGIC, e.what());
    } catch (const std::exception& e) {
        return fail(GD_ERR_LOGIC, e.what());
    }
}

tuple_array make_rows(const uint64_t* rows, uint64_t n, uint32_t arity,
                      bool canonical) {
    std::vector<value_t> d(rows, rows + n * arity);
    return tuple_array(arity, std::move(d), canonical);
}

operand to_operand(const gd_operand& o) {
    switch (o.kind) {
        case GD_OUTER_COL: return operand::outer(o.column);
        case GD_INNER_COL: return operand::inner(o.column);
        default: return operand::constant(o.value);
    }
}

row_filter to_filter(const gd_filter& f) {
    return {to_operand(f.lhs), to_operand(f.rhs), f.require_equal != 0};
}

gd_operand from_operand(const operand& o) {
    gd_operand g{};
    g.kind = o.from == operand::kind::outer_col   ? GD_OUTER_COL
             : o.from == operand::kind::inner_col ? GD_INNER_COL
                                                  : GD_CONSTANT;
    g.column = o.column;
    g.value = o.value;
    return g;
}

gd_filter from_filter(const row_filter& f) {
    gd_filter g{};
    g.lhs = from_operand(f.lhs);
    g.rhs = from_operand(f.rhs);
    g.require_equal = f.require_equal ? 1 : 0;
    return g;
}

relation_container make_view(const gd_container_view* v) {
    tuple_array t = make_rows(v->rows, v->n, v->arity, v->canonical != 0);
    if (v->index_prefix_len == 0) {
        relation_container c;
        c.tuples = std::move(t);
        c.permutation = identity_permutation(v->arity);
        return c;
    }
    return make_container(std::move(t), {}, v->index_prefix_len,
                          v->load_factor, 1);
}

join_spec to_spec(const gd_join_spec* s, const relation_container* o,
                  const relation_container* i) {
    join_spec spec;
    spec.join_column_count = s->join_column_count;
    spec.outer = o;
    spec.inner = i;
    for (uint32_t c = 0; c < s->proj_arity; ++c)
        spec.projection.sources.push_back(to_operand(s->proj[c]));
    for (uint32_t f = 0; f < s->nfilters; ++f)
        spec.filters.push_back(to_filter(s->filters[f]));
    return spec;
}

engine_config to_config(const gd_engine_config* c) {
    engine_config cfg;
    if (!c) return cfg;
    cfg.memory_budget_bytes = c->memory_budget_bytes == UINT64_MAX
                                  ? memory_accountant::unlimited
                                  : static_cast<std::size_t>(c->memory_budget_bytes);
    cfg.ebm_enabled = c->ebm_enabled != 0;
    cfg.alpha = c->alpha;
    cfg.load_factor = c->load_factor;
    cfg.workers = c->workers;
    cfg.stride_rows = c->stride_rows;
    return cfg;
}

struct ref_engine {
    program prog;
    std::unique_ptr<engine> eng;
    std::vector<std::string> names;  // relation id -> name
};

program load_program(const char* source) {
    std::string s(source);
    if (is_builtin_program(s)) return builtin_program(s);
    auto r = parse_program(s);
    if (!r.ok())
        throw plan_error("program failed to parse: " +
                         r.diagnostics.front().message);
    return std::move(r.prog);
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
const char* ref_last_error_phase(void) { return g_phase.c_str(); }

int ref_prefix_hash(const uint64_t* rows, uint64_t n, uint32_t arity,
                    uint32_t ncols, uint64_t* out) {
    return guard([&] {
        for (uint64_t i = 0; i < n; ++i)
            out[i] = slot_key({rows + i * arity, ncols});
    });
}

int ref_canonicalize(const uint64_t* rows, uint64_t n, uint32_t arity,
                     uint32_t workers, uint64_t* out, uint64_t* out_n) {
    return guard([&] {
        tuple_array c = canonicalize(make_rows(rows, n, arity, false), workers);
        std::memcpy(out, c.data.data(), c.data.size() * sizeof(uint64_t));
        *out_n = c.count();
    });
}

int ref_permute_columns(const uint64_t* rows, uint64_t n, uint32_t arity,
                        int canonical, const uint32_t* perm, uint32_t perm_len,
                        uint64_t* out, uint64_t* out_n) {
    return guard([&] {
        std::vector<uint32_t> p(perm, perm + perm_len);
        tuple_array c = permute_columns(make_rows(rows, n, arity, canonical != 0),
                                        p, 1);
        std::memcpy(out, c.data.data(), c.data.size() * sizeof(uint64_t));
        *out_n = c.count();
    });
}

int ref_group_starts(const uint64_t* rows, uint64_t n, uint32_t arity,
                     int canonical, uint32_t prefix_len, uint64_t* out_starts,
                     uint64_t* out_count) {
    return guard([&] {
        auto t = make_rows(rows, n, arity, canonical != 0);
        auto s = detail::group_starts(t, prefix_len, 1);
        std::memcpy(out_starts, s.data(), s.size() * sizeof(uint64_t));
        *out_count = s.size();
    });
}

// build_index + range_lookup; also exports the raw slot array so tests can
// pin the CPU layout (key_hash, offset pairs) if they want to.
int ref_index_lookup(const uint64_t* rows, uint64_t n, uint32_t arity,
                     int canonical, uint32_t prefix_len, double load_factor,
                     const uint64_t* keys, uint64_t nkeys, uint32_t key_len,
                     uint64_t* out_start, uint64_t* out_count,
                     uint64_t* out_slot_count, uint64_t* out_occupied) {
    return guard([&] {
        auto c = make_container(make_rows(rows, n, arity, canonical != 0), {},
                                prefix_len, load_factor, 1);
        for (uint64_t i = 0; i < nkeys; ++i) {
            row_range r = range_lookup(
                c, std::span<const value_t>(keys + i * key_len, key_len));
            out_start[i] = r.start;
            out_count[i] = r.count;
        }
        *out_slot_count = c.index->slot_count();
        *out_occupied = c.index->occupied();
    });
}

int ref_join_count(const gd_container_view* outer,
                   const gd_container_view* inner, const gd_join_spec* s,
                   uint32_t workers, uint64_t stride, uint64_t* out_total) {
    return guard([&] {
        auto o = make_view(outer);
        auto i = make_view(inner);
        *out_total = join_count(to_spec(s, &o, &i), workers, stride);
    });
}

int ref_join_materialize(const gd_container_view* outer,
                         const gd_container_view* inner, const gd_join_spec* s,
                         uint32_t workers, uint64_t stride, uint64_t* out,
                         uint64_t out_capacity_rows) {
    return guard([&] {
        auto o = make_view(outer);
        auto i = make_view(inner);
        tuple_array res(s->proj_arity ? s->proj_arity : 1);
        res.data.resize(out_capacity_rows * s->proj_arity);
        join_materialize(to_spec(s, &o, &i), res, workers, stride);
        std::memcpy(out, res.data.data(), res.data.size() * sizeof(uint64_t));
    });
}

int ref_select_project(const uint64_t* rows, uint64_t n, uint32_t arity,
                       const gd_operand* proj, uint32_t proj_arity,
                       const gd_filter* filters, uint32_t nfilters,
                       uint64_t* out, uint64_t* out_n) {
    return guard([&] {
        relation_container c;
        c.tuples = make_rows(rows, n, arity, false);
        column_map m;
        for (uint32_t k = 0; k < proj_arity; ++k)
            m.sources.push_back(to_operand(proj[k]));
        std::vector<row_filter> f;
        for (uint32_t k = 0; k < nfilters; ++k) f.push_back(to_filter(filters[k]));
        tuple_array r = select_project(c, m, f);
        std::memcpy(out, r.data.data(), r.data.size() * sizeof(uint64_t));
        *out_n = r.count();
    });
}

int ref_merge_sorted(const uint64_t* full, uint64_t nf, int full_canonical,
                     const uint64_t* delta, uint64_t nd, int delta_canonical,
                     uint32_t arity, uint64_t buffer_rows, uint32_t workers,
                     uint64_t* out) {
    return guard([&] {
        std::vector<value_t> buf(buffer_rows * arity);
        tuple_array r = merge_sorted(make_rows(full, nf, arity, full_canonical != 0),
                                     make_rows(delta, nd, arity, delta_canonical != 0),
                                     buf, workers);
        std::memcpy(out, r.data.data(), r.data.size() * sizeof(uint64_t));
    });
}

int ref_difference(const uint64_t* new_rows, uint64_t nn, int new_canonical,
                   const uint64_t* full, uint64_t nf, int full_canonical,
                   uint32_t arity, uint32_t workers, uint64_t* out,
                   uint64_t* out_n) {
    return guard([&] {
        tuple_array r = difference(make_rows(new_rows, nn, arity, new_canonical != 0),
                                   make_rows(full, nf, arity, full_canonical != 0),
                                   workers);
        std::memcpy(out, r.data.data(), r.data.size() * sizeof(uint64_t));
        *out_n = r.count();
    });
}

// ---- engine ----------------------------------------------------------
// Relation ids: EDB declarations in program order, then IDB relations in
// program::idb_relations() order (the same numbering the product uses).

void* ref_engine_create(const char* program_source,
                        const gd_engine_config* cfg) {
    ref_engine* r = nullptr;
    int rc = guard([&] {
        auto e = std::make_unique<ref_engine>();
        e->prog = load_program(program_source);
        for (const auto& d : e->prog.edbs) e->names.push_back(d.name);
        for (const auto& n : e->prog.idb_relations()) e->names.push_back(n);
        e->eng = std::make_unique<engine>(e->prog, to_config(cfg));
        r = e.release();
    });
    return rc == GD_OK ? r : nullptr;
}

void ref_engine_destroy(void* h) { delete static_cast<ref_engine*>(h); }

int ref_engine_num_relations(void* h) {
    return static_cast<int>(static_cast<ref_engine*>(h)->names.size());
}

const char* ref_engine_relation_name(void* h, uint32_t id) {
    auto* e = static_cast<ref_engine*>(h);
    return id < e->names.size() ? e->names[id].c_str() : "";
}

int ref_engine_relation_arity(void* h, uint32_t id) {
    auto* e = static_cast<ref_engine*>(h);
    return static_cast<int>(*e->prog.arity_of(e->names.at(id)));
}

int ref_engine_load_edb(void* h, uint32_t id, const uint64_t* rows, uint64_t n,
                        int canonical) {
    auto* e = static_cast<ref_engine*>(h);
    return guard([&] {
        uint32_t arity = *e->prog.arity_of(e->names.at(id));
        e->eng->load_edb(e->names.at(id), make_rows(rows, n, arity, canonical != 0));
    });
}

int ref_engine_run(void* h) {
    auto* e = static_cast<ref_engine*>(h);
    return guard([&] { e->eng->run(); });
}

int ref_engine_relation_count(void* h, uint32_t id, uint64_t* n) {
    auto* e = static_cast<ref_engine*>(h);
    return guard([&] { *n = e->eng->relation(e->names.at(id)).count(); });
}

int ref_engine_relation_download(void* h, uint32_t id, uint64_t* out,
                                 uint64_t capacity_rows) {
    auto* e = static_cast<ref_engine*>(h);
    return guard([&] {
        const auto& t = e->eng->relation(e->names.at(id));
        if (t.count() > capacity_rows) throw std::logic_error("capacity");
        std::memcpy(out, t.data.data(), t.data.size() * sizeof(uint64_t));
    });
}

int ref_engine_stats(void* h, gd_run_stats* out) {
    auto* e = static_cast<ref_engine*>(h);
    return guard([&] {
        run_stats s = e->eng->stats();
        std::memset(out, 0, sizeof(*out));
        for (std::size_t p = 0; p < kPhaseOrder.size(); ++p)
            out->phase_seconds[p] = std::string(kPhaseOrder[p]) == "other"
                                        ? s.other_seconds()
                                        : s.phase(kPhaseOrder[p]);
        out->total_seconds = s.total_seconds;
        out->iterations = s.iterations;
        out->buffer_allocations = s.buffer_allocations;
        out->charge_events = s.charge_events;
        out->peak_tracked_bytes = s.peak_tracked_bytes;
        out->peak_temp_bytes = s.peak_temp_bytes;
    });
}

int ref_engine_delta_history(void* h, uint32_t id, uint64_t* out,
                             uint64_t capacity, uint64_t* len) {
    auto* e = static_cast<ref_engine*>(h);
    return guard([&] {
        run_stats s = e->eng->stats();
        *len = 0;
        for (const auto& [rel, hist] : s.delta_history) {
            if (rel != e->names.at(id)) continue;
            *len = hist.size();
            for (std::size_t i = 0; i < hist.size() && i < capacity; ++i)
                out[i] = hist[i];
        }
    });
}

int ref_engine_stats_tsv(void* h, char* out, uint64_t capacity) {
    auto* e = static_cast<ref_engine*>(h);
    return guard([&] {
        std::string s = to_tsv(e->eng->stats());
        if (s.size() + 1 > capacity) throw std::logic_error("capacity");
        std::memcpy(out, s.c_str(), s.size() + 1);
    });
}

// The compiled plans of the program as gd_rule_plan blobs (the data
// contract the device engine consumes).
int ref_engine_plans(void* h, gd_rule_plan* out, uint32_t capacity,
                     uint32_t* nplans) {
    auto* e = static_cast<ref_engine*>(h);
    return guard([&] {
        const auto& plans = e->eng->plans();
        std::map<std::string, uint32_t> ids;
        for (uint32_t i = 0; i < e->names.size(); ++i) ids[e->names[i]] = i;
        *nplans = static_cast<uint32_t>(plans.size());
        if (plans.size() > capacity) throw std::logic_error("capacity");
        for (std::size_t p = 0; p < plans.size(); ++p) {
            const rule_plan& rp = plans[p];
            gd_rule_plan& g = out[p];
            std::memset(&g, 0, sizeof(g));
            g.rule_index = static_cast<uint32_t>(rp.rule_index);
            g.head_rel = ids.at(rp.head_relation);
            g.head_arity = rp.head_arity;
            g.recursive = rp.recursive ? 1 : 0;
            g.nvariants = static_cast<uint32_t>(rp.variants.size());
            for (std::size_t v = 0; v < rp.variants.size(); ++v) {
                const rule_variant& rv = rp.variants[v];
                gd_variant& gv = g.variants[v];
                gv.src_rel = ids.at(rv.source.relation);
                gv.src_version =
                    rv.source.version == version_tag::delta ? GD_DELTA : GD_FULL;
                for (std::size_t c = 0; c < rv.source.permutation.size(); ++c)
                    gv.src_perm[c] = rv.source.permutation[c];
                gv.nsteps = static_cast<uint32_t>(rv.steps.size());
                for (std::size_t s = 0; s < rv.steps.size(); ++s) {
                    const join_step& st = rv.steps[s];
                    gd_join_step& gs = gv.steps[s];
                    gs.inner_rel = ids.at(st.inner_relation);
                    gs.join_column_count = st.join_column_count;
                    for (std::size_t c = 0; c < st.inner_permutation.size(); ++c)
                        gs.inner_perm[c] = st.inner_permutation[c];
                    gs.proj_arity = st.projection.output_arity();
                    for (std::size_t c = 0; c < st.projection.sources.size(); ++c)
                        gs.proj[c] = from_operand(st.projection.sources[c]);
                    gs.nfilters = static_cast<uint32_t>(st.filters.size());
                    for (std::size_t f = 0; f < st.filters.size(); ++f)
                        gs.filters[f] = from_filter(st.filters[f]);
                }
                gv.sel_arity = rv.select_projection.output_arity();
                for (std::size_t c = 0; c < rv.select_projection.sources.size(); ++c)
                    gv.sel_proj[c] = from_operand(rv.select_projection.sources[c]);
                gv.nsel_filters = static_cast<uint32_t>(rv.select_filters.size());
                for (std::size_t f = 0; f < rv.select_filters.size(); ++f)
                    gv.sel_filters[f] = from_filter(rv.select_filters[f]);
            }
        }
    });
}

// ---- seeded generators (test fixtures) --------------------------------

// SURVEY §8d C1 generator: std::mt19937_64(seed), uniform_int_distribution
// over [0, n-1], src drawn then dst, m draws (libstdc++ semantics).
int ref_gen_tc_rand(uint64_t n, uint64_t m, uint64_t seed, uint64_t* out) {
    return guard([&] {
        std::mt19937_64 rng(seed);
        std::uniform_int_distribution<uint64_t> pick(0, n - 1);
        for (uint64_t i = 0; i < m; ++i) {
            out[2 * i] = pick(rng);
            out[2 * i + 1] = pick(rng);
        }
    });
}

// Acceptance corpora of tests/acceptance_test.cpp:58-89 (kind 0 = REACH,
// seed 20240601; 1 = SG, 20240602; 2 = CSPA, 20240603).  Writes graph
// `idx` (CSPA: assign rows then dereference rows) into out; counts[0..1].
int ref_acceptance_corpus(int kind, uint32_t idx, uint64_t* out, uint64_t cap_rows, uint64_t* counts) {
    return guard([&] {
        std::vector<oracles::row_set> parts;
        if (kind == 0) {
            std::mt19937_64 rng(20240601);
            for (uint32_t i = 0; i <= idx; ++i) {
                auto g = oracles::random_graph(rng, 50, 400);
                if (i == idx) parts.push_back(g);
            }
        } else if (kind == 1) {
            std::mt19937_64 rng(20240602);
            for (uint32_t i = 0; i <= idx; ++i) {
                auto g = oracles::random_dag(rng, 30, 60);
                if (i == idx) parts.push_back(g);
            }
        } else {
            std::mt19937_64 rng(20240603);
            std::uniform_int_distribution<value_t> node(1, 15);
            std::uniform_int_distribution<int> count(1, 100);
            for (uint32_t i = 0; i <= idx; ++i) {
                oracles::database db;
                int na = count(rng), nd = count(rng);
                for (int j = 0; j < na; ++j) db["assign"].insert({node(rng), node(rng)});
                for (int j = 0; j < nd; ++j) db["dereference"].insert({node(rng), node(rng)});
                if (i == idx) {
                    parts.push_back(db["assign"]);
                    parts.push_back(db["dereference"]);
                }
            }
        }
        uint64_t w = 0;
        for (std::size_t p = 0; p < parts.size(); ++p) {
            counts[p] = parts[p].size();
            for (const auto& r : parts[p]) {
                if (w >= cap_rows) throw std::logic_error("corpus capacity");
                out[2 * w] = r[0];
                out[2 * w + 1] = r[1];
                ++w;
            }
        }
    });
}

// ---- fact files / TSV (io.hpp) ----------------------------------------
// read_facts(path, arity[, dictionary]): canonical rows into out.
int ref_read_facts(const char* path, uint32_t arity, int use_dict, uint64_t* out, uint64_t cap_rows,
                   uint64_t* count) {
    return guard([&] {
        dictionary d;
        tuple_array t = read_facts(path, arity, use_dict ? &d : nullptr);
        *count = t.count();
        if (t.count() > cap_rows) throw std::logic_error("read_facts: capacity");
        if (!t.data.empty()) std::memcpy(out, t.data.data(), t.data.size() * sizeof(uint64_t));
    });
}

// to_tsv of rows (canonicalized first, like a relation) -> bytes.
int ref_to_tsv(const uint64_t* rows, uint64_t n, uint32_t arity, char* out, uint64_t cap, uint64_t* len) {
    return guard([&] {
        tuple_array t = canonicalize(make_rows(rows, n, arity, false));
        const std::string s = to_tsv(t);
        *len = s.size();
        if (s.size() > cap) throw std::logic_error("to_tsv: capacity");
        std::memcpy(out, s.data(), s.size());
    });
}

// read_facts with a dictionary, then write_relation with it: the decoded
// canonical TSV bytes.
int ref_dict_roundtrip(const char* path, uint32_t arity, char* out, uint64_t cap, uint64_t* len) {
    return guard([&] {
        dictionary d;
        tuple_array t = read_facts(path, arity, &d);
        const std::string s = to_tsv(t, &d);
        *len = s.size();
        if (s.size() > cap) throw std::logic_error("to_tsv: capacity");
        std::memcpy(out, s.data(), s.size());
    });
}

int ref_file_is_all_integers(const char* path, int* result) {
    return guard([&] { *result = file_is_all_integers(path) ? 1 : 0; });
}

}  // extern "C"
