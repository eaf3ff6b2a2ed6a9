// arraylog_b200.hpp — the reference C++ API on the B200 device engine.
//
// Drop-in for the hot path of /root/reference/proj/include/arraylog: the
// same types (tuple_array, relation_container, join_spec, engine_config,
// run_stats, program, rule_plan) and the same signatures, implemented on
// libgdlog_b200.so through the C-ABI of include/gdlog_b200.h.  A program that
// uses `arraylog::engine` switches by using `arraylog::b200::engine` (or a
// namespace alias); the frontend (parser, planner, I/O) stays
// the reference's own.
//
// Include AFTER the reference headers:
//     #include "arraylog/arraylog.hpp"        // reference (program, plans, types)
//     #include "arraylog_b200/arraylog_b200.hpp"
// and link -lgdlog_b200.
#pragma once

#include <cstring>
#include <map>
#include <filesystem>
#include <fstream>
#include <initializer_list>
#include <iterator>
#include <memory>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "../gdlog_b200.h"

namespace arraylog::b200 {

// ---- errors: gd_status -> the reference exception types (types.hpp) -------

class context {
public:
    explicit context(int device = 0) {
        gd_ctx* c = nullptr;
        const gd_status s = gd_ctx_create(device, nullptr, &c);
        if (s != GD_OK) throw std::runtime_error(std::string("B200 context: ") + gd_last_error(nullptr));
        ctx_.reset(c);
    }
    gd_ctx* get() const { return ctx_.get(); }

    void check(gd_status s) const {
        if (s == GD_OK) return;
        const std::string msg = gd_last_error(ctx_.get());
        switch (s) {
            case GD_ERR_CONFIG: throw config_error(msg);
            case GD_ERR_USAGE: throw usage_error(msg);
            case GD_ERR_LOAD: throw load_error(msg);
            case GD_ERR_PLAN: throw plan_error(msg);
            case GD_ERR_BUDGET: {
                std::string phase = gd_last_error_phase(ctx_.get());
                // budget_error prefixes "memory budget exceeded in <phase> phase: "
                const std::string pre = "memory budget exceeded in " + phase + " phase: ";
                throw budget_error(phase, msg.rfind(pre, 0) == 0 ? msg.substr(pre.size()) : msg);
            }
            case GD_ERR_LOGIC:
            case GD_ERR_INVALID_ARG: throw std::logic_error(msg);
            default: throw std::runtime_error(msg);
        }
    }

    static context& default_context() {
        static context c(0);
        return c;
    }

private:
    struct del {
        void operator()(gd_ctx* c) const { gd_ctx_destroy(c); }
    };
    std::unique_ptr<gd_ctx, del> ctx_;
};

namespace detail {

inline gd_operand to_c(const operand& o) {
    gd_operand g{};
    g.kind = o.from == operand::kind::outer_col   ? GD_OUTER_COL
             : o.from == operand::kind::inner_col ? GD_INNER_COL
                                                  : GD_CONSTANT;
    g.column = o.column;
    g.value = o.value;
    return g;
}

inline gd_filter to_c(const row_filter& f) {
    gd_filter g{};
    g.lhs = to_c(f.lhs);
    g.rhs = to_c(f.rhs);
    g.require_equal = f.require_equal ? 1 : 0;
    return g;
}

inline gd_container_view view(const relation_container& c) {
    gd_container_view v{};
    v.rows = c.tuples.data.data();
    v.n = c.tuples.count();
    v.arity = c.tuples.arity;
    v.canonical = c.tuples.canonical ? 1 : 0;
    v.index_prefix_len = c.index ? c.index->prefix_len : 0;
    v.load_factor = c.index ? c.index->load_factor : 0.8;
    return v;
}

inline gd_join_spec spec_of(const join_spec& s) {
    if (!s.outer || !s.inner) throw usage_error("join: outer and inner are required");
    gd_join_spec g{};
    g.join_column_count = s.join_column_count;
    g.proj_arity = s.projection.output_arity();
    if (g.proj_arity > GD_MAX_ARITY || s.filters.size() > GD_MAX_FILTERS)
        throw config_error("join spec exceeds the device limits");
    for (std::size_t i = 0; i < s.projection.sources.size(); ++i) g.proj[i] = to_c(s.projection.sources[i]);
    g.nfilters = static_cast<std::uint32_t>(s.filters.size());
    for (std::size_t i = 0; i < s.filters.size(); ++i) g.filters[i] = to_c(s.filters[i]);
    return g;
}

}  // namespace detail

// ---- kernel-level functions (tuple_array.hpp, index_map.hpp, ra.hpp) -------

// canonicalize (tuple_array.hpp:73-133)
inline tuple_array canonicalize(const tuple_array& raw, unsigned /*workers*/ = 1,
                                context& ctx = context::default_context()) {
    if (raw.arity == 0) throw std::logic_error("canonicalize: arity must be positive");
    tuple_array out(raw.arity);
    out.canonical = true;
    if (raw.count() == 0) return out;
    if (raw.canonical) {
        out.data = raw.data;
        return out;
    }
    out.data.resize(raw.data.size());
    std::uint64_t m = 0;
    ctx.check(gd_canonicalize(ctx.get(), raw.data.data(), raw.count(), raw.arity, out.data.data(), &m));
    out.data.resize(m * raw.arity);
    return out;
}

// permute_columns (ra.hpp:426-454)
inline tuple_array permute_columns(const tuple_array& rel, std::span<const std::uint32_t> perm,
                                   unsigned /*workers*/ = 1, context& ctx = context::default_context()) {
    tuple_array out(rel.arity);
    out.canonical = true;
    out.data.resize(rel.data.size());
    std::uint64_t m = 0;
    ctx.check(gd_permute_columns(ctx.get(), rel.data.data(), rel.count(), rel.arity, rel.canonical ? 1 : 0,
                                 perm.data(), static_cast<std::uint32_t>(perm.size()), out.data.data(), &m));
    out.data.resize(m * rel.arity);
    return out;
}

// Batched range_lookup (container.hpp:52-89) — one device index build, one
// probe per prefix; prefixes are row-major (count x prefix_len).
inline std::vector<row_range> range_lookup_batch(const relation_container& c, std::span<const value_t> prefixes,
                                                 context& ctx = context::default_context()) {
    if (!c.index) throw usage_error("range_lookup: container has no index");
    const std::uint32_t pl = c.index->prefix_len;
    const std::uint64_t nk = prefixes.size() / pl;
    std::vector<std::uint64_t> st(nk ? nk : 1), ct(nk ? nk : 1);
    std::uint64_t sc = 0, oc = 0;
    ctx.check(gd_index_lookup(ctx.get(), c.tuples.data.data(), c.tuples.count(), c.tuples.arity,
                              c.tuples.canonical ? 1 : 0, pl, c.index->load_factor, prefixes.data(), nk, pl,
                              st.data(), ct.data(), &sc, &oc));
    std::vector<row_range> out(nk);
    for (std::uint64_t i = 0; i < nk; ++i) out[i] = {st[i], ct[i]};
    return out;
}

inline row_range range_lookup(const relation_container& c, std::span<const value_t> prefix,
                              context& ctx = context::default_context()) {
    if (!c.index) throw usage_error("range_lookup: container has no index");
    if (c.index->prefix_len != prefix.size())
        throw usage_error("range_lookup: prefix length " + std::to_string(prefix.size()) +
                          " does not match index prefix_len " + std::to_string(c.index->prefix_len));
    return range_lookup_batch(c, prefix, ctx).at(0);
}

inline row_range range_lookup(const relation_container& c, std::initializer_list<value_t> prefix,
                              context& ctx = context::default_context()) {
    return range_lookup(c, std::span<const value_t>(prefix.begin(), prefix.size()), ctx);
}

// group_starts (index_map.hpp:46-66): first row of every distinct prefix
inline std::vector<std::uint64_t> group_starts(const tuple_array& tuples, std::uint32_t prefix_len,
                                               unsigned /*workers*/ = 1, context& ctx = context::default_context()) {
    std::vector<std::uint64_t> out(tuples.count() ? tuples.count() : 1);
    std::uint64_t m = 0;
    ctx.check(gd_group_starts(ctx.get(), tuples.data.data(), tuples.count(), tuples.arity, tuples.canonical ? 1 : 0,
                              prefix_len, out.data(), &m));
    out.resize(m);
    return out;
}

// join_count (ra.hpp:141-182)
inline std::size_t join_count(const join_spec& spec, unsigned /*workers*/ = 1, std::size_t /*stride*/ = 0,
                              context& ctx = context::default_context()) {
    const gd_join_spec g = detail::spec_of(spec);
    const gd_container_view o = detail::view(*spec.outer), i = detail::view(*spec.inner);
    std::uint64_t total = 0;
    ctx.check(gd_join_count(ctx.get(), &o, &i, &g, &total));
    return total;
}

// join_materialize (ra.hpp:189-263): `out` pre-sized to count * arity
inline void join_materialize(const join_spec& spec, tuple_array& out, unsigned /*workers*/ = 1,
                             std::size_t /*stride*/ = 0, context& ctx = context::default_context()) {
    const gd_join_spec g = detail::spec_of(spec);
    const gd_container_view o = detail::view(*spec.outer), i = detail::view(*spec.inner);
    const std::uint32_t arity = spec.projection.output_arity();
    out.arity = arity;
    out.canonical = false;
    ctx.check(gd_join_materialize(ctx.get(), &o, &i, &g, out.data.data(), arity ? out.data.size() / arity : 0));
}

// select_project (ra.hpp:267-293)
inline tuple_array select_project(const relation_container& src, const column_map& projection,
                                  std::span<const row_filter> filters = {},
                                  context& ctx = context::default_context()) {
    std::vector<gd_operand> p;
    for (const auto& s : projection.sources) p.push_back(detail::to_c(s));
    std::vector<gd_filter> f;
    for (const auto& x : filters) f.push_back(detail::to_c(x));
    tuple_array out(projection.output_arity());
    out.data.resize(src.tuples.count() * projection.output_arity());
    std::uint64_t m = 0;
    ctx.check(gd_select_project(ctx.get(), src.tuples.data.data(), src.tuples.count(), src.tuples.arity, p.data(),
                                static_cast<std::uint32_t>(p.size()), f.data(), static_cast<std::uint32_t>(f.size()),
                                out.data.data(), &m));
    out.data.resize(m * projection.output_arity());
    return out;
}

// merge_sorted (ra.hpp:299-381)
inline tuple_array merge_sorted(const tuple_array& full, const tuple_array& delta, std::span<value_t> buffer,
                                unsigned /*workers*/ = 1, context& ctx = context::default_context()) {
    if (full.arity != delta.arity) throw std::logic_error("merge_sorted: arity mismatch");
    tuple_array out(full.arity);
    out.canonical = true;
    out.data.resize(full.data.size() + delta.data.size());
    ctx.check(gd_merge_sorted(ctx.get(), full.data.data(), full.count(), full.canonical ? 1 : 0, delta.data.data(),
                              delta.count(), delta.canonical ? 1 : 0, full.arity,
                              full.arity ? buffer.size() / full.arity : 0, out.data.data()));
    return out;
}

// difference (ra.hpp:386-422)
inline tuple_array difference(const tuple_array& new_rel, const tuple_array& full, unsigned /*workers*/ = 1,
                              context& ctx = context::default_context()) {
    if (new_rel.arity != full.arity) throw std::logic_error("difference: arity mismatch");
    tuple_array out(new_rel.arity);
    out.canonical = true;
    out.data.resize(new_rel.data.size());
    std::uint64_t m = 0;
    ctx.check(gd_difference(ctx.get(), new_rel.data.data(), new_rel.count(), new_rel.canonical ? 1 : 0,
                            full.data.data(), full.count(), full.canonical ? 1 : 0, new_rel.arity, out.data.data(),
                            &m));
    out.data.resize(m * new_rel.arity);
    return out;
}

// ---- engine (engine.hpp:40-558) ---------------------------------------------

// ---- fact files / TSV (io.hpp:64-170), parsed and formatted on the device.
// Numeric files only; pass the reference's arraylog::dictionary to the
// reference's own read_facts / to_tsv for token files.

namespace detail {
inline std::string slurp(const std::filesystem::path& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw load_error("cannot open fact file '" + path.string() + "'");
    return std::string((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}
}  // namespace detail

// The reference's own functions (token files with a dictionary stay on the
// host, as in the reference); a build that renames the reference entry
// points (tests/cpp/reftests) redefines this.
#ifndef ARRAYLOG_B200_REF
#define ARRAYLOG_B200_REF(name) ::arraylog::name
#endif

inline tuple_array read_facts(const std::filesystem::path& path, std::uint32_t arity, dictionary* dict = nullptr,
                              unsigned workers = 1, context& ctx = context::default_context()) {
    if (dict) return ARRAYLOG_B200_REF(read_facts)(path, arity, dict, workers);
    if (arity == 0) throw load_error("read_facts: arity must be positive");
    const std::string text = detail::slurp(path);
    std::uint64_t cap = 1;
    for (char ch : text) cap += ch == '\n';
    tuple_array out(arity);
    out.data.resize(cap * arity);
    std::uint64_t n = 0;
    ctx.check(gd_parse_facts(ctx.get(), path.string().c_str(), text.data(), text.size(), arity, out.data.data(), cap,
                             &n));
    out.data.resize(n * arity);
    out.canonical = true;
    return out;
}

inline bool file_is_all_integers(const std::filesystem::path& path, context& ctx = context::default_context()) {
    const std::string text = detail::slurp(path);
    int r = 0;
    ctx.check(gd_facts_all_integers(ctx.get(), text.data(), text.size(), &r));
    return r != 0;
}

inline std::string to_tsv(const tuple_array& rel, const dictionary* dict = nullptr,
                          context& ctx = context::default_context()) {
    if (dict) return ARRAYLOG_B200_REF(to_tsv)(rel, dict);
    std::uint64_t len = 0;
    ctx.check(gd_rows_to_tsv(ctx.get(), rel.data.data(), rel.count(), rel.arity, nullptr, 0, &len));
    std::string out(len, '\0');
    if (len) ctx.check(gd_rows_to_tsv(ctx.get(), rel.data.data(), rel.count(), rel.arity, out.data(), len, &len));
    return out;
}

inline void write_relation(const tuple_array& rel, const std::filesystem::path& path,
                           const dictionary* dict = nullptr, context& ctx = context::default_context()) {
    if (!rel.canonical) throw std::logic_error("write_relation: relation must be canonical");
    const std::string text = to_tsv(rel, dict, ctx);
    std::ofstream out(path, std::ios::binary);
    if (!out) throw load_error("cannot open '" + path.string() + "' for writing");
    out << text;
    out.flush();
    if (!out) throw load_error("failed while writing '" + path.string() + "'");
}

class engine {
public:
    explicit engine(program p, engine_config cfg = {}, context& ctx = context::default_context())
        : prog_(std::move(p)), cfg_(cfg), ctx_(&ctx) {
        if (!(cfg_.load_factor > 0.0) || cfg_.load_factor >= 1.0)
            throw config_error("engine: load factor must be in (0, 1)");
        if (cfg_.alpha == 0) throw config_error("buffer_manager: alpha must be at least 1");
        for (const auto& e : prog_.edbs) add_rel(e.name, e.arity, true);
        for (const auto& n : prog_.idb_relations()) add_rel(n, *prog_.arity_of(n), false);
        std::vector<std::uint32_t> ar, edb;
        std::vector<const char*> nm;
        for (const auto& r : rels_) {
            ar.push_back(r.arity);
            edb.push_back(r.is_edb ? 1 : 0);
            nm.push_back(r.name.c_str());
        }
        gd_engine_config c{};
        c.memory_budget_bytes = cfg_.memory_budget_bytes == memory_accountant::unlimited
                                    ? UINT64_MAX
                                    : static_cast<std::uint64_t>(cfg_.memory_budget_bytes);
        c.ebm_enabled = cfg_.ebm_enabled ? 1 : 0;
        c.alpha = cfg_.alpha;
        c.load_factor = cfg_.load_factor;
        c.workers = cfg_.workers;
        c.stride_rows = cfg_.stride_rows;
        gd_engine* e = nullptr;
        ctx_->check(gd_engine_create(ctx_->get(), &c, static_cast<std::uint32_t>(rels_.size()), ar.data(),
                                     edb.data(), nm.data(), &e));
        eng_.reset(e);
        set_plans(plan_program(prog_));
    }

    engine(const engine&) = delete;
    engine& operator=(const engine&) = delete;

    void override_plans(std::vector<rule_plan> plans) {
        if (seeded_) throw std::logic_error("override_plans: engine already seeded");
        set_plans(std::move(plans));
    }
    const std::vector<rule_plan>& plans() const { return plans_; }
    const program& source_program() const { return prog_; }

    // load_edb(name, read_facts(path, arity)) with the file parsed on the
    // device straight into the relation.
    void load_edb_file(const std::string& name, const std::filesystem::path& path) {
        if (seeded_) throw std::logic_error("load_edb: engine already running");
        auto it = ids_.find(name);
        if (it == ids_.end() || !rels_[it->second].is_edb)
            throw load_error("load_edb: '" + name + "' is not a declared EDB relation");
        const std::string text = detail::slurp(path);
        ctx_->check(gd_engine_load_edb_tsv(eng_.get(), it->second, path.string().c_str(), text.data(), text.size()));
    }
    // write_relation(relation(name), path), formatted on the device.
    void write_relation_file(const std::string& name, const std::filesystem::path& path) {
        auto it = ids_.find(name);
        if (it == ids_.end()) throw usage_error("relation: unknown relation '" + name + "'");
        std::uint64_t len = 0;
        ctx_->check(gd_engine_relation_tsv(eng_.get(), it->second, nullptr, 0, &len));
        std::string text(len, '\0');
        if (len) ctx_->check(gd_engine_relation_tsv(eng_.get(), it->second, text.data(), len, &len));
        std::ofstream out(path, std::ios::binary);
        if (!out) throw load_error("cannot open '" + path.string() + "' for writing");
        out << text;
    }

    void load_edb(const std::string& name, tuple_array facts) {
        if (seeded_) throw std::logic_error("load_edb: engine already running");
        auto it = ids_.find(name);
        if (it == ids_.end() || !rels_[it->second].is_edb)
            throw load_error("load_edb: '" + name + "' is not a declared EDB relation");
        const auto& r = rels_[it->second];
        if (facts.arity != r.arity)
            throw load_error("load_edb: '" + name + "' expects arity " + std::to_string(r.arity) + ", got " +
                             std::to_string(facts.arity));
        ctx_->check(gd_engine_load_edb(eng_.get(), it->second, facts.data.data(), facts.count(),
                                       facts.canonical ? 1 : 0));
    }

    void run() {
        seed();
        iterate_to_fixpoint();
    }
    void seed() {
        if (seeded_) throw std::logic_error("seed: called twice");
        ctx_->check(gd_engine_seed(eng_.get()));
        seeded_ = true;
        cache_.clear();
    }
    void iterate_to_fixpoint() {
        if (!seeded_) seed();
        ctx_->check(gd_engine_iterate(eng_.get()));
        cache_.clear();
    }

    // Canonical rows, downloaded once and kept as the host mirror the
    // reference returns by reference (engine.hpp:259-264).
    const tuple_array& relation(const std::string& name) const {
        auto it = ids_.find(name);
        if (it == ids_.end()) throw usage_error("unknown relation '" + name + "'");
        auto c = cache_.find(name);
        if (c != cache_.end()) return c->second;
        std::uint64_t n = 0;
        ctx_->check(gd_engine_relation_count(eng_.get(), it->second, &n));
        tuple_array t(rels_[it->second].arity);
        t.canonical = true;
        t.data.resize(n * t.arity);
        ctx_->check(gd_engine_relation_download(eng_.get(), it->second, t.data.data(), n));
        return cache_.emplace(name, std::move(t)).first->second;
    }

    std::vector<std::string> idb_relations() const { return prog_.idb_relations(); }

    // accountant() (engine.hpp:103-105): the device engine's logical-byte
    // ledger, with memory_accountant's getters (budget.hpp:50-60).
    class accountant_state {
    public:
        std::size_t current(memory_accountant::category cat) const { return cur_[static_cast<std::size_t>(cat)]; }
        std::size_t current_total() const { return cur_[0] + cur_[1] + cur_[2]; }
        std::size_t peak_bytes() const { return peak_; }
        std::size_t peak_temp_bytes() const { return peak_temp_; }
        std::size_t charge_events() const { return events_; }
        std::size_t budget() const { return budget_; }

    private:
        friend class engine;
        std::uint64_t cur_[3] = {0, 0, 0};
        std::uint64_t peak_ = 0, peak_temp_ = 0, events_ = 0;
        std::size_t budget_ = memory_accountant::unlimited;
    };
    const accountant_state& accountant() const {
        std::uint64_t b = 0;
        ctx_->check(gd_engine_accountant(eng_.get(), acct_.cur_, &acct_.peak_, &acct_.peak_temp_, &acct_.events_, &b));
        acct_.budget_ = b == UINT64_MAX ? memory_accountant::unlimited : static_cast<std::size_t>(b);
        return acct_;
    }

    run_stats stats() const {
        gd_run_stats s{};
        ctx_->check(gd_engine_stats(eng_.get(), &s));
        run_stats out;
        for (std::size_t p = 0; p + 1 < kPhaseOrder.size(); ++p)
            if (s.phase_seconds[p] > 0) out.phase_seconds[kPhaseOrder[p]] = s.phase_seconds[p];
        out.total_seconds = s.total_seconds;
        out.iterations = s.iterations;
        out.buffer_allocations = s.buffer_allocations;
        out.charge_events = s.charge_events;
        out.peak_tracked_bytes = s.peak_tracked_bytes;
        out.peak_temp_bytes = s.peak_temp_bytes;
        std::map<std::string, std::vector<std::size_t>> hist;  // name order, engine.hpp:192,254
        for (const auto& p : plans_)
            if (p.recursive) hist[p.head_relation];
        for (auto& [name, h] : hist) {
            const std::uint32_t id = ids_.at(name);
            std::uint64_t len = 0;
            ctx_->check(gd_engine_delta_history(eng_.get(), id, nullptr, 0, &len));
            std::vector<std::uint64_t> v(len ? len : 1);
            ctx_->check(gd_engine_delta_history(eng_.get(), id, v.data(), len, &len));
            h.assign(v.begin(), v.begin() + len);
            out.delta_history.emplace_back(name, h);
        }
        return out;
    }

private:
    struct rel {
        std::string name;
        std::uint32_t arity;
        bool is_edb;
    };
    struct edel {
        void operator()(gd_engine* e) const { gd_engine_destroy(e); }
    };

    void add_rel(const std::string& n, std::uint32_t a, bool edb) {
        ids_[n] = static_cast<std::uint32_t>(rels_.size());
        rels_.push_back({n, a, edb});
    }

    // rule_plan (plan.hpp:52-58) -> gd_rule_plan blobs
    void set_plans(std::vector<rule_plan> plans) {
        std::vector<gd_rule_plan> blobs(plans.size());
        for (std::size_t p = 0; p < plans.size(); ++p) {
            const rule_plan& rp = plans[p];
            gd_rule_plan& g = blobs[p];
            std::memset(&g, 0, sizeof(g));
            auto rid = [&](const std::string& n) {
                auto it = ids_.find(n);
                if (it == ids_.end()) throw usage_error("plan references unknown relation '" + n + "'");
                return it->second;
            };
            g.rule_index = static_cast<std::uint32_t>(rp.rule_index);
            g.head_rel = rid(rp.head_relation);
            g.head_arity = rp.head_arity;
            g.recursive = rp.recursive ? 1 : 0;
            if (rp.variants.size() > GD_MAX_VARIANTS) throw plan_error("too many rule variants for the device");
            g.nvariants = static_cast<std::uint32_t>(rp.variants.size());
            for (std::size_t v = 0; v < rp.variants.size(); ++v) {
                const rule_variant& rv = rp.variants[v];
                gd_variant& gv = g.variants[v];
                gv.src_rel = rid(rv.source.relation);
                gv.src_version = rv.source.version == version_tag::delta ? GD_DELTA : GD_FULL;
                for (std::size_t c = 0; c < rv.source.permutation.size(); ++c) gv.src_perm[c] = rv.source.permutation[c];
                if (rv.steps.size() > GD_MAX_STEPS) throw plan_error("too many join steps for the device");
                gv.nsteps = static_cast<std::uint32_t>(rv.steps.size());
                for (std::size_t s = 0; s < rv.steps.size(); ++s) {
                    const join_step& st = rv.steps[s];
                    gd_join_step& gs = gv.steps[s];
                    gs.inner_rel = rid(st.inner_relation);
                    gs.join_column_count = st.join_column_count;
                    for (std::size_t c = 0; c < st.inner_permutation.size(); ++c) gs.inner_perm[c] = st.inner_permutation[c];
                    gs.proj_arity = st.projection.output_arity();
                    for (std::size_t c = 0; c < st.projection.sources.size(); ++c)
                        gs.proj[c] = detail::to_c(st.projection.sources[c]);
                    gs.nfilters = static_cast<std::uint32_t>(st.filters.size());
                    for (std::size_t f = 0; f < st.filters.size(); ++f) gs.filters[f] = detail::to_c(st.filters[f]);
                }
                gv.sel_arity = rv.select_projection.output_arity();
                for (std::size_t c = 0; c < rv.select_projection.sources.size(); ++c)
                    gv.sel_proj[c] = detail::to_c(rv.select_projection.sources[c]);
                gv.nsel_filters = static_cast<std::uint32_t>(rv.select_filters.size());
                for (std::size_t f = 0; f < rv.select_filters.size(); ++f)
                    gv.sel_filters[f] = detail::to_c(rv.select_filters[f]);
            }
        }
        ctx_->check(gd_engine_set_plans(eng_.get(), blobs.data(), static_cast<std::uint32_t>(blobs.size())));
        plans_ = std::move(plans);
    }

    program prog_;
    engine_config cfg_;
    context* ctx_;
    std::unique_ptr<gd_engine, edel> eng_;
    std::vector<rel> rels_;
    std::map<std::string, std::uint32_t> ids_;
    std::vector<rule_plan> plans_;
    bool seeded_ = false;
    mutable std::map<std::string, tuple_array> cache_;
    mutable accountant_state acct_;
};

}  // namespace arraylog::b200
