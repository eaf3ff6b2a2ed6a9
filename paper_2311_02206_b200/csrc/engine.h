// engine.h — the device fixpoint engine behind gd_engine_* (the drop-in for
// arraylog::engine, engine.hpp:40-558).  Orchestration is single-threaded
// host C++ (as in the reference); every bulk step is an sm_100a kernel on
// the context stream; relations stay resident in HBM across iterations and
// the host reads back a few counters per join step / merge.
#pragma once

#include <chrono>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "accounting.h"
#include "ctx.h"
#include "encoding.h"
#include "gdlog_b200.h"

namespace gd {

struct RelInfo {
    std::string name;
    u32 arity = 0;
    bool is_edb = false;
    // logical bytes charged to the accountant (engine.hpp:60-62)
    u64 full_bytes = 0, delta_bytes = 0, new_bytes = 0;
    std::vector<u64> history;
    std::vector<gd_iter_record> log;
};

class ImplBase {
public:
    virtual ~ImplBase() = default;
    virtual void seed() = 0;
    virtual void iterate() = 0;
    // True when the canonical output is still being sorted / packed on the
    // stream (segmented final sort): iterate() returns without a sync and
    // the download waits per segment.
    virtual bool output_pending() const { return false; }
    virtual u64 count(u32 rel) = 0;
    virtual void download(u32 rel, u64* out, bool device) = 0;
    virtual u64 digest(u32 rel) = 0;
    virtual void partition_begin(u64* send_counts, const void** d_send) = 0;
    virtual void partition_end(const void* d_recv, u64 recv_rows, u64* local_delta) = 0;
    virtual void partition_finish() = 0;
    virtual u64 partition_run(struct Comm& comm, u64 max_iters) = 0;
};

class Engine {
public:
    Engine(Ctx& c, const gd_engine_config& cfg, u32 nrels, const u32* arities, const u32* is_edb,
           const char* const* names);
    ~Engine();

    void set_plans(const gd_rule_plan* plans, u32 n);
    void load_edb(u32 rel, const u64* rows, u64 n, bool canonical, bool device);
    void seed();
    void iterate();
    void run() {
        seed();
        iterate();
    }
    u64 relation_count(u32 rel);
    void relation_download(u32 rel, u64* out, u64 capacity_rows, bool device);
    u64 relation_digest(u32 rel);
    void fill_stats(gd_run_stats* out) const;
    const RelInfo& rel(u32 r) const { return info_.at(check_rel(r)); }
    void encoding(u32* bits, u32* key_words, u32* dict) const;

    void set_partition(u32 rank, u32 nranks);
    u32 exchange_words() const;
    void partition_begin(u64* send_counts, const void** d_send);
    void partition_end(const void* d_recv, u64 recv_rows, u64* local_delta);
    void partition_finish();
    // Native driver (gd_engine_run_partitioned): the whole partitioned
    // fixpoint with NCCL exchanges; returns the iterations run.
    u64 partition_run(struct Comm& comm, u64 max_iters);

    // ---- shared with Impl<K> (engine.cu) ----
    u32 check_rel(u32 r) const {
        if (r >= info_.size()) throw_usage("unknown relation id " + std::to_string(r));
        return r;
    }
    void add_phase(const char* phase, double s) { phase_seconds_[phase] += s; }

    Ctx& c;
    gd_engine_config cfg;
    std::vector<RelInfo> info_;
    std::vector<gd_rule_plan> plans_;
    Accountant acct;
    BufferManager bufs;
    bool seeded = false;
    u64 iterations = 0;
    u64 join_tuples = 0;
    double total_seconds = 0;
    std::map<std::string, double> phase_seconds_;
    double kernel_seconds[6] = {0, 0, 0, 0, 0, 0};
    u64 algo_bytes[6] = {0, 0, 0, 0, 0, 0};
    // EDB rows uploaded before the encoding is fixed (canonical, u64 rows)
    std::vector<DevBuf<u64>> raw;
    std::vector<u64> raw_n;
    EncodingOwner enc;
    u32 rank = 0, nranks = 1;
    std::unique_ptr<ImplBase> impl;
};

// Phase timer: wall time into run_stats::phase_seconds (engine.hpp:280-286).
struct PhaseTimer {
    Engine& e;
    const char* phase;
    const char* prev;
    std::chrono::steady_clock::time_point t0;
    PhaseTimer(Engine& eng, const char* p) : e(eng), phase(p), prev(eng.c.cur_phase), t0(std::chrono::steady_clock::now()) {
        eng.c.cur_phase = p;
    }
    ~PhaseTimer() {
        e.add_phase(phase, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        e.c.cur_phase = prev;
    }
};

// Canonicalizes device u64 rows (any values but the sentinel) into out;
// returns the distinct count.  Shared by load_edb and gd_canonicalize.
u64 canonicalize_rows(Ctx& c, const u64* d_rows, u64 n, u32 arity, DevBuf<u64>& out);

}  // namespace gd
