// ctx.h — host-side context: device, stream, stream-ordered device memory,
// error types.  Internal to libgdlog_b200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <time.h>

#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gdlog_b200.h"

namespace gd {

// One exception type carrying the gd_status it maps to at the C boundary
// (types.hpp:19-72 for the reference exception each code stands for).
struct Error : std::runtime_error {
    gd_status code;
    std::string phase;
    Error(gd_status c, const std::string& msg, std::string ph = {})
        : std::runtime_error(msg), code(c), phase(std::move(ph)) {}
};

[[noreturn]] inline void throw_logic(const std::string& m) { throw Error(GD_ERR_LOGIC, m); }
[[noreturn]] inline void throw_config(const std::string& m) { throw Error(GD_ERR_CONFIG, m); }
[[noreturn]] inline void throw_usage(const std::string& m) { throw Error(GD_ERR_USAGE, m); }
[[noreturn]] inline void throw_load(const std::string& m) { throw Error(GD_ERR_LOAD, m); }
[[noreturn]] inline void throw_plan_error(const std::string& m) { throw Error(GD_ERR_PLAN, m); }
[[noreturn]] inline void throw_unsupported(const std::string& m) { throw Error(GD_ERR_UNSUPPORTED, m); }
[[noreturn]] inline void throw_budget(const std::string& phase, const std::string& detail) {
    throw Error(GD_ERR_BUDGET, "memory budget exceeded in " + phase + " phase: " + detail, phase);
}

#define GD_CUDA(call)                                                            \
    do {                                                                         \
        cudaError_t e_ = (call);                                                 \
        if (e_ != cudaSuccess)                                                   \
            throw ::gd::Error(GD_ERR_CUDA, std::string(#call) + ": " +           \
                                               cudaGetErrorString(e_));          \
    } while (0)

// Kernel classes for live per-kernel timing (bench roofline).
enum KClass : int {
    KC_SORT_PASS = 0,   // onesweep_kernel (one digit pass)
    KC_SORT_HIST,       // radix_hist_kernel
    KC_MERGE,           // diff_merge_kernel (+ its partition)
    KC_PROBE,           // join_probe_kernel
    KC_MATERIALIZE,     // join_materialize_kernel (+ its partition)
    KC_INDEX,           // group starts + index insert
    KC_SELECT,          // compaction / select_project / unique
    KC_OTHER,           // pack/unpack/permute/owner/...
    KC_DIFF,            // difference flags (search or streaming)
    KC_INSERT,          // loop_materialize_insert / loop_select_insert
    KC_LOOP_CTL,        // loop_gate / loop_end / loop_select_cand
    KC_COUNT
};

// Records CUDA events around instrumented launches when enabled; resolves
// them lazily (after a stream sync) into per-class time, launch counts and
// algorithmic bytes.
struct Profiler {
    struct Rec {
        int cls;
        cudaEvent_t a, b;
        uint64_t bytes;
    };
    bool on = false;
    std::vector<cudaEvent_t> free_events;
    std::vector<Rec> pending;
    double ms[KC_COUNT] = {};
    uint64_t launches[KC_COUNT] = {};
    uint64_t bytes[KC_COUNT] = {};

    cudaEvent_t take() {
        if (free_events.empty()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            return e;
        }
        cudaEvent_t e = free_events.back();
        free_events.pop_back();
        return e;
    }
    void resolve() {
        for (auto& r : pending) {
            float t = 0;
            if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess) ms[r.cls] += t;
            launches[r.cls] += 1;
            bytes[r.cls] += r.bytes;
            free_events.push_back(r.a);
            free_events.push_back(r.b);
        }
        pending.clear();
    }
    void reset() {
        pending.clear();
        for (int i = 0; i < KC_COUNT; ++i) ms[i] = 0, launches[i] = 0, bytes[i] = 0;
    }
    ~Profiler() {
        for (auto& r : pending) free_events.push_back(r.a), free_events.push_back(r.b);
        for (auto e : free_events) cudaEventDestroy(e);
    }
};

// Defaults of gd_device_config (gdlog_b200.h); the library reads no
// environment variables.
inline gd_device_config default_device_config() {
    gd_device_config d{};
    d.size = sizeof(gd_device_config);
    d.resident_loop = 1;
    d.loop_mode = GD_LOOP_GRAPH;
    d.loop_batch = 16;
    d.min_capacities = 0;
    d.split_insert = 0;
    d.dense_inner = 1;
    d.index_growth = 8;
    d.insert_waves = 0;
    d.rehash_cas_only = 0;
    d.zone_slots = 4096;
    d.partition_loop = 1;
    d.hash_dedup = 1;
    d.hash_dedup_min_rows = 1u << 20;
    d.dedup_part_slots = 8u << 20;
    d.dedup_split = 1;
    d.host_unpack = 1;
    d.download_direct_frac = 0.0;
    d.download_chunk_rows = 1u << 20;
    d.sort_items = 16;
    d.trace = 0;
    d.warp_expand = 1;
    d.sort_digit_bits = 10;
    d.heavy_rows = 4096;
    d.sort_pipeline = 0;
    d.partition_exchange = GD_EXCHANGE_PEER;
    d.sort_pipeline_min_keys = 1u << 20;
    d.temp_limit_rows = 0;
    d.peer_timeout_ms = 60000;
    d.insert_slots = 1;
    d.insert_pipeline = 0;
    d.insert_per_thread = 8;
    d.sort_ballot = 12;
    d.l2_fetch_bytes = 0;
    d.sort_min_ctas = 0;
    d.expand_keys_per_lane = 4;
    d.warp_append = 0;
    d.precount = 0;
    d.count_ctas_per_sm = 0;
    d.download_delta = 2;
    d.download_pipeline = 0;
    d.download_pipeline_min_rows = 1ull << 24;
    d.gate_in_insert = 1;
    d.pdl = 0;
    d.count_ahead = 0;
    d.log_growth = 4;
    return d;
}

struct Ctx {
    Profiler prof;
    gd_device_config cfg = default_device_config();
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int num_sms = 148;
    std::string err;
    std::string phase;
    uint64_t launches = 0;
    uint64_t bytes_in_use = 0;
    uint64_t bytes_peak = 0;
    const char* cur_phase = "other";  // for device-OOM -> budget_error(phase)
    unsigned long long* pinned = nullptr;  // small pinned readback area
    static constexpr int kPinnedWords = 64;
    void* pinned_big = nullptr;  // lazily allocated pinned area (loop control block)
    static constexpr size_t kPinnedBig = 64 << 10;
    void* pinned_area() {
        if (!pinned_big) GD_CUDA(cudaMallocHost(&pinned_big, kPinnedBig));
        return pinned_big;
    }
    // Pinned staging for chunked host downloads (kept for the context's life).
    void* staging = nullptr;
    size_t staging_bytes = 0;
    void* pinned_staging(size_t bytes) {
        if (staging_bytes < bytes) {
            if (staging) cudaFreeHost(staging);
            staging = nullptr;
            GD_CUDA(cudaMallocHost(&staging, bytes));
            staging_bytes = bytes;
        }
        return staging;
    }

    Ctx(int dev, void* s) : device(dev) {
        int n = 0;
        GD_CUDA(cudaGetDeviceCount(&n));
        if (n <= 0) throw Error(GD_ERR_CUDA, "no CUDA device present (no CPU fallback)");
        GD_CUDA(cudaSetDevice(dev));
        cudaDeviceProp prop;
        GD_CUDA(cudaGetDeviceProperties(&prop, dev));
        if (prop.major < 10)
            throw Error(GD_ERR_CUDA, std::string("device ") + prop.name +
                                         " is not sm_100-class; this build targets sm_100a only");
        num_sms = prop.multiProcessorCount;
        if (s) {
            stream = static_cast<cudaStream_t>(s);
        } else {
            GD_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
            own_stream = true;
        }
        GD_CUDA(cudaMallocHost(&pinned, kPinnedWords * sizeof(unsigned long long)));
        query_free();
    }
    ~Ctx() {
        flush_cache();
        cudaStreamSynchronize(stream);
        for (auto& kv : live_) cudaFree(kv.first);
        live_.clear();
        cudaStreamSynchronize(stream);
        if (pinned) cudaFreeHost(pinned);
        if (pinned_big) cudaFreeHost(pinned_big);
        if (staging) cudaFreeHost(staging);
        if (own_stream && stream) cudaStreamDestroy(stream);
    }
    Ctx(const Ctx&) = delete;
    Ctx& operator=(const Ctx&) = delete;

    // host-side counters (gd_ctx_host_counters): time spent in the
    // allocator and in stream synchronizations
    double alloc_seconds = 0, sync_seconds = 0;
    uint64_t alloc_count = 0, sync_count = 0;

    static double now_s() {
        timespec ts;
        clock_gettime(CLOCK_MONOTONIC, &ts);
        return ts.tv_sec + ts.tv_nsec * 1e-9;
    }

    // Stream-ordered caching allocator.  All work of a context is on one
    // stream, so a block released here may be handed out again at once:
    // any later use is ordered after the earlier one.  Sizes are rounded to
    // size classes (powers of two below 1 MiB, 1/8-octave steps above) and
    // reused from a per-class free list; cudaMallocAsync is only reached on
    // a miss, and the cache is flushed back to the pool before an
    // allocation is declared out of memory.
    std::multimap<size_t, void*> cache_;     // size class -> free blocks
    std::map<void*, size_t> live_;           // block -> size class
    uint64_t cached_bytes = 0;

    static size_t size_class(size_t bytes) {
        if (bytes <= 256) return 256;
        if (bytes <= (1u << 20)) {
            size_t c = 256;
            while (c < bytes) c <<= 1;
            return c;
        }
        size_t top = 1u << 20;
        while (top * 2 <= bytes) top <<= 1;
        const size_t step = top / 8;
        return (bytes + step - 1) / step * step;
    }

    // Bytes a new allocation could get: free device memory plus the blocks
    // cached here (alloc() returns them to the pool before giving up).
    // cudaMemGetInfo is an RM query that sporadically takes 10-100 ms on
    // the B200 boxes (the growth-time spikes of DESIGN.md §7), so free
    // memory is queried at context creation and then tracked through this
    // allocator's own cudaMalloc / cudaFree; exact = true re-queries (growth
    // near the memory limit, where other allocations in the process matter).
    mutable double meminfo_seconds = 0;
    mutable uint64_t free_est = 0;
    uint64_t available_bytes(bool exact = false) const {
        if (exact) query_free();
        return free_est + cached_bytes;
    }
    void query_free() const {
        size_t fr = 0, tot = 0;
        const double t0 = now_s();
        const cudaError_t e = cudaMemGetInfo(&fr, &tot);
        meminfo_seconds += now_s() - t0;
        free_est = e == cudaSuccess ? (uint64_t)fr : 0;
    }

    void flush_cache() {
        if (!cache_.empty()) cudaStreamSynchronize(stream);  // cached blocks may still be in use
        for (auto& kv : cache_) cudaFree(kv.second), free_est += kv.first;
        cache_.clear();
        cached_bytes = 0;
    }

    void* alloc(size_t bytes) {
        if (bytes == 0) bytes = 16;
        const size_t cls = size_class(bytes);
        const double t0 = now_s();
        ++alloc_count;
        void* p = nullptr;
        // exact size class from the cache; else a new block; when HBM is
        // exhausted, the smallest cached block up to 2x (a different workload
        // on the same context), and only then flush the cache and retry
        auto take = [&](std::multimap<size_t, void*>::iterator it) {
            p = it->second;
            const size_t got = it->first;
            cache_.erase(it);
            cached_bytes -= got;
            alloc_seconds += now_s() - t0;
            live_[p] = got;
            bytes_in_use += got;
            if (bytes_in_use > bytes_peak) bytes_peak = bytes_in_use;
            return p;
        };
        auto it = cache_.find(cls);
        if (it != cache_.end()) return take(it);
        // plain cudaMalloc: blocks live in this cache for the context's
        // life; pool (cudaMallocAsync) memory showed erratic speed for
        // large fills/copies in some processes
        cudaError_t e = cudaMalloc(&p, cls);
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            auto fit = cache_.lower_bound(cls);
            if (fit != cache_.end() && fit->first <= 2 * cls) return take(fit);
            flush_cache();
            e = cudaMalloc(&p, cls);
        }
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            alloc_seconds += now_s() - t0;
            throw_budget(cur_phase, "device allocation of " + std::to_string(bytes) +
                                        " bytes failed (HBM exhausted)");
        }
        if (e != cudaSuccess) throw Error(GD_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
        free_est -= std::min<uint64_t>(free_est, cls);
        alloc_seconds += now_s() - t0;
        live_[p] = cls;
        bytes_in_use += cls;
        if (bytes_in_use > bytes_peak) bytes_peak = bytes_in_use;
        return p;
    }
    void free(void* p, size_t /*bytes*/) {
        if (!p) return;
        auto it = live_.find(p);
        if (it == live_.end()) {
            cudaStreamSynchronize(stream);
            cudaFree(p);
            return;
        }
        const size_t cls = it->second;
        live_.erase(it);
        bytes_in_use -= cls;
        cache_.emplace(cls, p);
        cached_bytes += cls;
    }
    void sync() {
        const double t0 = now_s();
        GD_CUDA(cudaStreamSynchronize(stream));
        sync_seconds += now_s() - t0;
        ++sync_count;
    }

    // Instrumented launch bracket: t = prof_begin(); <launch>; prof_end(t, ...).
    cudaEvent_t prof_begin() {
        if (!prof.on) return nullptr;
        cudaEvent_t a = prof.take();
        cudaEventRecord(a, stream);
        return a;
    }
    // Returns the index of the pending record (to patch bytes later) or -1.
    long prof_end(cudaEvent_t a, int cls, uint64_t bytes) {
        if (!a) return -1;
        cudaEvent_t b = prof.take();
        cudaEventRecord(b, stream);
        prof.pending.push_back({cls, a, b, bytes});
        return (long)prof.pending.size() - 1;
    }
    void prof_add_bytes(long rec, uint64_t bytes) {
        if (rec >= 0 && rec < (long)prof.pending.size()) prof.pending[rec].bytes += bytes;
    }
    void check_launch() {
        ++launches;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw Error(GD_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
    }
    void memset(void* p, int v, size_t bytes) {
        if (bytes) GD_CUDA(cudaMemsetAsync(p, v, bytes, stream));
    }
    uint64_t h2d_bytes = 0, d2h_bytes = 0;  // gd_ctx_transfer_bytes
    void h2d(void* d, const void* h, size_t bytes) {
        if (bytes) GD_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, stream));
        h2d_bytes += bytes;
    }
    void d2h(void* h, const void* d, size_t bytes) {
        if (bytes) GD_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, stream));
        d2h_bytes += bytes;
    }
    void d2d(void* d, const void* s, size_t bytes) {
        if (bytes) GD_CUDA(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice, stream));
    }
    // Reads `n` (<= kPinnedWords) device words through pinned memory; syncs.
    void read_words(unsigned long long* out, const void* d, int n) {
        d2h(pinned, d, n * sizeof(unsigned long long));
        sync();
        for (int i = 0; i < n; ++i) out[i] = pinned[i];
    }
    // Two scattered device words with one synchronization.
    void read2(unsigned long long* a, const void* da, unsigned long long* b, const void* db) {
        d2h(pinned, da, sizeof(unsigned long long));
        d2h(pinned + 1, db, sizeof(unsigned long long));
        sync();
        *a = pinned[0];
        *b = pinned[1];
    }
};

// RAII device buffer of T elements from the context pool.
template <typename T>
struct DevBuf {
    Ctx* ctx = nullptr;
    T* p = nullptr;
    uint64_t cap = 0;  // elements

    DevBuf() = default;
    DevBuf(Ctx& c, uint64_t n) : ctx(&c), p(static_cast<T*>(c.alloc(n * sizeof(T)))), cap(n) {}
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : ctx(o.ctx), p(o.p), cap(o.cap) { o.p = nullptr; o.cap = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            ctx = o.ctx; p = o.p; cap = o.cap;
            o.p = nullptr; o.cap = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void release() {
        if (p && ctx) ctx->free(p, cap * sizeof(T));
        p = nullptr;
        cap = 0;
    }
    // Ensures capacity >= n (contents NOT preserved).
    void reserve_discard(Ctx& c, uint64_t n) {
        if (cap >= n && p) return;
        release();
        ctx = &c;
        p = static_cast<T*>(c.alloc((n ? n : 1) * sizeof(T)));
        cap = n ? n : 1;
    }
    void swap(DevBuf& o) noexcept {
        std::swap(ctx, o.ctx);
        std::swap(p, o.p);
        std::swap(cap, o.cap);
    }
};

}  // namespace gd
