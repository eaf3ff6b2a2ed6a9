// engine.cu — the semi-naive fixpoint driver on the device
// (engine::seed / iterate_to_fixpoint / refresh_copies / execute_chain /
// merge_into_full, engine.hpp:137-542), templated on the packed key type.
//
// Per iteration, for every recursive relation:
//   join   : join_probe (fused count+scan) + load-balanced materialize,
//            written straight into the head's new-tuple accumulator;
//   dedup  : onesweep radix sort of the accumulator (only significant bits);
//   diff+merge: ONE merge-path pass: F' = F U N and Δ = unique(N) \ F
//            (the adjacent-unique of canonicalize, difference and
//            merge_sorted of the reference fused), into ping-pong buffers.
// Indexed copies with a non-identity permutation are maintained
// incrementally (sorted permuted Δ merged into the copy)
// and their HISA index rebuilt; identity copies alias the full relation.
// The logical-byte accountant and EBM bookkeeping replay the reference's
// charges in the same order (accounting.h).
#include <cstdlib>
#include <cstring>
#include <set>
#include <atomic>
#include <functional>
#include <memory>
#include <optional>
#include <mutex>
#include <thread>
#include <type_traits>
#if defined(__x86_64__)
#include <immintrin.h>
#endif

#include "engine.h"
#include "host_decode.h"
#include "comm.h"
#include "loop.h"
#include "ops.h"

namespace gd {

namespace {

inline u64 rb(u64 rows, u32 arity) { return rows * arity * 8ull; }  // tuple_array::byte_size

inline bool is_identity(const u32* p, u32 k) {
    for (u32 i = 0; i < k; ++i)
        if (p[i] != i) return false;
    return true;
}

using CopyKey = std::pair<std::vector<u32>, u32>;

// Grows a device buffer to hold `need` elements, preserving the first
// `keep` elements.
template <typename K>
void ensure_keep(Ctx& c, DevBuf<K>& b, u64 need, u64 keep) {
    if (b.p && b.cap >= need) return;
    u64 cap = std::max<u64>(need + need / 4, 1024);
    DevBuf<K> nb(c, cap);
    if (keep && b.p) c.d2d(nb.p, b.p, keep * sizeof(K));
    b = std::move(nb);
}
template <typename K>
void ensure_discard(Ctx& c, DevBuf<K>& b, u64 need) {
    if (b.p && b.cap >= need) return;
    b.reserve_discard(c, std::max<u64>(need + need / 4, 1024));
}

template <typename K>
struct CopyState {
    std::vector<u32> perm;
    u32 prefix = 0;
    bool identity = false;
    DevBuf<K> rows, alt;
    u64 n = 0;
    DevIndex<K> index;
    u64 bytes = 0;  // accounted container bytes (engine.hpp:44-47)
    bool built = false;
    u64 synced_gen = 0;
};

template <typename K>
struct Run {
    DevBuf<K> buf;
    u64 n = 0;
};

// Tier ratio of the tiered (LSM) full relation: every run holds at least
// kTierRatio times the rows of the next smaller one.
constexpr u64 kTierRatio = 4;

// Segmented final sort with the download packed per segment
// (gd_device_config.download_pipeline): the loop's log is
// sorted by its top digit first (one stable pass), then every top-digit
// segment by its low digits, and each sorted segment is byte-offset packed
// (delta.cu byte_pack_into) into the other sort buffer with an event
// recorded behind it — a host download then copies and rebuilds segment s
// while the device still sorts the segments after it.
struct PipedPack {
    const u64* keys = nullptr;  // the sorted relation this pack belongs to (RelDev::full)
    u64 n = 0;
    DevBuf<u64> spare;          // the other sort buffer: segment s's payload at byte 8 * key_off
    DevBuf<u64> heads, offs, uoffs;
    DevBuf<uint8_t> cls;
    struct Seg {
        u64 key_off, cnt;    // rows [key_off, key_off + cnt)
        u64 blk_off, nblk;   // heads / cls entries (offs: blk_off + index, nblk + 1 of them)
        u64 unit_off, nunits;  // uoffs: unit_off + index, nunits + 1 entries
    };
    std::vector<Seg> segs;
    std::vector<cudaEvent_t> ev;  // ev[s]: segment s sorted and packed (context stream)
    static constexpr u64 kUnitB = 8192;  // blocks of 32 keys per download unit
    PipedPack() = default;
    PipedPack(const PipedPack&) = delete;
    PipedPack& operator=(const PipedPack&) = delete;
    ~PipedPack() {
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
    }
};

template <typename K>
struct RelDev {
    std::unique_ptr<PipedPack> piped;  // set by the resident loop's segmented final sort
    // full relation = `full` (the base run) U every run of `tail`; all
    // sorted and pairwise disjoint.  `tail` stays empty unless `lsm`.
    DevBuf<K> full, full_alt;
    u64 full_n = 0;
    std::vector<Run<K>> tail;
    bool lsm = false;
    DevBuf<K> delta, delta_alt;
    u64 delta_n = 0;
    DevBuf<K> new_acc;
    u64 new_n = 0;
    u64 last_unique = 0;  // distinct join rows of the last iteration (hash pre-dedup sizing)
    std::map<CopyKey, CopyState<K>> copies;
    bool dirty = true;
    u64 merge_gen = 0;
    bool last_merge_was_delta = false;
};

template <typename K>
class Impl final : public ImplBase {
public:
    explicit Impl(Engine& e) : E(e), c(e.c), bits(e.enc.e.bits) {
        const u32 nrels = (u32)E.info_.size();
        rels.resize(nrels);
        // Constant encodings (every plan constant is in the dictionary).
        for (const auto& p : E.plans_) for_each_constant(p, [&](u64 v) { encode_const(v); });
        // Indexed copies registered by set_plans (engine.hpp:300-310).
        for (const auto& p : E.plans_)
            for (u32 v = 0; v < p.nvariants; ++v)
                for (u32 s = 0; s < p.variants[v].nsteps; ++s) {
                    const gd_join_step& st = p.variants[v].steps[s];
                    const u32 ar = E.info_[st.inner_rel].arity;
                    CopyKey key{std::vector<u32>(st.inner_perm, st.inner_perm + ar), st.join_column_count};
                    auto& cp = rels[st.inner_rel].copies[key];
                    cp.perm = key.first;
                    cp.prefix = key.second;
                    cp.identity = is_identity(st.inner_perm, ar);
                }
        // Relations that are never a join inner (no indexed copy) keep their
        // full version tiered: Δ is appended as a small sorted run and runs
        // are merged (merge-path) only when a run reaches 1/kTierRatio of its
        // larger neighbour — the per-iteration O(|F|) merge of the reference
        // becomes O(|F| log |F|) over the whole fixpoint.
        for (u32 r = 0; r < nrels; ++r) rels[r].lsm = !E.info_[r].is_edb && rels[r].copies.empty();
        // EDB rows: pack under the engine encoding; order is preserved, so
        // canonical raw rows stay canonical (no re-sort).
        for (u32 r = 0; r < nrels; ++r) {
            if (!E.info_[r].is_edb) continue;
            const u64 n = E.raw_n[r];
            auto& st = rels[r];
            ensure_discard(c, st.full, n);
            if (n) pack_rows<K>(c, E.raw[r].p, n, E.info_[r].arity, E.enc.e, st.full.p);
            st.full_n = n;
            E.raw[r].release();
        }
    }

    // ------------------------------------------------------------------
    void seed() override {
        const u64 join0 = E.join_tuples;
        // nonrecursive_topo_order, engine.hpp:322-353
        std::vector<u32> nonrec;
        for (u32 i = 0; i < E.plans_.size(); ++i)
            if (!E.plans_[i].recursive) nonrec.push_back(i);
        std::vector<bool> done(nonrec.size(), false);
        size_t ndone = 0;
        while (ndone < nonrec.size()) {
            bool progressed = false;
            for (size_t i = 0; i < nonrec.size(); ++i) {
                if (done[i]) continue;
                const gd_rule_plan& pi = E.plans_[nonrec[i]];
                bool ready = true;
                for (size_t j = 0; j < nonrec.size() && ready; ++j) {
                    if (done[j] || j == i) continue;
                    const u32 h = E.plans_[nonrec[j]].head_rel;
                    if (!E.info_[h].is_edb && reads(pi, h)) ready = false;
                }
                if (!ready) continue;
                done[i] = true;
                ++ndone;
                progressed = true;
                seed_rule(pi);
            }
            if (!progressed) throw_logic("nonrecursive rules form a dependency cycle");
        }
        // delta := full for every IDB (engine.hpp:170-174)
        for (u32 r = 0; r < rels.size(); ++r) {
            if (E.info_[r].is_edb) continue;
            auto& st = rels[r];
            compact(st);
            ensure_discard(c, st.delta, st.full_n);
            if (st.full_n) c.d2d(st.delta.p, st.full.p, st.full_n * sizeof(K));
            assign_delta(r, st.full_n, "other");
            st.delta_n = st.full_n;
        }
        check_temp_watermark();
        if (E.nranks > 1) {
            keep_owned();
            // every rank ran the seed rules on the replicated EDB: rank 0
            // alone reports their join tuples, so the ranks' sum is the
            // single engine's count
            if (E.rank != 0) E.join_tuples = join0;
        }
    }

    // Partitioned mode: each rank keeps the IDB tuples it owns
    // (owner = hash(tuple) % nranks); EDB relations stay replicated.
    void keep_owned() {
        for (u32 r = 0; r < rels.size(); ++r) {
            if (E.info_[r].is_edb) continue;
            auto& st = rels[r];
            compact(st);
            if (st.full_n == 0) continue;
            DevBuf<u32> own(c, st.full_n);
            DevBuf<uint8_t> flags(c, st.full_n);
            owner_of<K>(c, st.full.p, st.full_n, E.nranks, own.p);
            owner_flags(c, own.p, st.full_n, E.rank, flags.p);
            DevBuf<K> kept(c, st.full_n);
            const u64 m = compact_flagged<K>(c, st.full.p, flags.p, st.full_n, kept.p);
            st.full.swap(kept);
            st.full_n = m;
            ensure_discard(c, st.delta, m);
            if (m) c.d2d(st.delta.p, st.full.p, m * sizeof(K));
            st.delta_n = m;
        }
    }

    void iterate() override {
        std::vector<u32> rec;
        for (const auto& p : E.plans_)
            if (p.recursive && std::find(rec.begin(), rec.end(), p.head_rel) == rec.end()) rec.push_back(p.head_rel);
        // refresh order = the reference's name-keyed map order
        std::vector<u32> by_name(rels.size());
        for (u32 i = 0; i < by_name.size(); ++i) by_name[i] = i;
        std::sort(by_name.begin(), by_name.end(),
                  [&](u32 a, u32 b) { return E.info_[a].name < E.info_[b].name; });
        if constexpr (std::is_same_v<K, u64>) {
            if (loop_eligible(rec)) {
                iterate_loop(rec, by_name);
                return;
            }
        }

        for (;;) {
            bool active = false;
            for (u32 r : rec) active |= rels[r].delta_n > 0;
            if (!active) break;
            ++E.iterations;
            std::vector<u64> delta_in(rec.size());
            for (size_t i = 0; i < rec.size(); ++i) {
                delta_in[i] = rels[rec[i]].delta_n;
                E.info_[rec[i]].history.push_back(delta_in[i]);
            }
            // (1) refresh indexed copies
            for (u32 r : by_name)
                if (rels[r].dirty) refresh_copies(r);
            // (2) every variant of every recursive rule on the deltas
            std::vector<u64> joined(rels.size(), 0);
            for (const auto& p : E.plans_) {
                if (!p.recursive) continue;
                auto& head = rels[p.head_rel];
                for (u32 v = 0; v < p.nvariants; ++v) {
                    const gd_variant& var = p.variants[v];
                    if (var.src_version == GD_DELTA && rels[var.src_rel].delta_n == 0) continue;
                    u64 m = 0;
                    execute_chain(var, head.new_acc, head.new_n, &m);
                    joined[p.head_rel] += m;
                    append_new(p.head_rel, m);
                }
                check_temp_watermark();
            }
            // (3) dedup, (4) difference, (5) merge — fused
            for (size_t i = 0; i < rec.size(); ++i) {
                const u32 r = rec[i];
                gd_iter_record log{delta_in[i], joined[r], 0, 0, 0};
                dedup_diff_merge(r, log);
                E.info_[r].log.push_back(log);
            }
        }
        // the fixpoint's canonical output: one sorted array per relation
        for (auto& st : rels) compact(st);
    }

    bool output_pending() const override {
        for (const auto& st : rels)
            if (st.piped) return true;
        return false;
    }

    u64 count(u32 r) override {
        if (pl && pl->heads[0].rel == r) return pl->hc->h[0].log_n;
        return total_n(rels[r]);
    }

    void download(u32 r, u64* out, bool device) override {
        if (pl) part_loop_finish();
        auto& st = rels[r];
        compact(st);
        const u32 ar = E.info_[r].arity;
        if (st.full_n == 0) return;
        if (device) {
            unpack_rows<K>(c, st.full.p, st.full_n, ar, E.enc.e, out);
            c.sync();
            return;
        }
        if constexpr (std::is_same_v<K, u64>) {
            if (!E.enc.e.dict && ar > 1 && st.full_n >= (1u << 20) &&
                c.cfg.host_unpack) {
                // (packing per fixed-size chunk with an event behind each, so the
                // host starts before the device has packed everything, measured
                // 83-87 ms vs 81-85 ms: the host rebuild bounds it, and the issuing
                // thread is one rebuilding thread fewer)
                std::unique_ptr<PipedPack> pp = std::move(st.piped);
                if (pp && pp->keys == st.full.p && pp->n == st.full_n && st.tail.empty() &&
                    c.cfg.download_delta == 2 && c.cfg.download_direct_frac == 0.0) {
                    download_piped_rows(*pp, ar, out);
                    return;
                }
                pp.reset();
                download_packed(st.full.p, st.full_n, ar, out);
                return;
            }
        }
        DevBuf<u64> tmp(c, st.full_n * ar);
        unpack_rows<K>(c, st.full.p, st.full_n, ar, E.enc.e, tmp.p);
        c.d2h(out, tmp.p, st.full_n * ar * sizeof(u64));
        c.sync();
    }

    // Host download of identity-encoded u64 keys: the packed keys cross PCIe
    // (8 B per row instead of 8·arity) into two pinned staging buffers, and
    // host threads unpack chunk k into the caller's rows while chunk k+1 is
    // in flight.  Bytes equal unpack_rows + copy.
    void download_packed(const u64* keys, u64 n_all, u32 ar, u64* out) {
        // Into a pinned destination, the tail rows [n, n_all) are unpacked on
        // the device and DMA'd straight into the caller's rows on a second
        // stream while the host unpacks the packed head: PCIe carries 16 B
        // per direct row, host memory 16 B instead of 32 (staging write +
        // read + row write), balancing the two (GD_DL_DIRECT_FRAC, 0.25).
        u64 n = n_all;
        DevBuf<u64> direct;
        cudaStream_t s2 = nullptr;
        cudaEvent_t ev_un = nullptr;
        cudaEvent_t ev[2] = {nullptr, nullptr};
        std::vector<std::thread> pool;
        std::atomic<bool> quit{false};
        // Runs on every exit, a throw included (GD_CUDA inside the chunk
        // loop): stop and join the unpack threads, drain both streams so no
        // DMA still reads `direct` or writes the staging area, then release
        // the events and the side stream; `direct` (declared earlier) is
        // freed after this.
        struct Cleanup {
            std::function<void()> f;
            ~Cleanup() { f(); }
        } cleanup{[&] {
            quit.store(true, std::memory_order_release);
            for (auto& th : pool)
                if (th.joinable()) th.join();
            if (s2) {
                cudaStreamSynchronize(s2);
                cudaStreamDestroy(s2);
            }
            cudaStreamSynchronize(c.stream);
            if (ev_un) cudaEventDestroy(ev_un);
            for (auto e : ev)
                if (e) cudaEventDestroy(e);
            cudaGetLastError();
        }};
        {
            const double frac = c.cfg.download_direct_frac;
            cudaPointerAttributes pa{};
            const bool pinned = cudaPointerGetAttributes(&pa, out) == cudaSuccess && pa.type == cudaMemoryTypeHost;
            cudaGetLastError();
            const u64 nd = pinned && frac > 0 && frac < 1 ? (u64)((double)n_all * frac) : 0;
            if (nd && nd * ar * sizeof(u64) + (1ull << 30) < c.available_bytes()) {
                n = n_all - nd;
                direct = DevBuf<u64>(c, nd * ar);
                unpack_rows<u64>(c, keys + n, nd, ar, E.enc.e, direct.p);
                GD_CUDA(cudaEventCreateWithFlags(&ev_un, cudaEventDisableTiming));
                GD_CUDA(cudaEventRecord(ev_un, c.stream));
                GD_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
                GD_CUDA(cudaStreamWaitEvent(s2, ev_un, 0));
                GD_CUDA(cudaMemcpyAsync(out + n * ar, direct.p, nd * ar * sizeof(u64), cudaMemcpyDeviceToHost, s2));
                c.d2h_bytes += nd * ar * sizeof(u64);
            }
        }
        const bool trace = (c.cfg.trace & 2) != 0;
        double t_wait = 0, t_unpack = 0;
        const unsigned hw = std::thread::hardware_concurrency();
        const unsigned nt = std::max(1u, std::min(hw ? hw : 8u, 32u));
        if (c.cfg.download_delta == 2 && n > 0 && c.cfg.download_overlap_pack &&
            n * sizeof(u64) + (1ull << 30) < c.available_bytes()) {
            download_bytes_rows_overlap(keys, n, ar, out, nt, t_wait, t_unpack);
        } else if (c.cfg.download_delta == 2 && n > 0) {
            download_bytes_rows(keys, n, ar, out, nt, t_wait, t_unpack);
        } else if (c.cfg.download_delta == 1 && n > 0) {
            download_delta_rows(keys, n, ar, out, nt, t_wait, t_unpack);
        } else {
        const u64 kChunk = c.cfg.download_chunk_rows;
        u64* stage[2];
        void* area = c.pinned_staging(2 * kChunk * sizeof(u64));
        stage[0] = static_cast<u64*>(area);
        stage[1] = stage[0] + kChunk;
        GD_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
        GD_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
        const u32 bits = E.enc.e.bits;
        const u64 mask = bits >= 64 ? ~0ull : (1ull << bits) - 1;
        const u64 nchunks = (n + kChunk - 1) / kChunk;
        auto issue = [&](u64 k) {
            const u64 b = k * kChunk, m = std::min(kChunk, n - b);
            c.d2h(stage[k & 1], keys + b, m * sizeof(u64));
            GD_CUDA(cudaEventRecord(ev[k & 1], c.stream));
        };
        // one pool of nt threads for the whole download; chunk k is handed
        // out by a generation counter once its copy has landed
        std::atomic<u64> gen{0};
        std::atomic<unsigned> left{0};
        const u64* cur_src = nullptr;
        u64* cur_dst = nullptr;
        u64 cur_m = 0;
        auto unpack = [&](unsigned t) {
            const u64 m = cur_m, lo = m * t / nt, hi = m * (t + 1) / nt;
            const u64* src = cur_src;
            u64* dst = cur_dst;
            if (ar == 2) {
#if defined(__x86_64__)
                // non-temporal stores: the rows are written once and not read
                // back here, so skip the read-for-ownership of each line
                long long* d = reinterpret_cast<long long*>(dst);
                u64 i = lo;
                if (!(reinterpret_cast<uintptr_t>(dst) & 15)) {
                    // two rows per step: one 16-byte load of two keys, two
                    // 16-byte non-temporal row stores
                    const __m128i mv = _mm_set1_epi64x((long long)mask);
                    const __m128i sh = _mm_cvtsi32_si128((int)bits);
                    for (; i + 2 <= hi; i += 2) {
                        const __m128i k = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
                        const __m128i a = _mm_and_si128(_mm_srl_epi64(k, sh), mv);
                        const __m128i b = _mm_and_si128(k, mv);
                        _mm_stream_si128(reinterpret_cast<__m128i*>(d + 2 * i), _mm_unpacklo_epi64(a, b));
                        _mm_stream_si128(reinterpret_cast<__m128i*>(d + 2 * i + 2), _mm_unpackhi_epi64(a, b));
                    }
                }
                for (; i < hi; ++i) {
                    const u64 key = src[i];
                    _mm_stream_si64(d + 2 * i, (long long)((key >> bits) & mask));
                    _mm_stream_si64(d + 2 * i + 1, (long long)(key & mask));
                }
                _mm_sfence();
#else
                for (u64 i = lo; i < hi; ++i) {
                    const u64 key = src[i];
                    dst[2 * i] = (key >> bits) & mask;
                    dst[2 * i + 1] = key & mask;
                }
#endif
            } else {
                for (u64 i = lo; i < hi; ++i) {
                    const u64 key = src[i];
                    for (u32 col = 0; col < ar; ++col) dst[i * ar + col] = (key >> ((ar - 1 - col) * bits)) & mask;
                }
            }
        };
        for (unsigned t = 1; t < nt; ++t)
            pool.emplace_back([&, t] {
                u64 seen = 0;
                while (true) {
                    u64 g;
                    while ((g = gen.load(std::memory_order_acquire)) == seen && !quit.load(std::memory_order_acquire))
                        std::this_thread::yield();
                    if (quit.load(std::memory_order_acquire)) return;
                    seen = g;
                    unpack(t);
                    left.fetch_sub(1, std::memory_order_acq_rel);
                }
            });
        issue(0);
        for (u64 k = 0; k < nchunks; ++k) {
            const double tw = Ctx::now_s();
            GD_CUDA(cudaEventSynchronize(ev[k & 1]));
            t_wait += Ctx::now_s() - tw;
            const double tu = Ctx::now_s();
            if (k + 1 < nchunks) issue(k + 1);  // staging[(k+1)&1] was unpacked at step k-1
            const u64 b = k * kChunk;
            cur_m = std::min(kChunk, n - b);
            cur_src = stage[k & 1];
            cur_dst = out + b * ar;
            left.store(nt - 1, std::memory_order_release);
            gen.fetch_add(1, std::memory_order_acq_rel);
            unpack(0);
            while (left.load(std::memory_order_acquire) != 0) std::this_thread::yield();
            t_unpack += Ctx::now_s() - tu;
        }
        quit.store(true, std::memory_order_release);
        for (auto& th : pool) th.join();
        pool.clear();
        }
        double t_direct = 0;
        if (s2) {
            const double td = Ctx::now_s();
            GD_CUDA(cudaStreamSynchronize(s2));
            t_direct = Ctx::now_s() - td;
        }
        if (trace)
            fprintf(stderr,
                    "[download] %llu rows (%llu direct), %u threads: waiting on PCIe %.1f ms, unpacking %.1f ms, "
                    "direct tail %.1f ms\n",
                    (unsigned long long)n_all, (unsigned long long)(n_all - n), nt, t_wait * 1e3, t_unpack * 1e3,
                    t_direct * 1e3);
    }

    // Download of a segment-packed relation (PipedPack): the calling thread
    // issues, segment by segment as each one's event completes, the copies of
    // its units (heads | classes | payload) on a side stream into a ring of
    // pinned staging areas; nt - 1 threads claim units in order and rebuild
    // their rows (host_decode.cpp) — so the host rebuild of segment s overlaps
    // the device sort of the segments after it.
    void download_piped_rows(PipedPack& pp, u32 ar, u64* out) {
        const bool trace = (c.cfg.trace & 2) != 0;
        const double t_start = Ctx::now_s();
        constexpr u64 kUnitB = PipedPack::kUnitB;
        const u64 nseg = pp.segs.size();
        u64 nunits = 0;
        for (const auto& sg : pp.segs) nunits += sg.nunits;

        struct Unit { u64 seg, j; };
        std::vector<Unit> units;
        units.reserve(nunits);
        for (u64 sgi = 0; sgi < nseg; ++sgi)
            for (u64 j = 0; j < pp.segs[sgi].nunits; ++j) units.push_back({sgi, j});
        const u64 R = std::min<u64>(std::max<u64>(nunits, 1), 32);
        auto up = [](u64 v) { return (v + 63) & ~63ull; };
        const u64 a_heads = kUnitB * sizeof(u64), a_cls = up(kUnitB);
        const u64 area = a_heads + a_cls + up(kUnitB * kByteBlock * sizeof(u64) + 64);
        // pinned: the ring of staging areas, then every segment's unit offsets
        uint8_t* stage = static_cast<uint8_t*>(c.pinned_staging(R * area + (nunits + nseg) * sizeof(u64)));
        u64* uo = reinterpret_cast<u64*>(stage + R * area);  // per segment: its nunits + 1 unit offsets
        const uint8_t* payload = reinterpret_cast<const uint8_t*>(pp.spare.p);
        cudaStream_t s2 = nullptr, sm = nullptr;
        std::vector<cudaEvent_t> ev(R, nullptr), evm(nseg, nullptr);
        std::unique_ptr<std::atomic<int>[]> issued(new std::atomic<int>[nunits + 1]);
        std::unique_ptr<std::atomic<int>[]> finished(new std::atomic<int>[nunits + 1]);
        for (u64 u = 0; u <= nunits; ++u) {
            issued[u].store(0);
            finished[u].store(0);
        }
        std::atomic<u64> next{0};
        std::atomic<bool> quit{false};
        std::exception_ptr err;
        std::mutex err_mu;
        std::vector<std::thread> pool;
        struct Cleanup {
            std::function<void()> f;
            ~Cleanup() { f(); }
        } cleanup{[&] {
            quit.store(true, std::memory_order_release);
            for (auto& th : pool)
                if (th.joinable()) th.join();
            if (s2) {
                cudaStreamSynchronize(s2);
                cudaStreamDestroy(s2);
            }
            if (sm) {
                cudaStreamSynchronize(sm);
                cudaStreamDestroy(sm);
            }
            cudaStreamSynchronize(c.stream);
            for (auto e : ev)
                if (e) cudaEventDestroy(e);
            for (auto e : evm)
                if (e) cudaEventDestroy(e);
            cudaGetLastError();
        }};
        GD_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        GD_CUDA(cudaStreamCreateWithFlags(&sm, cudaStreamNonBlocking));
        for (auto& e : ev) GD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        // every segment's unit offsets are requested up front on their own
        // stream (each behind its segment's event), so reading them never
        // queues behind the unit copies already in flight
        for (u64 sgi = 0; sgi < nseg; ++sgi) {
            const PipedPack::Seg& sg = pp.segs[sgi];
            GD_CUDA(cudaEventCreateWithFlags(&evm[sgi], cudaEventDisableTiming));
            GD_CUDA(cudaStreamWaitEvent(sm, pp.ev[sgi], 0));
            GD_CUDA(cudaMemcpyAsync(uo + sg.unit_off + sgi, pp.uoffs.p + sg.unit_off + sgi,
                                    (sg.nunits + 1) * sizeof(u64), cudaMemcpyDeviceToHost, sm));
            GD_CUDA(cudaEventRecord(evm[sgi], sm));
        }
        const u32 bits = E.enc.e.bits;
        auto worker = [&] {
            try {
                while (!quit.load(std::memory_order_acquire)) {
                    const u64 u = next.fetch_add(1, std::memory_order_acq_rel);
                    if (u >= nunits) return;
                    while (!issued[u].load(std::memory_order_acquire)) {
                        if (quit.load(std::memory_order_acquire)) return;
                        std::this_thread::yield();
                    }
                    GD_CUDA(cudaEventSynchronize(ev[u % R]));
                    const PipedPack::Seg& sg = pp.segs[units[u].seg];
                    const u64 j = units[u].j, b0 = j * kUnitB, nbu = std::min(kUnitB, sg.nblk - b0);
                    const uint8_t* a = stage + (u % R) * area;
                    byte_decode_rows(reinterpret_cast<const u64*>(a), a + a_heads, a + a_heads + a_cls,
                                     sg.key_off + b0 * kByteBlock, nbu, sg.key_off + sg.cnt, ar, bits, out);
                    finished[u].store(1, std::memory_order_release);
                }
            } catch (...) {
                std::lock_guard<std::mutex> g(err_mu);
                if (!err) err = std::current_exception();
                quit.store(true, std::memory_order_release);
            }
        };
        const unsigned hw = std::thread::hardware_concurrency();
        const unsigned nt = std::max(2u, std::min(hw ? hw : 8u, 32u));
        for (unsigned t = 1; t < nt; ++t) pool.emplace_back(worker);
        u64 bytes = 0;
        double t_seg_wait = 0;
        u64 u = 0;
        for (u64 sgi = 0; sgi < nseg && !quit.load(std::memory_order_acquire); ++sgi) {
            const PipedPack::Seg& sg = pp.segs[sgi];
            const u64* suo = uo + sg.unit_off + sgi;
            const double tw = Ctx::now_s();
            GD_CUDA(cudaEventSynchronize(evm[sgi]));
            t_seg_wait += Ctx::now_s() - tw;
            bytes += (sg.nunits + 1) * sizeof(u64);
            GD_CUDA(cudaStreamWaitEvent(s2, pp.ev[sgi], 0));
            for (u64 j = 0; j < sg.nunits; ++j, ++u) {
                if (u >= R) {  // area u % R is free once unit u - R is rebuilt
                    while (!finished[u - R].load(std::memory_order_acquire)) {
                        if (quit.load(std::memory_order_acquire)) break;
                        std::this_thread::yield();
                    }
                    if (quit.load(std::memory_order_acquire)) break;
                }
                uint8_t* a = stage + (u % R) * area;
                const u64 b0 = j * kUnitB, nbu = std::min(kUnitB, sg.nblk - b0);
                const u64 p0 = suo[j], p1 = suo[j + 1];
                GD_CUDA(cudaMemcpyAsync(a, pp.heads.p + sg.blk_off + b0, nbu * sizeof(u64), cudaMemcpyDeviceToHost,
                                        s2));
                GD_CUDA(cudaMemcpyAsync(a + a_heads, pp.cls.p + sg.blk_off + b0, nbu, cudaMemcpyDeviceToHost, s2));
                if (p1 > p0)
                    GD_CUDA(cudaMemcpyAsync(a + a_heads + a_cls, payload + sg.key_off * sizeof(u64) + p0, p1 - p0,
                                            cudaMemcpyDeviceToHost, s2));
                GD_CUDA(cudaEventRecord(ev[u % R], s2));
                bytes += nbu * (sizeof(u64) + 1) + (p1 - p0);
                issued[u].store(1, std::memory_order_release);
            }
        }
        for (auto& th : pool) th.join();
        pool.clear();
        if (err) std::rethrow_exception(err);
        if (quit.load() && next.load() < nunits) throw Error(GD_ERR_CUDA, "segmented download stopped early");
        c.d2h_bytes += bytes;
        if (trace)
            fprintf(stderr, "[download] %llu rows in %llu segments (%llu units), %u threads: %.1f ms, waiting on "
                            "segments %.1f ms\n",
                    (unsigned long long)pp.n, (unsigned long long)nseg, (unsigned long long)nunits, nt,
                    (Ctx::now_s() - t_start) * 1e3, t_seg_wait * 1e3);
    }

    // Byte-offset download of n canonical keys into rows (download_delta = 2):
    // the device writes every 32-key block as its first key plus byte-aligned
    // offsets (delta.cu byte_pack; C2: ~2.5 B per row over PCIe), chunks of
    // kChunkB blocks cross PCIe into a ring of pinned staging areas, and nt
    // host threads (the caller included) claim units of kUnitB blocks in
    // order from one counter and rebuild their rows with vector loads, adds
    // and non-temporal stores (host_decode.cpp).  No barrier per chunk: a
    // unit waits only for its own chunk's copy, and the thread that finishes
    // a chunk's last unit issues the copy that reuses its staging area.
    void download_bytes_rows(const u64* keys, u64 n, u32 ar, u64* out, unsigned nt, double& t_wait,
                             double& t_unpack) {
        BytePacked d;
        byte_pack(c, keys, n, d);
        constexpr u64 kUnitB = 8192;      // blocks per unit (256 K rows)
        constexpr u64 kChunkUnits = 16;   // units per chunk (4 M rows)
        constexpr u64 kChunkB = kUnitB * kChunkUnits;
        const u64 nunits = (d.nb + kUnitB - 1) / kUnitB;
        const u64 nchunks = (nunits + kChunkUnits - 1) / kChunkUnits;
        std::vector<u64> uoff(nunits + 1);
        {
            DevBuf<u64> duo(c, nunits + 1);
            byte_unit_offsets(c, d, kUnitB, nunits, duo.p);
            c.d2h(uoff.data(), duo.p, (nunits + 1) * sizeof(u64));
            c.sync();
        }
        auto chunk_units = [&](u64 k) { return std::min(kChunkUnits, nunits - k * kChunkUnits); };
        u64 maxp = 0;
        for (u64 k = 0; k < nchunks; ++k)
            maxp = std::max(maxp, uoff[k * kChunkUnits + chunk_units(k)] - uoff[k * kChunkUnits]);
        // staging area: heads | classes | payload, 64-byte aligned parts
        auto up = [](u64 v) { return (v + 63) & ~63ull; };
        const u64 a_heads = kChunkB * sizeof(u64), a_cls = up(kChunkB), area = a_heads + a_cls + up(maxp + 64);
        const u64 R = std::min<u64>(nchunks, 6);
        uint8_t* stage = static_cast<uint8_t*>(c.pinned_staging(R * area));
        std::vector<cudaEvent_t> ev(nchunks, nullptr);
        std::unique_ptr<std::atomic<int>[]> issued(new std::atomic<int>[nchunks]);
        std::unique_ptr<std::atomic<u64>[]> finished(new std::atomic<u64>[nchunks]);
        for (u64 k = 0; k < nchunks; ++k) {
            issued[k].store(0);
            finished[k].store(0);
        }
        std::atomic<u64> next{0};
        std::atomic<bool> quit{false};
        std::atomic<u64> d2h_total{0};
        std::exception_ptr err;
        std::mutex err_mu;
        std::vector<std::thread> pool;
        struct Cleanup {
            std::function<void()> f;
            ~Cleanup() { f(); }
        } cleanup{[&] {
            quit.store(true, std::memory_order_release);
            for (auto& th : pool)
                if (th.joinable()) th.join();
            cudaStreamSynchronize(c.stream);
            for (auto e : ev)
                if (e) cudaEventDestroy(e);
            cudaGetLastError();
        }};
        for (u64 k = 0; k < nchunks; ++k) GD_CUDA(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
        auto issue = [&](u64 k) {  // chunk k into area k % R
            uint8_t* a = stage + (k % R) * area;
            const u64 b0 = k * kChunkB, nbk = std::min(kChunkB, d.nb - b0);
            const u64 p0 = uoff[k * kChunkUnits], p1 = uoff[k * kChunkUnits + chunk_units(k)];
            GD_CUDA(cudaMemcpyAsync(a, d.heads.p + b0, nbk * sizeof(u64), cudaMemcpyDeviceToHost, c.stream));
            GD_CUDA(cudaMemcpyAsync(a + a_heads, d.cls.p + b0, nbk, cudaMemcpyDeviceToHost, c.stream));
            if (p1 > p0)
                GD_CUDA(cudaMemcpyAsync(a + a_heads + a_cls, d.payload.p + p0, p1 - p0, cudaMemcpyDeviceToHost,
                                        c.stream));
            GD_CUDA(cudaEventRecord(ev[k], c.stream));
            d2h_total.fetch_add(nbk * sizeof(u64) + nbk + (p1 - p0), std::memory_order_relaxed);
            issued[k].store(1, std::memory_order_release);
        };
        const u32 bits = E.enc.e.bits;
        std::atomic<u64> wait_ns{0}, work_ns{0};
        auto worker = [&] {
            try {
                while (!quit.load(std::memory_order_acquire)) {
                    const u64 u = next.fetch_add(1, std::memory_order_acq_rel);
                    if (u >= nunits) return;
                    const u64 k = u / kChunkUnits;
                    const double tw = Ctx::now_s();
                    while (!issued[k].load(std::memory_order_acquire)) {
                        if (quit.load(std::memory_order_acquire)) return;
                        std::this_thread::yield();
                    }
                    GD_CUDA(cudaEventSynchronize(ev[k]));
                    const double tu = Ctx::now_s();
                    const uint8_t* a = stage + (k % R) * area;
                    const u64 b0 = u * kUnitB, nbu = std::min(kUnitB, d.nb - b0), cb = b0 - k * kChunkB;
                    byte_decode_rows(reinterpret_cast<const u64*>(a) + cb, a + a_heads + cb,
                                     a + a_heads + a_cls + (uoff[u] - uoff[k * kChunkUnits]), b0 * kByteBlock, nbu,
                                     n, ar, bits, out);
                    const double te = Ctx::now_s();
                    wait_ns.fetch_add((u64)((tu - tw) * 1e9), std::memory_order_relaxed);
                    work_ns.fetch_add((u64)((te - tu) * 1e9), std::memory_order_relaxed);
                    if (finished[k].fetch_add(1, std::memory_order_acq_rel) + 1 == chunk_units(k) && k + R < nchunks)
                        issue(k + R);  // area k % R is free again
                }
            } catch (...) {
                std::lock_guard<std::mutex> g(err_mu);
                if (!err) err = std::current_exception();
                quit.store(true, std::memory_order_release);
            }
        };
        for (u64 k = 0; k < R; ++k) issue(k);
        for (unsigned t = 1; t < nt; ++t) pool.emplace_back(worker);
        worker();
        for (auto& th : pool) th.join();
        pool.clear();
        if (err) std::rethrow_exception(err);
        c.d2h_bytes += d2h_total.load() + (nunits + 1) * sizeof(u64);
        t_wait += wait_ns.load() * 1e-9 / nt;
        t_unpack += work_ns.load() * 1e-9 / nt;
    }

    // The same download with the packing overlapped (download_overlap_pack):
    // each 4 M-row chunk is packed on its own (byte_pack_into: chunk-relative
    // offsets, payload at 8 B per row of the chunk's first row) with an event
    // behind it, every chunk's unit offsets are requested up front on a side
    // stream behind its pack, and the copies run on a second side stream, so
    // the host rebuild of chunk 0 starts while the device packs the rest and
    // no thread is set aside for issuing.
    void download_bytes_rows_overlap(const u64* keys, u64 n, u32 ar, u64* out, unsigned nt, double& t_wait,
                                     double& t_unpack) {
        constexpr u64 kUnitB = 8192;      // blocks per unit (256 K rows)
        constexpr u64 kChunkUnits = 16;   // units per chunk (4 M rows)
        constexpr u64 kChunkB = kUnitB * kChunkUnits;
        const u64 nb = (n + kByteBlock - 1) / kByteBlock;
        const u64 nunits = (nb + kUnitB - 1) / kUnitB;
        const u64 nchunks = (nunits + kChunkUnits - 1) / kChunkUnits;
        auto chunk_units = [&](u64 k) { return std::min(kChunkUnits, nunits - k * kChunkUnits); };
        DevBuf<u64> heads(c, std::max<u64>(nb, 1)), offs(c, nb + nchunks), uoffs(c, nchunks * (kChunkUnits + 1));
        DevBuf<uint8_t> cls(c, std::max<u64>(nb, 1));
        DevBuf<u64> payload(c, std::max<u64>(n, 1));  // chunk k's bytes at 8 * (its first row)
        auto up = [](u64 v) { return (v + 63) & ~63ull; };
        const u64 a_heads = kChunkB * sizeof(u64), a_cls = up(kChunkB);
        const u64 area = a_heads + a_cls + up(kChunkB * kByteBlock * sizeof(u64) + 64);
        const u64 R = std::min<u64>(nchunks, 6);
        uint8_t* stage = static_cast<uint8_t*>(c.pinned_staging(R * area + nchunks * (kChunkUnits + 1) * sizeof(u64)));
        u64* uo = reinterpret_cast<u64*>(stage + R * area);  // chunk k: kChunkUnits + 1 unit offsets
        std::vector<cudaEvent_t> evp(nchunks, nullptr), evm(nchunks, nullptr), ev(nchunks, nullptr);
        cudaStream_t s2 = nullptr, sm = nullptr;
        std::unique_ptr<std::atomic<int>[]> issued(new std::atomic<int>[nchunks]);
        std::unique_ptr<std::atomic<u64>[]> finished(new std::atomic<u64>[nchunks]);
        for (u64 k = 0; k < nchunks; ++k) {
            issued[k].store(0);
            finished[k].store(0);
        }
        std::atomic<u64> next{0};
        std::atomic<bool> quit{false};
        std::atomic<u64> d2h_total{0};
        std::exception_ptr err;
        std::mutex err_mu;
        std::mutex issue_mu;  // issue() may run on two threads at once
        std::vector<std::thread> pool;
        struct Cleanup {
            std::function<void()> f;
            ~Cleanup() { f(); }
        } cleanup{[&] {
            quit.store(true, std::memory_order_release);
            for (auto& th : pool)
                if (th.joinable()) th.join();
            for (cudaStream_t st : {s2, sm})
                if (st) {
                    cudaStreamSynchronize(st);
                    cudaStreamDestroy(st);
                }
            cudaStreamSynchronize(c.stream);
            for (auto* v : {&evp, &evm, &ev})
                for (auto e : *v)
                    if (e) cudaEventDestroy(e);
            cudaGetLastError();
        }};
        GD_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        GD_CUDA(cudaStreamCreateWithFlags(&sm, cudaStreamNonBlocking));
        for (u64 k = 0; k < nchunks; ++k) {
            GD_CUDA(cudaEventCreateWithFlags(&evp[k], cudaEventDisableTiming));
            GD_CUDA(cudaEventCreateWithFlags(&evm[k], cudaEventDisableTiming));
            GD_CUDA(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
        }
        uint8_t* pay = reinterpret_cast<uint8_t*>(payload.p);
        for (u64 k = 0; k < nchunks; ++k) {
            const u64 r0 = k * kChunkB * kByteBlock, cnt = std::min(kChunkB * kByteBlock, n - r0);
            byte_pack_into(c, keys + r0, cnt, heads.p + k * kChunkB, cls.p + k * kChunkB, offs.p + k * kChunkB + k,
                           pay + r0 * sizeof(u64), kUnitB, uoffs.p + k * (kChunkUnits + 1));
            GD_CUDA(cudaEventRecord(evp[k], c.stream));
            GD_CUDA(cudaStreamWaitEvent(sm, evp[k], 0));
            GD_CUDA(cudaMemcpyAsync(uo + k * (kChunkUnits + 1), uoffs.p + k * (kChunkUnits + 1),
                                    (chunk_units(k) + 1) * sizeof(u64), cudaMemcpyDeviceToHost, sm));
            GD_CUDA(cudaEventRecord(evm[k], sm));
        }
        auto issue = [&](u64 k) {  // chunk k into area k % R, once its offsets are on the host
            std::lock_guard<std::mutex> g(issue_mu);
            GD_CUDA(cudaEventSynchronize(evm[k]));
            uint8_t* a = stage + (k % R) * area;
            const u64 b0 = k * kChunkB, nbk = std::min(kChunkB, nb - b0);
            const u64* ku = uo + k * (kChunkUnits + 1);
            const u64 p0 = ku[0], p1 = ku[chunk_units(k)];
            GD_CUDA(cudaMemcpyAsync(a, heads.p + b0, nbk * sizeof(u64), cudaMemcpyDeviceToHost, s2));
            GD_CUDA(cudaMemcpyAsync(a + a_heads, cls.p + b0, nbk, cudaMemcpyDeviceToHost, s2));
            if (p1 > p0)
                GD_CUDA(cudaMemcpyAsync(a + a_heads + a_cls, pay + b0 * kByteBlock * sizeof(u64) + p0, p1 - p0,
                                        cudaMemcpyDeviceToHost, s2));
            GD_CUDA(cudaEventRecord(ev[k], s2));
            d2h_total.fetch_add(nbk * sizeof(u64) + nbk + (p1 - p0) + (chunk_units(k) + 1) * sizeof(u64),
                                std::memory_order_relaxed);
            issued[k].store(1, std::memory_order_release);
        };
        const u32 bits = E.enc.e.bits;
        std::atomic<u64> wait_ns{0}, work_ns{0};
        auto worker = [&] {
            try {
                while (!quit.load(std::memory_order_acquire)) {
                    const u64 u = next.fetch_add(1, std::memory_order_acq_rel);
                    if (u >= nunits) return;
                    const u64 k = u / kChunkUnits, j = u - k * kChunkUnits;
                    const double tw = Ctx::now_s();
                    while (!issued[k].load(std::memory_order_acquire)) {
                        if (quit.load(std::memory_order_acquire)) return;
                        std::this_thread::yield();
                    }
                    GD_CUDA(cudaEventSynchronize(ev[k]));
                    const double tu = Ctx::now_s();
                    const uint8_t* a = stage + (k % R) * area;
                    const u64* ku = uo + k * (kChunkUnits + 1);
                    const u64 b0 = u * kUnitB, nbu = std::min(kUnitB, nb - b0), cb = b0 - k * kChunkB;
                    byte_decode_rows(reinterpret_cast<const u64*>(a) + cb, a + a_heads + cb,
                                     a + a_heads + a_cls + (ku[j] - ku[0]), b0 * kByteBlock, nbu, n, ar, bits, out);
                    const double te = Ctx::now_s();
                    wait_ns.fetch_add((u64)((tu - tw) * 1e9), std::memory_order_relaxed);
                    work_ns.fetch_add((u64)((te - tu) * 1e9), std::memory_order_relaxed);
                    if (finished[k].fetch_add(1, std::memory_order_acq_rel) + 1 == chunk_units(k) && k + R < nchunks)
                        issue(k + R);  // area k % R is free again
                }
            } catch (...) {
                std::lock_guard<std::mutex> g(err_mu);
                if (!err) err = std::current_exception();
                quit.store(true, std::memory_order_release);
            }
        };
        for (unsigned t = 1; t < nt; ++t) pool.emplace_back(worker);
        for (u64 k = 0; k < R; ++k) issue(k);  // each as soon as its chunk is packed
        worker();
        for (auto& th : pool) th.join();
        pool.clear();
        if (err) std::rethrow_exception(err);
        c.d2h_bytes += d2h_total.load();
        t_wait += wait_ns.load() * 1e-9 / nt;
        t_unpack += work_ns.load() * 1e-9 / nt;
    }

    // Delta-compressed download of n canonical keys into rows (download_delta = 1):
    // the device bit-packs the gaps of every 64-key block (delta.cu), chunks
    // of 16 K blocks cross PCIe into two pinned staging areas (heads, widths,
    // payload), and nt host threads rebuild the keys — a running sum per
    // block — and unpack them into the caller's rows while the next chunk is
    // in flight.  C2: ~3 bytes per row over PCIe instead of 8.
    void download_delta_rows(const u64* keys, u64 n, u32 ar, u64* out, unsigned nt, double& t_wait,
                             double& t_unpack) {
        DeltaPacked d;
        delta_pack(c, keys, n, d);
        constexpr u64 kBPC = 16384;  // blocks per chunk (1 M keys)
        const u64 nchunks = (d.nb + kBPC - 1) / kBPC;
        std::vector<u64> coff(nchunks + 1);
        {
            DevBuf<u64> dco(c, nchunks + 1);
            delta_chunk_offsets(c, d, kBPC, nchunks, dco.p);
            c.d2h(coff.data(), dco.p, (nchunks + 1) * sizeof(u64));
            c.sync();
        }
        u64 maxw = 0;
        for (u64 k = 0; k < nchunks; ++k) maxw = std::max(maxw, coff[k + 1] - coff[k]);
        // staging area per buffer: heads | widths (padded to words) | payload
        const u64 area = kBPC + kBPC / 8 + maxw + 8;
        u64* stage0 = static_cast<u64*>(c.pinned_staging(2 * area * sizeof(u64)));
        u64* stage[2] = {stage0, stage0 + area};
        cudaEvent_t ev[2] = {nullptr, nullptr};
        std::vector<std::thread> pool;
        std::atomic<bool> quit{false};
        struct Cleanup {
            std::function<void()> f;
            ~Cleanup() { f(); }
        } cleanup{[&] {
            quit.store(true, std::memory_order_release);
            for (auto& th : pool)
                if (th.joinable()) th.join();
            cudaStreamSynchronize(c.stream);
            for (auto e : ev)
                if (e) cudaEventDestroy(e);
        }};
        GD_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
        GD_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
        auto issue = [&](u64 k) {
            const u64 b0 = k * kBPC, nbk = std::min(kBPC, d.nb - b0);
            u64* st = stage[k & 1];
            c.d2h(st, d.heads.p + b0, nbk * sizeof(u64));
            c.d2h(st + kBPC, d.widths.p + b0, nbk);
            if (coff[k + 1] > coff[k])
                c.d2h(st + kBPC + kBPC / 8, d.payload.p + coff[k], (coff[k + 1] - coff[k]) * sizeof(u64));
            GD_CUDA(cudaEventRecord(ev[k & 1], c.stream));
        };
        const u32 bits = E.enc.e.bits;
        const u64 cmask = bits >= 64 ? ~0ull : (1ull << bits) - 1;
        const bool aligned16 = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
        (void)aligned16;
        std::atomic<u64> gen{0};
        std::atomic<unsigned> left{0};
        u64 cur_k = 0;
        auto decode = [&](unsigned t) {
            const u64 k = cur_k, b0 = k * kBPC, nbk = std::min(kBPC, d.nb - b0);
            const u64 lo = nbk * t / nt, hi = nbk * (t + 1) / nt;
            const u64* st = stage[k & 1];
            const u64* heads = st;
            const uint8_t* widths = reinterpret_cast<const uint8_t*>(st + kBPC);
            const u64* pay = st + kBPC + kBPC / 8;
            u64 wo = 0;  // payload word offset of block lo within the chunk
            for (u64 b = 0; b < lo; ++b) {
                const u64 cnt = std::min<u64>(kDeltaBlock, n - (b0 + b) * kDeltaBlock);
                wo += ((cnt - 1) * widths[b] + 63) / 64;
            }
            for (u64 b = lo; b < hi; ++b) {
                const u64 first = (b0 + b) * kDeltaBlock;
                const u64 cnt = std::min<u64>(kDeltaBlock, n - first);
                const u32 w = widths[b];
                const u64 wm = w >= 64 ? ~0ull : (1ull << w) - 1;
                const u64* p = pay + wo;
                u64 key = heads[b];
                u64* dst = out + first * ar;
                for (u64 i = 0;; ++i) {
                    if (ar == 2) {
#if defined(__x86_64__)
                        if (aligned16) {  // one 16-byte non-temporal store per row
                            _mm_stream_si128(reinterpret_cast<__m128i*>(dst),
                                             _mm_set_epi64x((long long)(key & cmask), (long long)((key >> bits) & cmask)));
                        } else {
                            _mm_stream_si64(reinterpret_cast<long long*>(dst), (long long)((key >> bits) & cmask));
                            _mm_stream_si64(reinterpret_cast<long long*>(dst + 1), (long long)(key & cmask));
                        }
#else
                        dst[0] = (key >> bits) & cmask;
                        dst[1] = key & cmask;
#endif
                    } else {
                        for (u32 col = 0; col < ar; ++col) dst[col] = (key >> ((ar - 1 - col) * bits)) & cmask;
                    }
                    dst += ar;
                    if (i + 1 >= cnt) break;
                    const u64 pos = i * w;
                    const u32 q = (u32)(pos >> 6), sh = (u32)(pos & 63);
                    u64 v = p[q] >> sh;
                    if (sh && sh + w > 64) v |= p[q + 1] << (64 - sh);
                    key += v & wm;
                }
                wo += ((cnt - 1) * w + 63) / 64;
            }
#if defined(__x86_64__)
            _mm_sfence();
#endif
        };
        for (unsigned t = 1; t < nt; ++t)
            pool.emplace_back([&, t] {
                u64 seen = 0;
                while (true) {
                    u64 g;
                    while ((g = gen.load(std::memory_order_acquire)) == seen && !quit.load(std::memory_order_acquire))
                        std::this_thread::yield();
                    if (quit.load(std::memory_order_acquire)) return;
                    seen = g;
                    decode(t);
                    left.fetch_sub(1, std::memory_order_acq_rel);
                }
            });
        issue(0);
        for (u64 k = 0; k < nchunks; ++k) {
            const double tw = Ctx::now_s();
            GD_CUDA(cudaEventSynchronize(ev[k & 1]));
            t_wait += Ctx::now_s() - tw;
            const double tu = Ctx::now_s();
            if (k + 1 < nchunks) issue(k + 1);  // stage[(k+1)&1] was decoded at step k-1
            cur_k = k;
            left.store(nt - 1, std::memory_order_release);
            gen.fetch_add(1, std::memory_order_acq_rel);
            decode(0);
            while (left.load(std::memory_order_acquire) != 0) std::this_thread::yield();
            t_unpack += Ctx::now_s() - tu;
        }
    }

    u64 digest(u32 r) override {
        if (pl) part_loop_finish();
        compact(rels[r]);
        return digest_rows<K>(c, rels[r].full.p, rels[r].full_n, E.info_[r].arity, E.enc.e);
    }

    // ---- tiered full relation ---------------------------------------------
    static u64 total_n(const RelDev<K>& st) {
        u64 t = st.full_n;
        for (const auto& r : st.tail) t += r.n;
        return t;
    }

    // Merges the tail runs (smallest first) and then into the base run.
    void compact(RelDev<K>& st) {
        while (st.tail.size() > 1) {
            Run<K> b = std::move(st.tail.back());
            st.tail.pop_back();
            Run<K>& a = st.tail.back();
            Run<K> m;
            m.buf = DevBuf<K>(c, a.n + b.n);
            merge_disjoint<K>(c, a.buf.p, a.n, b.buf.p, b.n, m.buf.p);
            m.n = a.n + b.n;
            a = std::move(m);
        }
        if (!st.tail.empty()) {
            Run<K> b = std::move(st.tail.back());
            st.tail.pop_back();
            ensure_discard(c, st.full_alt, st.full_n + b.n);
            merge_disjoint<K>(c, st.full.p, st.full_n, b.buf.p, b.n, st.full_alt.p);
            st.full.swap(st.full_alt);
            st.full_n += b.n;
        }
    }

    // D = unique(N) \ full (N sorted, duplicates allowed).
    MergeResult difference_full(RelDev<K>& st, const K* N, u64 nn, K* Dout) {
        if (!st.tail.empty() && nn * 24 >= total_n(st)) compact(st);
        if (st.tail.empty()) return difference_sorted<K>(c, st.full.p, st.full_n, N, nn, Dout);
        std::vector<const K*> ptr{st.full.p};
        std::vector<u64> ns{st.full_n};
        for (const auto& r : st.tail) {
            ptr.push_back(r.buf.p);
            ns.push_back(r.n);
        }
        return difference_runs<K>(c, ptr.data(), ns.data(), (u32)ptr.size(), N, nn, Dout);
    }

    // full <- full U D (D disjoint from full, canonical).
    void add_to_full(RelDev<K>& st, const K* D, u64 nd) {
        if (nd == 0) return;
        if (!st.lsm) {
            ensure_discard(c, st.full_alt, st.full_n + nd);
            merge_disjoint<K>(c, st.full.p, st.full_n, D, nd, st.full_alt.p);
            st.full.swap(st.full_alt);
            st.full_n += nd;
            return;
        }
        Run<K> run;
        run.buf = DevBuf<K>(c, nd);
        c.d2d(run.buf.p, D, nd * sizeof(K));
        run.n = nd;
        st.tail.push_back(std::move(run));
        // restore the tier invariant (each run >= kTierRatio x the next one)
        while (!st.tail.empty()) {
            const size_t k = st.tail.size();
            const u64 prev = k >= 2 ? st.tail[k - 2].n : st.full_n;
            if (prev >= kTierRatio * st.tail[k - 1].n) break;
            Run<K> b = std::move(st.tail.back());
            st.tail.pop_back();
            if (k >= 2) {
                Run<K>& a = st.tail.back();
                Run<K> m;
                m.buf = DevBuf<K>(c, a.n + b.n);
                merge_disjoint<K>(c, a.buf.p, a.n, b.buf.p, b.n, m.buf.p);
                m.n = a.n + b.n;
                a = std::move(m);
            } else {
                ensure_discard(c, st.full_alt, st.full_n + b.n);
                merge_disjoint<K>(c, st.full.p, st.full_n, b.buf.p, b.n, st.full_alt.p);
                st.full.swap(st.full_alt);
                st.full_n += b.n;
            }
        }
    }

    // ---- resident device loop (loop.h) ---------------------
    // Eligible when every recursive head is never a join inner (so its full
    // version is only probed for membership and read back at the end), keys
    // are u64, one rank, and Δ = full (the state seed() leaves).  A finite
    // memory budget is enforced by the bookkeeping replay after the device
    // loop: the accountant sees the reference's charges in the reference's
    // order, so a budget_error surfaces at the same charge with the same
    // phase (the device work past that point is discarded with the error).
    bool loop_eligible(const std::vector<u32>& rec) {
        if (E.nranks > 1) return false;
        if (!c.cfg.resident_loop) return false;
        if (rec.empty() || rec.size() > kLoopMaxHeads) return false;
        u32 nsteps = 0;
        for (u32 r : rec) {
            const auto& st = rels[r];
            if (!st.lsm || st.delta_n != total_n(st)) return false;
        }
        auto is_head = [&](u32 r) { return std::find(rec.begin(), rec.end(), r) != rec.end(); };
        for (const auto& p : E.plans_) {
            if (!p.recursive) continue;
            for (u32 v = 0; v < p.nvariants; ++v) {
                const gd_variant& var = p.variants[v];
                if (var.src_version == GD_DELTA && !is_head(var.src_rel)) return false;
                nsteps += std::max<u32>(1, var.nsteps);
                for (u32 s = 0; s < var.nsteps; ++s)
                    if (is_head(var.steps[s].inner_rel)) return false;
            }
        }
        return nsteps <= kLoopMaxSteps;
    }

    struct LStep {
        u32 plan = 0, var = 0;
        bool final = false, select = false;
        // GD_LOOP_SPLIT=1: materialize the final step's rows, then insert
        // them (comparison mode; the fused kernel moves fewer bytes)
        bool split_insert = false;
        // final step over a dense inner: loop_count + loop_expand_insert
        // (gd_device_config.warp_expand)
        bool xp = false;
        u32 head = 0;            // loop-head index (final steps)
        u32 kind = LO_STATIC;    // outer source
        u32 src_head = 0, src_step = 0;
        const u64* static_ptr = nullptr;
        u64 static_n = 0;
        DevJoin jd{};
        bool has_iv = false;
        IndexView<u64> iv{};
        DevBuf<u32> dense;  // dense (CSR) form of the inner's index, if built
        LoopDense dv{nullptr, 0, 0};
        const u64* inner = nullptr;
        u64 inner_n = 0;
        u32 proj_arity = 0;
        DevBuf<u64> row_start, row_off, splits, temp;
        u64 rows_cap = 0, splits_cap = 0, temp_cap = 0;
        DevBuf<u64> rc;  // xp steps: each outer row's inner range (start << 32 | count), from loop_count
        // precounted step (gd_device_config.precount): second set of the
        // per-row buffers, written by the insert for the next iteration
        bool pre = false;
        DevBuf<u64> rc2, row_start2, row_off2;
        LoopStepBufs bufs() const {
            return LoopStepBufs{row_start.p, row_off.p, rows_cap, splits.p, splits_cap, xp ? rc.p : nullptr,
                                pre ? rc2.p : nullptr, pre ? row_start2.p : nullptr, pre ? row_off2.p : nullptr};
        }
        void alloc_rows(Ctx& c) {
            row_start = DevBuf<u64>(c, rows_cap);
            row_off = DevBuf<u64>(c, rows_cap);
            if (xp) rc = DevBuf<u64>(c, rows_cap);
            if (pre) {
                rc2 = DevBuf<u64>(c, rows_cap);
                row_start2 = DevBuf<u64>(c, rows_cap);
                row_off2 = DevBuf<u64>(c, rows_cap);
            }
        }
    };
    struct LHead {
        u32 rel = 0;
        DevBuf<u64> log;
        DevBuf<u64> tab;  // tab_cap slots of loop_slot_bytes(sbits)
        u64 log_cap = 0, tab_cap = 0, tab_limit = 0;
        u32 sbits = 0;
        // clear = false: the caller writes every slot (loop_table_rehash)
        void alloc_tab(Ctx& c, u64 cap, bool dense = false, bool clear = true) {
            tab.release();
            tab_cap = cap;
            tab_limit = dense ? cap / 4 * 3 : tab_limit_of(c, cap);
            tab = DevBuf<u64>(c, cap * loop_slot_bytes(sbits) / 8);
            if (clear) loop_table_clear(c, tab.p, cap, sbits);
        }
    };
    // Linear probing stays short (~1.5 slot reads per new key with the
    // sector scan) at load <= 1/2; a full table grows 4x (to load 1/8), so
    // the re-spreads move about a third of the final key count in total.
    static u64 tab_limit_of(const Ctx& c, u64 cap) {
        const u64 pct = c.cfg.index_load_pct ? c.cfg.index_load_pct : 50;
        return cap / 100 * pct + cap % 100 * pct / 100;
    }

    // The recursive variants as loop steps (plan order, variant order): outer
    // source, join descriptor, inner copy and index (dense form when
    // worthwhile) of every step.  Shared by iterate_loop and partition mode.
    void build_loop_steps(const std::vector<u32>& rec, std::vector<LStep>& steps) {
        auto head_of = [&](u32 r) -> u32 {
            return (u32)(std::find(rec.begin(), rec.end(), r) - rec.begin());
        };
    for (u32 pi = 0; pi < E.plans_.size(); ++pi) {
        const gd_rule_plan& p = E.plans_[pi];
        if (!p.recursive) continue;
        for (u32 v = 0; v < p.nvariants; ++v) {
            const gd_variant& var = p.variants[v];
            const u32 ar = E.info_[var.src_rel].arity;
            u32 cur_ar = ar;
            u32 cur_perm[kMaxArity];
            for (u32 i = 0; i < kMaxArity; ++i) cur_perm[i] = i < ar ? var.src_perm[i] : i;
            const u32 first = (u32)steps.size();
            const u32 n = std::max<u32>(1, var.nsteps);
            for (u32 s = 0; s < n; ++s) {
                steps.emplace_back();
                LStep& L = steps.back();
                L.plan = pi;
                L.var = v;
                L.final = s + 1 == n;
                L.split_insert = c.cfg.split_insert != 0;
                L.head = head_of(p.head_rel);
                if (s == 0) {
                    auto it = std::find(rec.begin(), rec.end(), var.src_rel);
                    if (it != rec.end()) {
                        L.kind = var.src_version == GD_DELTA ? LO_DELTA : LO_FULL;
                        L.src_head = (u32)(it - rec.begin());
                    } else {
                        auto& src = rels[var.src_rel];
                        compact(src);
                        L.kind = LO_STATIC;
                        L.static_ptr = reinterpret_cast<const u64*>(src.full.p);
                        L.static_n = src.full_n;
                    }
                } else {
                    L.kind = LO_TEMP;
                    L.src_step = first + s - 1;
                }
                if (var.nsteps == 0) {
                    L.select = true;
                    L.jd = make_desc(0, cur_ar, cur_perm, 0, var.sel_arity, var.sel_proj, var.nsel_filters,
                                     var.sel_filters);
                    continue;
                }
                const gd_join_step& st = var.steps[s];
                auto& in = rels[st.inner_rel];
                const u32 iar = E.info_[st.inner_rel].arity;
                CopyState<K>& cp = in.copies.at(CopyKey{std::vector<u32>(st.inner_perm, st.inner_perm + iar),
                                                        st.join_column_count});
                L.inner = reinterpret_cast<const u64*>(cp.identity ? in.full.p : cp.rows.p);
                L.inner_n = cp.identity ? in.full_n : cp.n;
                L.jd = make_desc(st.join_column_count, cur_ar, cur_perm, iar, st.proj_arity, st.proj,
                                 st.nfilters, st.filters);
                L.proj_arity = st.proj_arity;
                if (st.join_column_count > 0 && L.inner_n > 0) {
                    L.has_iv = true;
                    L.iv = IndexView<u64>{cp.index.slots.p, cp.index.slot_count, L.inner, L.inner_n, iar, bits,
                                          st.join_column_count};
                    if (st.join_column_count == 1 && c.cfg.dense_inner &&
                        loop_dense_build(c, L.inner, L.inner_n, iar, bits, L.dense, L.dv.lo, L.dv.span))
                        L.dv.off = L.dense.p;
                }
                // split_insert + xp: warp expansion into the temp, then the insert kernel
                L.xp = L.final && L.dv.off && c.cfg.warp_expand;
                cur_ar = st.proj_arity;
                for (u32 i = 0; i < kMaxArity; ++i) cur_perm[i] = i;
            }
        }
    }
    }

    void iterate_loop(const std::vector<u32>& rec, const std::vector<u32>& by_name) {
        bool active = false;
        for (u32 r : rec) active |= rels[r].delta_n > 0;
        if (!active) return;
        loop_prepare();
        // iteration 1, step (1): refresh the (static) indexed copies
        for (u32 r : by_name)
            if (rels[r].dirty) refresh_copies(r);

        // min_capacities starts every capacity at its minimum so tests walk
        // the overflow -> rollback -> grow -> re-run path on small inputs.
        const bool tiny = c.cfg.min_capacities != 0;
        const u32 nh = (u32)rec.size();
        std::vector<LHead> heads(nh);
        auto head_of = [&](u32 r) -> u32 {
            return (u32)(std::find(rec.begin(), rec.end(), r) - rec.begin());
        };
        for (u32 h = 0; h < nh; ++h) {
            auto& st = rels[rec[h]];
            compact(st);
            heads[h].rel = rec[h];
            const u64 f0 = st.full_n;
            heads[h].log_cap = tiny ? std::max<u64>(f0, 1) : std::max<u64>(2 * f0, 1 << 16);
            heads[h].log = DevBuf<u64>(c, heads[h].log_cap);
            if (f0) loop_copy_u64(c, heads[h].log.p, reinterpret_cast<const u64*>(st.full.p), f0);
            heads[h].sbits = loop_stamp_bits(E.info_[rec[h]].arity * bits);
            heads[h].alloc_tab(c, tiny ? 2 * f0 + 16 : std::max<u64>(4 * f0, 1 << 16));
            loop_table_fill(c, heads[h].tab.p, heads[h].tab_cap, heads[h].sbits, heads[h].log.p, f0);
        }

        // variant-steps in execution order (plan order, variant order)
        std::vector<LStep> steps;
        build_loop_steps(rec, steps);
        // Precount: a single self-recursive warp-expanded step (TC) lets its
        // insert compute the next iteration's row ranges (loop.cu InsertSink).
        if (steps.size() == 1 && steps[0].xp && steps[0].final && !steps[0].split_insert &&
            steps[0].kind == LO_DELTA && steps[0].src_head == steps[0].head && c.cfg.precount)
            steps[0].pre = true;
        const u32 ns = (u32)steps.size();
        const u64 d0 = rels[rec[0]].delta_n;
        for (auto& L : steps) {
            L.rows_cap = tiny ? 2 : std::max<u64>(d0 + 1, 1 << 12);
            L.splits_cap = tiny ? 2 : std::max<u64>(2 * d0 / kLoopMatTile + 2, 1 << 12);
            if (!L.select) {
                L.alloc_rows(c);
                L.splits = DevBuf<u64>(c, L.splits_cap);
            }
            if (!L.final || (L.split_insert && !L.select)) {  // chain temps / split-insert input
                L.temp_cap = tiny ? 1 : std::max<u64>(4 * d0, 1 << 16);
                L.temp = DevBuf<u64>(c, L.temp_cap);
            }
        }
        DevBuf<u64> block_sums(c, (u64)loop_grid(c));
        u64 hist_cap = tiny ? 1 : 1024;
        DevBuf<gd_iter_record> hist_rec(c, hist_cap * nh);
        DevBuf<u64> hist_steps(c, hist_cap * ns);

        // control block
        DevBuf<LoopCtl> ctl(c, 1);
        LoopCtl* hc = static_cast<LoopCtl*>(c.pinned_area());
        std::memset(hc, 0, sizeof(LoopCtl));
        hc->nheads = nh;
        hc->hist_cap = hist_cap;
        for (u32 h = 0; h < nh; ++h) {
            const auto& st = rels[rec[h]];
            hc->h[h].log_n = st.full_n;
            hc->h[h].dlo = st.full_n - st.delta_n;
            hc->h[h].dhi = st.full_n;
        }
        c.h2d(ctl.p, hc, sizeof(LoopCtl));

        // Count ahead (gd_device_config.count_ahead): a single self-recursive
        // warp-expanded step whose inner groups are all light (no heavy
        // segments possible) drops loop_count from the iteration: the insert
        // sums the next iteration's candidates as it appends the rows, loop_end
        // makes that the next gate's total, the insert evaluates the gate, and
        // the rows' ranges are read inline.  loop_count runs eagerly only
        // before the first graph launch and after a rollback.
        const bool loop_eager = c.prof.on || c.cfg.loop_mode == GD_LOOP_EAGER;
        const bool count_ahead = c.cfg.count_ahead && c.cfg.gate_in_insert && !loop_eager &&
                                 c.cfg.loop_mode != GD_LOOP_BATCH && ns == 1 && steps[0].xp && steps[0].final &&
                                 !steps[0].split_insert && !steps[0].pre && steps[0].kind == LO_DELTA &&
                                 steps[0].src_head == steps[0].head &&
                                 loop_dense_max_group(c, steps[0].dv) <= c.cfg.heavy_rows;
        auto light_bufs = [&](const LStep& L) {  // no row ranges handed over: read inline
            LoopStepBufs b = L.bufs();
            b.rc = b.rc2 = nullptr;
            return b;
        };

        auto outer_of = [&](const LStep& L) {
            LoopOuter o{};
            o.kind = L.kind;
            o.head = L.src_head;
            o.src_step = L.src_step;
            if (L.kind == LO_STATIC) {
                o.ptr = L.static_ptr;
                o.n = L.static_n;
            } else if (L.kind == LO_TEMP) {
                o.ptr = steps[L.src_step].temp.p;
            } else {
                o.ptr = heads[L.src_head].log.p;
            }
            return o;
        };
        auto bufs_of = [&](u32 h) {
            return LoopHeadBufs{heads[h].log.p, heads[h].log_cap, heads[h].tab.p, heads[h].tab_cap,
                                heads[h].tab_limit, heads[h].sbits, c.cfg.warp_append};
        };
        // One iteration's kernel sequence (captured into the graph, or
        // launched eagerly when profiling).  The gate runs in the last CTA
        // of the last scan and loop_end in the last CTA of the last insert
        // when the sequence allows it.
        // (profiler record, kind, step): algorithmic bytes are patched in
        // after the iteration, once its sizes are known (eager mode only)
        struct ProfRec {
            long rec;
            int kind;  // 0 probe, 1 temp, 2 insert, 3 select insert, 4 count (warp expansion)
            u32 step;
        };
        std::vector<ProfRec> prof_recs;
        auto record_iteration = [&](cudaStream_t s, bool use_cond, unsigned long long cond) {
            auto br = [&]() { return c.prof_begin(); };
            LoopGateDesc g{};
            g.stamp_max = 0xfffffffeu;
            for (u32 i = 0; i < ns; ++i)
                if (steps[i].final) {
                    g.final_step[g.nfinal] = i;
                    g.final_head[g.nfinal] = steps[i].head;
                    ++g.nfinal;
                }
            for (u32 h = 0; h < nh; ++h) {
                g.log_cap[h] = heads[h].log_cap;
                g.tab_limit[h] = heads[h].tab_limit;
                if (heads[h].sbits) g.stamp_max = std::min<u32>(g.stamp_max, (1u << heads[h].sbits) - 1);
            }
            const bool fuse_gate = !steps[ns - 1].select;
            // a single warp-expanded step (TC): its insert kernel evaluates the gate
            // in every CTA, so loop_count needs no last-CTA epilogue
            const bool gate_ins = c.cfg.gate_in_insert && ns == 1 && steps[0].xp && !steps[0].split_insert &&
                                  steps[0].final && !steps[0].pre && fuse_gate;
            for (u32 i = 0; i < ns; ++i) {
                LStep& L = steps[i];
                const LoopOuter o = outer_of(L);
                if (L.select) {
                    cudaEvent_t t = br();
                    loop_select_cand(c, s, ctl.p, i, o);
                    c.prof_end(t, KC_LOOP_CTL, 0);
                    continue;
                }
                cudaEvent_t t = br();
                if (L.xp) {
                    if (count_ahead) continue;  // the last insert counted this iteration's rows
                    loop_count(c, s, ctl.p, i, o, L.jd, L.dv, L.bufs(), c.cfg.heavy_rows,
                               fuse_gate && !gate_ins && i + 1 == ns ? &g : nullptr);
                    prof_recs.push_back({c.prof_end(t, KC_PROBE, 0), 4, i});
                    continue;
                }
                loop_probe(c, s, ctl.p, i, o, L.jd, L.has_iv ? &L.iv : nullptr, L.dv, L.inner_n, L.bufs(),
                           block_sums.p);
                prof_recs.push_back({c.prof_end(t, KC_PROBE, 0), 0, i});
                t = br();
                loop_scan(c, s, ctl.p, i, o, L.bufs(), block_sums.p, fuse_gate && i + 1 == ns ? &g : nullptr);
                c.prof_end(t, KC_SELECT, 0);
                if (!L.final || L.split_insert) {
                    t = br();
                    loop_materialize_temp(c, s, ctl.p, i, o, L.inner, L.jd, L.bufs(), L.temp.p, L.temp_cap);
                    prof_recs.push_back({c.prof_end(t, KC_MATERIALIZE, 0), 1, i});
                }
            }
            if (!fuse_gate) {
                cudaEvent_t t = br();
                loop_gate(c, s, ctl.p, g);
                c.prof_end(t, KC_LOOP_CTL, 0);
            }
            const LoopEndDesc end{LoopHist{hist_rec.p, hist_steps.p, ns}, cond, use_cond ? 1 : 0,
                                  ns == 1 && (steps[0].pre || count_ahead) ? 0u : ~0u};
            u32 last_final = 0;
            for (u32 i = 0; i < ns; ++i)
                if (steps[i].final) last_final = i;
            for (u32 i = 0; i < ns; ++i) {
                LStep& L = steps[i];
                if (!L.final) continue;
                const LoopOuter o = outer_of(L);
                const LoopEndDesc* e = i == last_final ? &end : nullptr;
                cudaEvent_t t = br();
                if (L.select)
                    loop_select_insert(c, s, ctl.p, i, L.head, o, L.jd, bufs_of(L.head), e);
                else if (L.xp && L.split_insert) {
                    loop_expand_temp(c, s, ctl.p, i, o, L.inner, L.jd, L.dv, L.bufs(), c.cfg.heavy_rows, L.temp.p,
                                     L.temp_cap);
                    loop_insert_keys(c, s, ctl.p, i, L.head, L.temp.p, bufs_of(L.head), e);
                } else if (L.xp && count_ahead)
                    loop_expand_insert(c, s, ctl.p, i, L.head, o, L.inner, L.jd, L.dv, light_bufs(L), ~0ull,
                                       bufs_of(L.head), e, &g, true);
                else if (L.xp)
                    loop_expand_insert(c, s, ctl.p, i, L.head, o, L.inner, L.jd, L.dv, L.bufs(), c.cfg.heavy_rows,
                                       bufs_of(L.head), e, gate_ins ? &g : nullptr);
                else if (L.split_insert)
                    loop_insert_keys(c, s, ctl.p, i, L.head, L.temp.p, bufs_of(L.head), e);
                else
                    loop_materialize_insert(c, s, ctl.p, i, L.head, o, L.inner, L.jd, L.bufs(), bufs_of(L.head), e);
                prof_recs.push_back({c.prof_end(t, KC_INSERT, 0), L.select ? 3 : 2, i});
            }
        };

        // CUDA graph: while (some Δ non-empty) { iteration }
        // Modes: "graph" (default) one launch of a graph whose conditional
        // while node repeats the iteration until loop_end clears it;
        // "batch" a plain graph of one iteration launched GD_LOOP_BATCH
        // times per host check; "eager" direct launches, one check per
        // iteration (used when per-kernel profiling is on).
        const bool eager = c.prof.on || c.cfg.loop_mode == GD_LOOP_EAGER;
        const bool batch = !eager && c.cfg.loop_mode == GD_LOOP_BATCH;
        const int batch_n = (int)c.cfg.loop_batch;
        cudaGraphExec_t exec = nullptr;
        cudaGraph_t graph = nullptr;
        cudaStream_t cap_stream = nullptr;
        u64 kernels_per_iter = 0;
        auto destroy_graph = [&]() {
            if (exec) cudaGraphExecDestroy(exec);
            if (graph) cudaGraphDestroy(graph);
            exec = nullptr;
            graph = nullptr;
        };
        auto build_graph = [&]() {
            destroy_graph();
            if (!cap_stream) GD_CUDA(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
            if (batch) {
                GD_CUDA(cudaStreamBeginCapture(cap_stream, cudaStreamCaptureModeThreadLocal));
                const u64 l0 = c.launches;
                try {
                    record_iteration(cap_stream, false, 0);
                } catch (...) {
                    cudaStreamEndCapture(cap_stream, &graph);
                    throw;
                }
                kernels_per_iter = c.launches - l0;
                c.launches = l0;
                GD_CUDA(cudaStreamEndCapture(cap_stream, &graph));
                GD_CUDA(cudaGraphInstantiate(&exec, graph, 0));
                return;
            }
            GD_CUDA(cudaGraphCreate(&graph, 0));
            cudaGraphConditionalHandle hdl;
            GD_CUDA(cudaGraphConditionalHandleCreate(&hdl, graph, 1, cudaGraphCondAssignDefault));
            cudaGraphNodeParams np{};
            np.type = cudaGraphNodeTypeConditional;
            np.conditional.handle = hdl;
            np.conditional.type = cudaGraphCondTypeWhile;
            np.conditional.size = 1;
            cudaGraphNode_t node;
            GD_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &np));
            cudaGraph_t body = np.conditional.phGraph_out[0];
            GD_CUDA(cudaStreamBeginCaptureToGraph(cap_stream, body, nullptr, nullptr, 0,
                                                  cudaStreamCaptureModeThreadLocal));
            const u64 l0 = c.launches;
            try {
                record_iteration(cap_stream, true, (unsigned long long)hdl);
            } catch (...) {
                cudaStreamEndCapture(cap_stream, &body);
                throw;
            }
            kernels_per_iter = c.launches - l0;
            c.launches = l0;
            GD_CUDA(cudaStreamEndCapture(cap_stream, &body));
            GD_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        };

        // After an overflow: grows what the kernels asked for (step buffers,
        // head logs and indexes, history, stamp epoch); temps of chain steps
        // stop at the temp limit (those steps then run in windows).
        const u64 temp_limit = c.cfg.temp_limit_rows ? c.cfg.temp_limit_rows
                                                     : std::max<u64>(1 << 20, c.available_bytes() / 2 / sizeof(u64));
        double tlast = 0;
        const bool trace = (c.cfg.trace & 1) != 0;
        u64 windowed_iters = 0;
        auto grow_after_overflow = [&]() {
            for (u32 i = 0; i < ns; ++i)
                if (!steps[i].final && hc->need_temp[i] > temp_limit) hc->need_temp[i] = temp_limit;
            for (u32 i = 0; i < ns; ++i) {
                LStep& L = steps[i];
                if (hc->need_rows[i] > L.rows_cap) {
                    L.rows_cap = hc->need_rows[i] + hc->need_rows[i] / 2;
                    L.alloc_rows(c);
                }
                if (hc->need_splits[i] > L.splits_cap) {
                    L.splits_cap = hc->need_splits[i] + hc->need_splits[i] / 2;
                    L.splits = DevBuf<u64>(c, L.splits_cap);
                }
                if (hc->need_temp[i] > L.temp_cap) {
                    L.temp_cap = std::min<u64>(hc->need_temp[i] + hc->need_temp[i] / 2, L.final ? ~0ull : temp_limit);
                    L.temp = DevBuf<u64>(c, L.temp_cap);
                }
                hc->need_rows[i] = hc->need_splits[i] = hc->need_temp[i] = 0;
            }
            for (u32 h = 0; h < nh; ++h) {
                LHead& H = heads[h];
                const u64 ln = hc->h[h].log_n;
                cudaEvent_t ev0 = nullptr, ev1 = nullptr;
                auto tr = [&](const char* what, u64 a, u64 b2) {
                    if (!trace) return;
                    cudaEventRecord(ev1, c.stream);
                    c.sync();
                    const double t1 = Ctx::now_s();
                    float gms = 0;
                    cudaEventElapsedTime(&gms, ev0, ev1);
                    fprintf(stderr, "[loop] iter %u %s %llu -> %llu: %.3f ms (gpu %.3f ms)\n", hc->iter, what,
                            (unsigned long long)a, (unsigned long long)b2, (t1 - tlast) * 1e3, gms);
                    tlast = t1;
                    std::swap(ev0, ev1);
                    cudaEventRecord(ev0, c.stream);
                };
                if (trace) {
                    cudaEventCreate(&ev0);
                    cudaEventCreate(&ev1);
                    c.sync();
                    tlast = Ctx::now_s();
                    cudaEventRecord(ev0, c.stream);
                }
                // Growth is sized against free HBM (C5-scale runs): 2x
                // for the log and 4x for the index when they fit, else
                // the largest size that does (index load up to 3/4).
                const u64 reserve = 1ull << 30;
                if (hc->need_log[h] > H.log_cap) {
                    const u64 need = hc->need_log[h];
                    u64 avail = c.available_bytes();
                    const u64 lg = c.cfg.log_growth ? c.cfg.log_growth : 2;
                    if (lg * need * sizeof(u64) + reserve > avail / 2) avail = c.available_bytes(true);
                    const u64 fit = avail > reserve ? (avail - reserve) / sizeof(u64) : 0;
                    const u64 cap = std::max(need + need / 16 + 1024, std::min(lg * need, fit));
                    DevBuf<u64> nl(c, cap);
                    if (ln) loop_copy_u64(c, nl.p, H.log.p, ln);
                    H.log = std::move(nl);
                    tr("log", H.log_cap, cap);
                    H.log_cap = cap;
                }
                if (hc->need_tab[h] > H.tab_limit) {  // grow: stream the old table into the new
                    const u64 need = hc->need_tab[h];
                    const u64 sb = loop_slot_bytes(H.sbits);
                    const u64 spill = (ln / 16 + (1u << 20)) * sizeof(u64);  // re-spread spill list
                    u64 avail = c.available_bytes();
                    // load 1/8 after a growth (index_growth: 4 / 6 / 8 / 12
                    // measured on C1-C5, 8 best or within 1%)
                    const u64 gf = c.cfg.index_growth;
                    if (gf * need * sb + spill + reserve > avail / 2) avail = c.available_bytes(true);
                    const u64 fit = avail > reserve + spill ? (avail - reserve - spill) / sb : 0;
                    const u64 cap = std::min(gf * need, fit);  // load 1/gf after growth when it fits
                    if (cap < need / 3 * 4 + 16)
                        throw_budget("index", "device memory cannot hold the full-tuple index of " +
                                                  std::to_string(need) + " keys");
                    DevBuf<u64> old = std::move(H.tab);
                    const u64 old_cap = H.tab_cap;
                    H.alloc_tab(c, cap, cap < 2 * need, false);
                    tr("tab-alloc", old_cap, H.tab_cap);
                    loop_table_rehash(c, old.p, old_cap, H.tab.p, H.tab_cap, H.sbits, ln);
                    tr("tab-rehash", old_cap, H.tab_cap);
                } else if (hc->need_restamp) {
                    loop_table_restamp(c, H.tab.p, H.tab_cap, H.sbits);
                }
                hc->need_log[h] = hc->need_tab[h] = 0;
            }
            if (hc->need_hist > hist_cap) {
                const u64 cap = hc->need_hist;
                DevBuf<gd_iter_record> r2(c, cap * nh);
                DevBuf<u64> s2(c, cap * ns);
                c.d2d(r2.p, hist_rec.p, hist_cap * nh * sizeof(gd_iter_record));
                c.d2d(s2.p, hist_steps.p, hist_cap * ns * sizeof(u64));
                hist_rec = std::move(r2);
                hist_steps = std::move(s2);
                hist_cap = cap;
                hc->hist_cap = cap;
            }
            hc->need_hist = 0;
            if (hc->need_restamp) hc->epoch_base = hc->iter;
            hc->need_restamp = 0;
        };
        // One iteration with chain step `wi`'s temp materialized in windows of
        // at most temp_limit rows (engine.hpp:401-484 charges
        // the whole temp, and so does the replay: only device memory is
        // bounded).  Eager launches: first every step outside wi's variant and
        // that variant's steps up to wi's scan (their inserts gated as usual),
        // then per window wi's temp window, the rest of the variant, its gate
        // and insert; an overflow inside a window grows and redoes only that
        // window (nothing of it was inserted).  The iteration ends on the
        // device as in the graph (loop_end); step totals are the window sums.
        auto windowed_iteration = [&](u32 wi) {
            PhaseTimer tw(E, "join");
            const LStep& W0 = steps[wi];
            auto in_v = [&](u32 j) { return steps[j].plan == W0.plan && steps[j].var == W0.var; };
            auto cand = [&](u32 i, bool temp) {
                LStep& L = steps[i];
                const LoopOuter o = outer_of(L);
                if (L.select) {
                    loop_select_cand(c, c.stream, ctl.p, i, o);
                    return;
                }
                if (L.xp) {
                    loop_count(c, c.stream, ctl.p, i, o, L.jd, L.dv, L.bufs(), c.cfg.heavy_rows, nullptr);
                    return;
                }
                loop_probe(c, c.stream, ctl.p, i, o, L.jd, L.has_iv ? &L.iv : nullptr, L.dv, L.inner_n, L.bufs(),
                           block_sums.p);
                loop_scan(c, c.stream, ctl.p, i, o, L.bufs(), block_sums.p, nullptr);
                if (temp && (!L.final || L.split_insert))
                    loop_materialize_temp(c, c.stream, ctl.p, i, o, L.inner, L.jd, L.bufs(), L.temp.p, L.temp_cap);
            };
            auto gate_and_insert = [&](bool variant) {
                LoopGateDesc g{};
                g.stamp_max = 0xfffffffeu;
                for (u32 i = 0; i < ns; ++i)
                    if (steps[i].final && in_v(i) == variant) {
                        g.final_step[g.nfinal] = i;
                        g.final_head[g.nfinal] = steps[i].head;
                        ++g.nfinal;
                    }
                for (u32 h = 0; h < nh; ++h) {
                    g.log_cap[h] = heads[h].log_cap;
                    g.tab_limit[h] = heads[h].tab_limit;
                    if (heads[h].sbits) g.stamp_max = std::min<u32>(g.stamp_max, (1u << heads[h].sbits) - 1);
                }
                if (!g.nfinal) return;
                loop_gate(c, c.stream, ctl.p, g);
                for (u32 k = 0; k < g.nfinal; ++k) {
                    const u32 i = g.final_step[k];
                    LStep& L = steps[i];
                    const LoopOuter o = outer_of(L);
                    if (L.select)
                        loop_select_insert(c, c.stream, ctl.p, i, L.head, o, L.jd, bufs_of(L.head), nullptr);
                    else if (L.xp && L.split_insert) {
                        loop_expand_temp(c, c.stream, ctl.p, i, o, L.inner, L.jd, L.dv, L.bufs(), c.cfg.heavy_rows,
                                         L.temp.p, L.temp_cap);
                        loop_insert_keys(c, c.stream, ctl.p, i, L.head, L.temp.p, bufs_of(L.head), nullptr);
                    } else if (L.xp)
                        loop_expand_insert(c, c.stream, ctl.p, i, L.head, o, L.inner, L.jd, L.dv, L.bufs(),
                                           c.cfg.heavy_rows, bufs_of(L.head), nullptr);
                    else if (L.split_insert)
                        loop_insert_keys(c, c.stream, ctl.p, i, L.head, L.temp.p, bufs_of(L.head), nullptr);
                    else
                        loop_materialize_insert(c, c.stream, ctl.p, i, L.head, o, L.inner, L.jd, L.bufs(),
                                                bufs_of(L.head), nullptr);
                }
            };
            // Per-step counters of the steps about to run (again): the
            // candidate counts accumulate atomically; finals keep their
            // post-filter totals (inserted rows of earlier windows / phase A).
            // (phase B keeps step wi's candidate count and scan: the windows
            // are cut from them)
            auto clear_steps = [&](bool phase_b) {
                for (u32 j = 0; j < ns; ++j) {
                    const bool runs = phase_b ? in_v(j) && j > wi : !in_v(j) || j <= wi;
                    if (!runs) continue;
                    hc->step_cand[j] = hc->heavy_n[j] = 0;
                    if (!steps[j].final) hc->step_total[j] = 0;
                }
            };
            u32 redos = 0;
            auto settle = [&](bool phase_b) {  // false: overflowed, grown, state cleared for a redo
                c.d2h(hc, ctl.p, sizeof(LoopCtl));
                c.sync();
                if (!hc->overflow) return true;
                if (++redos > 256) {
                    std::string need;
                    for (u32 j = 0; j < ns; ++j)
                        need += " step" + std::to_string(j) + "(rows " + std::to_string(hc->need_rows[j]) + "/" +
                                std::to_string(steps[j].rows_cap) + " splits " + std::to_string(hc->need_splits[j]) +
                                "/" + std::to_string(steps[j].splits_cap) + " temp " +
                                std::to_string(hc->need_temp[j]) + "/" + std::to_string(steps[j].temp_cap) + ")";
                    throw_logic("windowed iteration: overflow persists after growth:" + need + " log " +
                                std::to_string(hc->need_log[0]) + " tab " + std::to_string(hc->need_tab[0]));
                }
                grow_after_overflow();
                hc->overflow = 0;
                clear_steps(phase_b);
                c.h2d(ctl.p, hc, sizeof(LoopCtl));
                return false;
            };
            do {  // (A) everything outside the windowed part
                for (u32 i = 0; i < ns; ++i)
                    if (!in_v(i) || i <= wi) cand(i, i != wi);
                gate_and_insert(false);
            } while (!settle(false));
            const u64 T = hc->step_cand[wi];
            std::vector<u64> sums(ns, 0);
            for (u64 w = 0; w < T;) {  // (B) the windows
                const u64 hi = std::min(T, w + steps[wi].temp_cap);
                for (u32 j = wi + 1; j < ns; ++j)
                    if (in_v(j)) {
                        hc->step_cand[j] = hc->heavy_n[j] = 0;
                        if (!steps[j].final) hc->step_total[j] = 0;
                    }
                hc->step_total[wi] = 0;
                hc->win_step = wi;
                hc->win_lo = w;
                hc->win_hi = hi;
                c.h2d(ctl.p, hc, sizeof(LoopCtl));
                loop_materialize_temp(c, c.stream, ctl.p, wi, outer_of(steps[wi]), steps[wi].inner, steps[wi].jd,
                                      steps[wi].bufs(), steps[wi].temp.p, steps[wi].temp_cap);
                for (u32 j = wi + 1; j < ns; ++j)
                    if (in_v(j)) cand(j, true);
                gate_and_insert(true);
                if (!settle(true)) continue;
                for (u32 j = wi; j < ns; ++j)
                    if (in_v(j) && !steps[j].final) sums[j] += hc->step_total[j];
                w = hi;
            }
            for (u32 j = wi; j < ns; ++j)
                if (in_v(j) && !steps[j].final) hc->step_total[j] = sums[j];
            hc->win_hi = hc->win_lo = 0;
            c.h2d(ctl.p, hc, sizeof(LoopCtl));
            loop_end(c, c.stream, ctl.p, LoopEndDesc{LoopHist{hist_rec.p, hist_steps.p, ns}, 0, 0, ~0u});
            c.d2h(hc, ctl.p, sizeof(LoopCtl));
            c.sync();
            ++windowed_iters;
        };

        u64 rollbacks = 0;
        u32 done_iters = 0;
        bool need_count = true;  // count_ahead: the current Δ has no candidate total yet
        std::vector<u64> prev_log_n(nh);
        for (u32 h = 0; h < nh; ++h) prev_log_n[h] = hc->h[h].log_n;
        {
            PhaseTimer t(E, "join");
            for (;;) {
                if (eager) {
                    prof_recs.clear();
                    record_iteration(c.stream, false, 0);
                } else {
                    if (count_ahead && need_count) {  // this iteration's candidates, counted once here
                        const LStep& L = steps[0];
                        loop_count(c, c.stream, ctl.p, 0, outer_of(L), L.jd, L.dv, light_bufs(L), ~0ull, nullptr);
                        need_count = false;
                    }
                    const double tb = Ctx::now_s();
                    const bool built = !exec;
                    if (!exec) build_graph();
                    const double tl = Ctx::now_s();
                    for (int b = 0; b < (batch ? batch_n : 1); ++b) GD_CUDA(cudaGraphLaunch(exec, c.stream));
                    if (trace) {
                        const double te = Ctx::now_s();
                        c.d2h(hc, ctl.p, sizeof(LoopCtl));
                        c.sync();
                        fprintf(stderr, "[loop] graph%s: build %.3f ms, launch %.3f ms, run to iter %u %.3f ms\n",
                                built ? " (new)" : "", (tl - tb) * 1e3, (te - tl) * 1e3, hc->iter,
                                (Ctx::now_s() - te) * 1e3);
                    }
                }
                c.d2h(hc, ctl.p, sizeof(LoopCtl));
                c.sync();
                if (!eager)  // kernels that did work (batch: the early-exiting tail too)
                    c.launches += kernels_per_iter * (batch ? (u64)batch_n
                                                            : hc->iter - done_iters + (hc->overflow ? 1 : 0));
                done_iters = hc->iter;
                if (c.prof.on) {
                    // algorithmic bytes: probe = outer key + one
                    // index slot per row; temp = inner row read + row written;
                    // insert = inner row + one membership slot per candidate,
                    // plus the new rows appended (charged to the head's first
                    // final step)
                    std::vector<bool> charged(nh, false);
                    for (const ProfRec& pr : prof_recs) {
                        const LStep& L = steps[pr.step];
                        u64 by = 0;
                        if (pr.kind == 0) by = hc->step_n[pr.step] * (8 + (L.has_iv ? sizeof(Slot) : 0));
                        else if (pr.kind == 4) by = hc->step_n[pr.step] * 16;  // outer key + dense offsets
                        else if (pr.kind == 1) by = hc->last_cand[pr.step] * 16;
                        else {
                            // one key read (kind 2: materialized row; 3: outer row) + one slot
                            by = hc->last_cand[pr.step] * 16;
                            if (!charged[L.head]) {
                                charged[L.head] = true;
                                by += (hc->h[L.head].log_n - prev_log_n[L.head]) * 8;
                            }
                        }
                        c.prof_add_bytes(pr.rec, by);
                    }
                    for (u32 h = 0; h < nh; ++h) prev_log_n[h] = hc->h[h].log_n;
                    c.prof.resolve();
                }
                if (hc->overflow) {
                    // growth / restamp time is index (HISA) build time
                    std::optional<PhaseTimer> tg;
                    tg.emplace(E, "index");
                    const double tblock = Ctx::now_s();
                    ++rollbacks;
                    // a chain temp above the limit: this iteration runs in windows
                    u32 wstep = UINT32_MAX;
                    for (u32 i = 0; i < ns; ++i)
                        if (!steps[i].final && hc->need_temp[i] > temp_limit && wstep == UINT32_MAX) wstep = i;
                    grow_after_overflow();
                    hc->overflow = 0;
                    need_count = true;  // the rollback cleared the candidate totals
                    c.h2d(ctl.p, hc, sizeof(LoopCtl));
                    c.sync();
                    destroy_graph();
                    tg.reset();
                    if (wstep != UINT32_MAX) windowed_iteration(wstep);
                    if (trace)
                        fprintf(stderr, "[loop] iter %u rollback block %.3f ms (meminfo total %.3f ms, alloc total %.3f ms)\n",
                                hc->iter, (Ctx::now_s() - tblock) * 1e3, c.meminfo_seconds * 1e3,
                                c.alloc_seconds * 1e3);
                    continue;
                }
                if (hc->done) break;
            }
        }
        destroy_graph();
        if (cap_stream) cudaStreamDestroy(cap_stream);
        (void)rollbacks;
        if (trace && windowed_iters)
            fprintf(stderr, "[loop] %llu iterations ran with windowed chain temps\n", (unsigned long long)windowed_iters);

        // replay the reference's bookkeeping from the device history
        const u64 iters = hc->iter;
        std::vector<gd_iter_record> recs(iters * nh);
        std::vector<u64> totals(iters * ns);
        if (iters) {
            c.d2h(recs.data(), hist_rec.p, recs.size() * sizeof(gd_iter_record));
            c.d2h(totals.data(), hist_steps.p, totals.size() * sizeof(u64));
            c.sync();
        }
        for (u64 i = 0; i < iters; ++i) replay_iteration(rec, &recs[i * nh], &totals[i * ns], steps);

        // the fixpoint's canonical output: sort each head's log once
        PhaseTimer t(E, "dedup");
        for (u32 h = 0; h < nh; ++h) {
            auto& st = rels[rec[h]];
            LHead& H = heads[h];
            H.tab.release();
            const u64 f = hc->h[h].log_n;
            const u32 ar = E.info_[rec[h]].arity;
            DevBuf<u64> scratch(c, std::max<u64>(f, 1));
            st.piped.reset();
            if (c.cfg.download_pipeline && f >= c.cfg.download_pipeline_min_rows && ar * bits > 8 && ar > 1 &&
                !E.enc.e.dict && c.cfg.sort_pipeline == 0) {
                segmented_final_sort(st, H.log, scratch, f, ar * bits);
                continue;
            }
            u64* sorted = radix_sort<u64>(c, H.log.p, scratch.p, f, ar * bits);
            DevBuf<u64>& res = sorted == H.log.p ? H.log : scratch;
            st.full.release();
            st.full.ctx = res.ctx;
            st.full.p = reinterpret_cast<K*>(res.p);
            st.full.cap = res.cap;
            res.p = nullptr;
            res.cap = 0;
            st.full_n = f;
            st.tail.clear();
            st.delta_n = 0;
            st.new_n = 0;
        }
    }

    // Segmented final sort (PipedPack): the top digit first (one stable pass,
    // its histogram read back for the segment bounds), then each top-digit
    // segment on its low digits (the ranking choice sampled on the first
    // segment and reused), each sorted segment packed for the download with
    // an event behind it.  Same passes and the same sorted keys as
    // radix_sort; the relation's full array is the buffer the segments end
    // in, the other one holds the packed payloads until the download.
    void segmented_final_sort(RelDev<K>& st, DevBuf<u64>& log, DevBuf<u64>& scratch, u64 f, u32 nbits) {
        const u32 npass = (nbits + 7) / 8;
        std::vector<u64> top;
        u64* msd = radix_sort_passes<u64>(c, log.p, scratch.p, f, nbits, npass - 1, npass, nullptr, &top);
        DevBuf<u64>& mbuf = msd == log.p ? log : scratch;
        DevBuf<u64>& obuf = msd == log.p ? scratch : log;
        // the low passes ping-pong between the two buffers: odd counts end in obuf
        DevBuf<u64>& tbuf = (npass - 1) % 2 ? obuf : mbuf;
        auto pp = std::make_unique<PipedPack>();
        u64 off = 0, blk = 0, unit = 0;
        for (u64 d = 0; d < top.size(); ++d) {
            if (!top[d]) continue;
            PipedPack::Seg sg;
            sg.key_off = off;
            sg.cnt = top[d];
            sg.blk_off = blk;
            sg.nblk = (sg.cnt + kByteBlock - 1) / kByteBlock;
            sg.unit_off = unit;
            sg.nunits = (sg.nblk + PipedPack::kUnitB - 1) / PipedPack::kUnitB;
            pp->segs.push_back(sg);
            off += sg.cnt;
            blk += sg.nblk;
            unit += sg.nunits;
        }
        if (off != f) throw Error(GD_ERR_CUDA, "segmented sort: digit counts do not add up to the row count");
        const u64 nseg = pp->segs.size();
        pp->heads = DevBuf<u64>(c, std::max<u64>(blk, 1));
        pp->cls = DevBuf<uint8_t>(c, std::max<u64>(blk, 1));
        pp->offs = DevBuf<u64>(c, blk + nseg);
        pp->uoffs = DevBuf<u64>(c, unit + nseg);
        pp->ev.assign(nseg, nullptr);
        for (auto& e : pp->ev) GD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        std::vector<char> ballot;
        const bool trace = (c.cfg.trace & 4) != 0;
        const double t0 = Ctx::now_s();
        for (u64 i = 0; i < nseg; ++i) {
            if (trace && (i < 4 || i % 16 == 0 || i + 1 == nseg))
                fprintf(stderr, "[segsort] segment %llu/%llu (%llu keys) enqueued at +%.2f ms\n",
                        (unsigned long long)i, (unsigned long long)nseg, (unsigned long long)pp->segs[i].cnt,
                        (Ctx::now_s() - t0) * 1e3);
            const PipedPack::Seg& sg = pp->segs[i];
            u64* r = npass > 1 ? radix_sort_passes<u64>(c, mbuf.p + sg.key_off, obuf.p + sg.key_off, sg.cnt, nbits, 0,
                                                        npass - 1, &ballot, nullptr)
                               : mbuf.p + sg.key_off;
            if (r != tbuf.p + sg.key_off) c.d2d(tbuf.p + sg.key_off, r, sg.cnt * sizeof(u64));
            DevBuf<u64>& sbuf = &tbuf == &mbuf ? obuf : mbuf;
            byte_pack_into(c, tbuf.p + sg.key_off, sg.cnt, pp->heads.p + sg.blk_off, pp->cls.p + sg.blk_off,
                           pp->offs.p + sg.blk_off + i, reinterpret_cast<uint8_t*>(sbuf.p + sg.key_off),
                           PipedPack::kUnitB, pp->uoffs.p + sg.unit_off + i);
            GD_CUDA(cudaEventRecord(pp->ev[i], c.stream));
        }
        if (trace) fprintf(stderr, "[segsort] all segments enqueued at +%.2f ms\n", (Ctx::now_s() - t0) * 1e3);
        DevBuf<u64>& sbuf = &tbuf == &mbuf ? obuf : mbuf;
        st.full.release();
        st.full.ctx = tbuf.ctx;
        st.full.p = reinterpret_cast<K*>(tbuf.p);
        st.full.cap = tbuf.cap;
        tbuf.p = nullptr;
        tbuf.cap = 0;
        st.full_n = f;
        st.tail.clear();
        st.delta_n = 0;
        st.new_n = 0;
        pp->keys = reinterpret_cast<const u64*>(st.full.p);
        pp->n = f;
        pp->spare = std::move(sbuf);
        st.piped = std::move(pp);
    }

    // The reference's per-iteration bookkeeping (engine.hpp:196-251) from the
    // device history: Δ history, iteration records, join tuples and the
    // accountant / EBM charges in the reference's order.
    void replay_iteration(const std::vector<u32>& rec, const gd_iter_record* r, const u64* totals,
                          const std::vector<LStep>& steps) {
        ++E.iterations;
        auto head_of = [&](u32 rel) -> int {
            auto it = std::find(rec.begin(), rec.end(), rel);
            return it == rec.end() ? -1 : (int)(it - rec.begin());
        };
        for (size_t i = 0; i < rec.size(); ++i) E.info_[rec[i]].history.push_back(r[i].delta_in);
        std::vector<u64> joined(rels.size(), 0);
        size_t g = 0;
        for (const auto& p : E.plans_) {
            if (!p.recursive) continue;
            for (u32 v = 0; v < p.nvariants; ++v) {
                const gd_variant& var = p.variants[v];
                const u32 n = std::max<u32>(1, var.nsteps);
                const int sh = head_of(var.src_rel);
                const bool use_delta = var.src_version == GD_DELTA;
                u64 cur_n;
                if (sh >= 0) cur_n = use_delta ? r[sh].delta_in : r[sh].full_after - r[sh].delta_out;
                else cur_n = rels[var.src_rel].full_n;
                if (!(use_delta && cur_n == 0)) {
                    const u64 m = replay_chain(var, cur_n, totals + g);
                    joined[p.head_rel] += m;
                    append_new(p.head_rel, m);
                }
                g += n;
            }
        }
        for (size_t i = 0; i < rec.size(); ++i) {
            const u32 rr = rec[i];
            RelInfo& ri = E.info_[rr];
            const u32 ar = ri.arity;
            if (joined[rr] != r[i].join) throw_logic("device loop: join count mismatch in the iteration record");
            const u64 m = r[i].join;
            if (m > 0) Tracked scratch(E.acct, Accountant::kTemp, m * 8 + rb(m, ar), "dedup");
            Tracked fresh_charge(E.acct, Accountant::kTemp, rb(r[i].new_unique, ar), "dedup");
            E.acct.release(Accountant::kContainer, ri.new_bytes);
            ri.new_bytes = 0;
            fresh_charge.reset();
            assign_delta(rr, r[i].delta_out, "difference");
            if (r[i].delta_out > 0) {
                merge_accounting(rr, r[i].full_after - r[i].delta_out, r[i].delta_out, "merge");
                ++rels[rr].merge_gen;
                rels[rr].last_merge_was_delta = true;
                rels[rr].dirty = true;
            }
            ri.log.push_back(r[i]);
        }
    }

    // execute_chain's charges (engine.hpp:401-484) for known step totals.
    u64 replay_chain(const gd_variant& v, u64 cur_n, const u64* totals) {
        const u32 ar = E.info_[v.src_rel].arity;
        Tracked permuted_charge;
        if (!is_identity(v.src_perm, ar)) {
            Tracked scratch(E.acct, Accountant::kTemp, 2 * rb(cur_n, ar) + cur_n * 8, "join");
            scratch.reset();
            permuted_charge = Tracked(E.acct, Accountant::kTemp, rb(cur_n, ar), "join");
        }
        if (v.nsteps == 0) return totals[0];
        Tracked chained_charge;
        for (u32 s = 0; s < v.nsteps; ++s) {
            const u64 total = totals[s];
            Tracked out_charge(E.acct, Accountant::kTemp, total * v.steps[s].proj_arity * 8ull, "join");
            E.join_tuples += total;
            if (s + 1 == v.nsteps) return total;
            chained_charge = std::move(out_charge);
            permuted_charge.reset();
        }
        return 0;
    }

    // ---- hash-partitioned mode -----------------------------
    void partition_begin(u64* send_counts, const void** d_send) override;
    void partition_end(const void* d_recv, u64 recv_rows, u64* local_delta) override;
    u64 partition_run(Comm& comm, u64 max_iters) override;
    void partition_finish() override { part_loop_finish(); }

    // ---- partitioned mode on the loop kernels ------------------------------
    // Per iteration (driven by partition.py): probe / scan / materialize of
    // the local Δ into the final step's temp, rows grouped by owner on the
    // device (the NCCL all-to-all sends them), then the received rows are
    // inserted into this rank's full-tuple index and log (loop_insert_keys).
    // The Δ window and the iteration record are kept on the host; capacities
    // are grown before the kernels that need them, so nothing rolls back.
    struct PartLoop {
        std::vector<u32> rec;
        std::vector<LHead> heads;
        std::vector<LStep> steps;
        DevBuf<LoopCtl> ctl;
        // own pinned host copy (several engines may share one context;
        // pageable copies would stage through the driver every transfer)
        struct PartHost {
            LoopCtl ctl;
            unsigned long long cnt[kLoopMaxRanks], off[kLoopMaxRanks];
            u64 rmeta[3 * kLoopMaxRanks];  // native driver: (count, |Δ|, overflow) from each peer
        };
        DevBuf<u64> recv, meta_send, meta_recv;  // native driver
        DevBuf<gd_iter_record> hist;
        u64 hist_cap = 0;
        struct PinnedFree {
            void operator()(PartHost* p) const { cudaFreeHost(p); }
        };
        std::unique_ptr<PartHost, PinnedFree> host;
        LoopCtl* hc = nullptr;
        DevBuf<u64> block_sums, send;
        DevBuf<unsigned long long> counts, offs, cursors;
        u32 final_step = 0;
    };
    std::unique_ptr<PartLoop> pl;

    bool part_loop_eligible(u32 rec_rel) {
        if constexpr (!std::is_same_v<K, u64>) return false;
        if (!c.cfg.partition_loop) return false;
        if (E.nranks > kLoopMaxRanks) return false;
        const auto& st = rels[rec_rel];
        if (!st.lsm || st.delta_n != total_n(st)) return false;
        u32 nv = 0;
        for (const auto& p : E.plans_) {
            if (!p.recursive) continue;
            for (u32 v = 0; v < p.nvariants; ++v) {
                const gd_variant& var = p.variants[v];
                if (var.src_rel != rec_rel || var.src_version != GD_DELTA || var.nsteps == 0) return false;
                ++nv;
            }
        }
        return nv == 1;  // one variant: the final step's temp is the send set
    }

    void part_loop_setup(u32 rec_rel) {
        pl.reset(new PartLoop);
        PartLoop& P = *pl;
        loop_prepare();
        std::vector<u32> by_name(rels.size());
        for (u32 i = 0; i < by_name.size(); ++i) by_name[i] = i;
        for (u32 r : by_name)
            if (rels[r].dirty && !rels[r].copies.empty()) refresh_copies(r);
        P.rec = {rec_rel};
        P.heads.resize(1);
        LHead& H = P.heads[0];
        auto& st = rels[rec_rel];
        compact(st);
        H.rel = rec_rel;
        const u64 f0 = st.full_n;
        // min_capacities: the log and index start full, so the growth paths
        // (host-driven growth; stalls of the peer-memory loop) run on small inputs
        const bool tiny0 = c.cfg.min_capacities != 0;
        H.log_cap = tiny0 ? std::max<u64>(f0, 1) : std::max<u64>(2 * f0, 1 << 16);
        H.log = DevBuf<u64>(c, H.log_cap);
        if (f0) c.d2d(H.log.p, st.full.p, f0 * sizeof(u64));
        H.sbits = loop_stamp_bits(E.info_[rec_rel].arity * bits);
        H.alloc_tab(c, tiny0 ? 2 * f0 + 16 : std::max<u64>(4 * f0, 1 << 16));
        loop_table_fill(c, H.tab.p, H.tab_cap, H.sbits, H.log.p, f0);
        build_loop_steps(P.rec, P.steps);
        P.final_step = (u32)P.steps.size() - 1;
        for (auto& L : P.steps) {
            // min_capacities: tests walk the overflow -> grow -> redo path of
            // both partitioned drivers
            const bool tiny = c.cfg.min_capacities != 0;
            L.rows_cap = tiny ? 2 : std::max<u64>(f0 + 1, 1 << 12);
            L.splits_cap = tiny ? 2 : std::max<u64>(2 * f0 / kLoopMatTile + 2, 1 << 12);
            L.alloc_rows(c);
            L.splits = DevBuf<u64>(c, L.splits_cap);
            L.temp_cap = tiny ? 1 : std::max<u64>(4 * f0, 1 << 16);
            L.temp = DevBuf<u64>(c, L.temp_cap);
        }
        P.block_sums = DevBuf<u64>(c, (u64)loop_grid(c));
        P.counts = DevBuf<unsigned long long>(c, kLoopMaxRanks);
        P.offs = DevBuf<unsigned long long>(c, kLoopMaxRanks);
        P.cursors = DevBuf<unsigned long long>(c, kLoopMaxRanks);
        P.ctl = DevBuf<LoopCtl>(c, 1);
        {
            void* hp = nullptr;
            GD_CUDA(cudaMallocHost(&hp, sizeof(typename PartLoop::PartHost)));
            P.host.reset(static_cast<typename PartLoop::PartHost*>(hp));
        }
        P.hc = &P.host->ctl;
        std::memset(P.hc, 0, sizeof(LoopCtl));
        P.hc->nheads = 1;
        P.hc->hist_cap = ~0ull;
        P.hc->h[0].log_n = f0;
        P.hc->h[0].dlo = f0 - st.delta_n;
        P.hc->h[0].dhi = f0;
        c.h2d(P.ctl.p, P.hc, sizeof(LoopCtl));
    }

    LoopHeadBufs part_bufs() {
        LHead& H = pl->heads[0];
        LoopHeadBufs b{};
        b.log = H.log.p;
        b.log_cap = H.log_cap;
        b.tab = H.tab.p;
        b.tab_cap = H.tab_cap;
        b.tab_limit = H.tab_limit;
        b.sbits = H.sbits;
        b.warp_append = c.cfg.warp_append;
        return b;
    }

    void part_loop_begin(u64* send_counts, const void** d_send) {
        PartLoop& P = *pl;
        LoopCtl* hc = P.hc;
        const u32 ns = (u32)P.steps.size();
        const u32 R = E.nranks;
        const LStep& F = P.steps[P.final_step];
        const u64* n_ptr = &P.ctl.p->step_total[P.final_step];
        unsigned long long* cnt = P.host->cnt;
        for (;;) {  // the join part; regrown and rerun on a capacity overflow
            for (u32 i = 0; i < ns; ++i) {
                LStep& L = P.steps[i];
                LoopOuter o{};
                o.kind = L.kind;
                o.head = L.src_head;
                o.src_step = L.src_step;
                o.ptr = L.kind == LO_TEMP ? P.steps[L.src_step].temp.p : P.heads[0].log.p;
                loop_probe(c, c.stream, P.ctl.p, i, o, L.jd, L.has_iv ? &L.iv : nullptr, L.dv, L.inner_n, L.bufs(),
                           P.block_sums.p);
                loop_scan(c, c.stream, P.ctl.p, i, o, L.bufs(), P.block_sums.p, nullptr);
                loop_materialize_temp(c, c.stream, P.ctl.p, i, o, L.inner, L.jd, L.bufs(), L.temp.p, L.temp_cap);
            }
            // owner counts of the final step's rows, read back with the
            // control block (one round trip; discarded on an overflow)
            c.memset(P.counts.p, 0, R * sizeof(unsigned long long));
            loop_owner_count(c, F.temp.p, n_ptr, F.temp_cap, R, P.counts.p);
            c.d2h(hc, P.ctl.p, sizeof(LoopCtl));
            c.d2h(cnt, P.counts.p, R * sizeof(unsigned long long));
            c.sync();
            if (!hc->overflow) break;
            for (u32 i = 0; i < ns; ++i) {
                LStep& L = P.steps[i];
                if (hc->need_rows[i] > L.rows_cap) {
                    L.rows_cap = hc->need_rows[i] + hc->need_rows[i] / 2;
                    L.alloc_rows(c);
                }
                if (hc->need_splits[i] > L.splits_cap) {
                    L.splits_cap = hc->need_splits[i] + hc->need_splits[i] / 2;
                    L.splits = DevBuf<u64>(c, L.splits_cap);
                }
                if (hc->need_temp[i] > L.temp_cap) {
                    L.temp_cap = hc->need_temp[i] + hc->need_temp[i] / 2;
                    L.temp = DevBuf<u64>(c, L.temp_cap);
                }
                hc->need_rows[i] = hc->need_splits[i] = hc->need_temp[i] = 0;
                hc->step_total[i] = 0;
            }
            hc->overflow = 0;
            c.h2d(P.ctl.p, hc, sizeof(LoopCtl));
        }
        for (u32 i = 0; i < ns; ++i) E.join_tuples += hc->step_total[i];
        // group the final step's rows by owner
        const u64 m = hc->step_total[P.final_step];
        P.send.reserve_discard(c, std::max<u64>(m, 1));
        c.memset(P.cursors.p, 0, R * sizeof(unsigned long long));
        unsigned long long* off = P.host->off;
        u64 acc = 0;
        for (u32 k = 0; k < R; ++k) {
            off[k] = acc;
            acc += cnt[k];
            send_counts[k] = cnt[k];
        }
        c.h2d(P.offs.p, off, R * sizeof(unsigned long long));
        if (m) loop_owner_scatter(c, F.temp.p, n_ptr, R, P.offs.p, P.cursors.p, P.send.p);
        c.sync();
        // clear the per-iteration step totals for the next iteration
        for (u32 i = 0; i < ns; ++i) hc->step_total[i] = 0;
        c.h2d(P.ctl.p, hc, sizeof(LoopCtl));
        *d_send = m ? P.send.p : nullptr;
    }

    void part_loop_end(const void* d_recv, u64 recv_rows, u64* local_delta) {
        PartLoop& P = *pl;
        LoopCtl* hc = P.hc;
        LHead& H = P.heads[0];
        const u32 r = H.rel;
        const u64 din = hc->h[0].dhi - hc->h[0].dlo;
        ++E.iterations;
        E.info_[r].history.push_back(din);
        // capacities before the inserts (no rollback in this mode)
        const u64 ln = hc->h[0].log_n;
        const u64 need = ln + recv_rows;
        if (need > H.log_cap) {
            const u64 cap = 2 * need;
            DevBuf<u64> nl(c, cap);
            if (ln) loop_copy_u64(c, nl.p, H.log.p, ln);
            H.log = std::move(nl);
            H.log_cap = cap;
        }
        if (need > H.tab_limit) {
            DevBuf<u64> old = std::move(H.tab);
            const u64 old_cap = H.tab_cap;
            H.alloc_tab(c, 8 * need, false, false);
            loop_table_rehash(c, old.p, old_cap, H.tab.p, H.tab_cap, H.sbits, ln);
        }
        if (hc->iter + 1 - hc->epoch_base > (H.sbits ? (1u << H.sbits) - 1 : 0xfffffffeu)) {
            loop_table_restamp(c, H.tab.p, H.tab_cap, H.sbits);
            hc->epoch_base = hc->iter;
        }
        hc->step_total[P.final_step] = recv_rows;  // the insert kernel's row count
        hc->h[0].J = hc->h[0].N = hc->h[0].D = 0;
        c.h2d(P.ctl.p, hc, sizeof(LoopCtl));
        if (recv_rows)
            loop_insert_keys(c, c.stream, P.ctl.p, P.final_step, 0, static_cast<const u64*>(d_recv), part_bufs(),
                             nullptr);
        c.d2h(hc, P.ctl.p, sizeof(LoopCtl));
        c.sync();
        const u64 D = hc->h[0].D, N = hc->h[0].N;
        hc->h[0].dlo = hc->h[0].dhi;
        hc->h[0].dhi = hc->h[0].log_n;
        hc->iter += 1;
        hc->step_total[P.final_step] = 0;
        c.h2d(P.ctl.p, hc, sizeof(LoopCtl));
        E.info_[r].log.push_back(gd_iter_record{din, recv_rows, N, D, hc->h[0].log_n});
        *local_delta = D;
    }

    // Native partitioned driver (gd_engine_run_partitioned):
    // the iteration of part_loop_begin / exchange / part_loop_end with the
    // exchanges as NCCL send/recv on the engine's stream and one host
    // synchronisation per iteration (the counts readback).  An overflow on
    // any rank travels in the counts exchange, so every rank redoes the
    // join together; |Δ| travels there too (termination without an
    // all-reduce); the end-of-iteration bookkeeping runs on the device and
    // the per-iteration records are read once at the end.
    u64 part_loop_run(Comm& comm, u64 max_iters) {
        PartLoop& P = *pl;
        LoopCtl* hc = P.hc;
        const u32 ns = (u32)P.steps.size();
        const u32 R = E.nranks;
        if (comm.nranks != R || comm.rank != E.rank)
            throw_usage("gd_engine_run_partitioned: communicator does not match set_partition");
        const LStep& F = P.steps[P.final_step];
        const u64* n_ptr = &P.ctl.p->step_total[P.final_step];
        LHead& H = P.heads[0];
        const u32 r = H.rel;
        auto* ph = P.host.get();
        if (!P.meta_send.p) {
            P.meta_send = DevBuf<u64>(c, 3 * (u64)R);
            P.meta_recv = DevBuf<u64>(c, 3 * (u64)R);
        }
        const u64 hist0 = hc->iter;  // records already kept on the host (Python protocol)
        auto grow_hist = [&](u64 need) {
            if (need <= P.hist_cap) return;
            const u64 cap = std::max<u64>(need, 2 * P.hist_cap + 256);
            DevBuf<gd_iter_record> h2(c, cap);
            if (P.hist_cap) c.d2d(h2.p, P.hist.p, P.hist_cap * sizeof(gd_iter_record));
            P.hist = std::move(h2);
            P.hist_cap = cap;
        };
        grow_hist(hist0 + 256);
        u64 it = 0;
        bool first = true;  // the seeded Δ: the first iteration always runs (as run_partitioned)
        while (it < max_iters) {
            // (1) joins on the local Δ, owner counts, counts + |Δ| + overflow to every peer
            for (u32 i = 0; i < ns; ++i) {
                LStep& L = P.steps[i];
                LoopOuter o{};
                o.kind = L.kind;
                o.head = L.src_head;
                o.src_step = L.src_step;
                o.ptr = L.kind == LO_TEMP ? P.steps[L.src_step].temp.p : H.log.p;
                loop_probe(c, c.stream, P.ctl.p, i, o, L.jd, L.has_iv ? &L.iv : nullptr, L.dv, L.inner_n, L.bufs(),
                           P.block_sums.p);
                loop_scan(c, c.stream, P.ctl.p, i, o, L.bufs(), P.block_sums.p, nullptr);
                loop_materialize_temp(c, c.stream, P.ctl.p, i, o, L.inner, L.jd, L.bufs(), L.temp.p, L.temp_cap);
            }
            c.memset(P.counts.p, 0, R * sizeof(unsigned long long));
            loop_owner_count(c, F.temp.p, n_ptr, F.temp_cap, R, P.counts.p);
            loop_part_meta(c, P.counts.p, P.ctl.p, R, first ? 1 : 0, P.meta_send.p);
            comm.t->group_start();
            for (u32 q = 0; q < R; ++q) {
                comm.t->send(P.meta_send.p + 3 * q, 3, q, c.stream);
                comm.t->recv(P.meta_recv.p + 3 * q, 3, q, c.stream);
            }
            comm.t->group_end(c.stream);
            c.d2h(hc, P.ctl.p, sizeof(LoopCtl));
            c.d2h(ph->rmeta, P.meta_recv.p, 3 * R * sizeof(u64));
            c.d2h(ph->cnt, P.counts.p, R * sizeof(unsigned long long));
            c.sync();
            bool any_over = false;
            u64 gdelta = 0;
            for (u32 q = 0; q < R; ++q) {
                gdelta += ph->rmeta[3 * q + 1];
                any_over |= ph->rmeta[3 * q + 2] != 0;
            }
            if (any_over) {  // some rank outgrew a buffer: all ranks redo the join
                for (u32 i = 0; i < ns; ++i) {
                    LStep& L = P.steps[i];
                    if (hc->need_rows[i] > L.rows_cap) {
                        L.rows_cap = hc->need_rows[i] + hc->need_rows[i] / 2;
                        L.alloc_rows(c);
                    }
                    if (hc->need_splits[i] > L.splits_cap) {
                        L.splits_cap = hc->need_splits[i] + hc->need_splits[i] / 2;
                        L.splits = DevBuf<u64>(c, L.splits_cap);
                    }
                    if (hc->need_temp[i] > L.temp_cap) {
                        L.temp_cap = hc->need_temp[i] + hc->need_temp[i] / 2;
                        L.temp = DevBuf<u64>(c, L.temp_cap);
                    }
                    hc->need_rows[i] = hc->need_splits[i] = hc->need_temp[i] = 0;
                    hc->step_total[i] = 0;
                }
                hc->overflow = 0;
                c.h2d(P.ctl.p, hc, sizeof(LoopCtl));
                continue;
            }
            first = false;
            if (gdelta == 0) {  // every rank's Δ was empty: no rows were produced anywhere
                for (u32 i = 0; i < ns; ++i) hc->step_total[i] = 0;
                c.h2d(P.ctl.p, hc, sizeof(LoopCtl));
                break;
            }
            for (u32 i = 0; i < ns; ++i) E.join_tuples += hc->step_total[i];
            // (2) group the final step's rows by owner
            const u64 m = hc->step_total[P.final_step];
            P.send.reserve_discard(c, std::max<u64>(m, 1));
            u64 acc = 0;
            for (u32 q = 0; q < R; ++q) {
                ph->off[q] = acc;
                acc += ph->cnt[q];
            }
            c.memset(P.cursors.p, 0, R * sizeof(unsigned long long));
            c.h2d(P.offs.p, ph->off, R * sizeof(unsigned long long));
            if (m) loop_owner_scatter(c, F.temp.p, n_ptr, R, P.offs.p, P.cursors.p, P.send.p);
            // (3) rows all-to-all-v
            u64 total_recv = 0;
            for (u32 q = 0; q < R; ++q) total_recv += ph->rmeta[3 * q];
            P.recv.reserve_discard(c, std::max<u64>(total_recv, 1));
            comm.t->group_start();
            u64 roff = 0;
            for (u32 q = 0; q < R; ++q) {
                if (ph->cnt[q])
                    comm.t->send(P.send.p + ph->off[q], ph->cnt[q], q, c.stream);
                const u64 rc = ph->rmeta[3 * q];
                if (rc) comm.t->recv(P.recv.p + roff, rc, q, c.stream);
                roff += rc;
            }
            comm.t->group_end(c.stream);
            // (4) capacities, insert, device-side end of the iteration
            const u64 ln = hc->h[0].log_n;
            const u64 need = ln + total_recv;
            if (need > H.log_cap) {
                const u64 cap = 2 * need;
                DevBuf<u64> nl(c, cap);
                if (ln) loop_copy_u64(c, nl.p, H.log.p, ln);
                H.log = std::move(nl);
                H.log_cap = cap;
            }
            if (need > H.tab_limit) {
                DevBuf<u64> old = std::move(H.tab);
                const u64 old_cap = H.tab_cap;
                H.alloc_tab(c, 8 * need, false, false);
                loop_table_rehash(c, old.p, old_cap, H.tab.p, H.tab_cap, H.sbits, ln);
            }
            if (hc->iter + 1 - hc->epoch_base > (H.sbits ? (1u << H.sbits) - 1 : 0xfffffffeu)) {
                loop_table_restamp(c, H.tab.p, H.tab_cap, H.sbits);
                hc->epoch_base = hc->iter;
            }
            grow_hist(hc->iter + 1);
            hc->step_total[P.final_step] = total_recv;  // the insert kernel's row count
            hc->h[0].J = hc->h[0].N = hc->h[0].D = 0;
            c.h2d(P.ctl.p, hc, sizeof(LoopCtl));
            if (total_recv)
                loop_insert_keys(c, c.stream, P.ctl.p, P.final_step, 0, P.recv.p, part_bufs(), nullptr);
            loop_part_advance(c, P.ctl.p, P.final_step, total_recv, P.hist.p);
            ++it;
        }
        // the host mirror and the per-iteration records, once
        c.d2h(hc, P.ctl.p, sizeof(LoopCtl));
        std::vector<gd_iter_record> recs(it);
        if (it) c.d2h(recs.data(), P.hist.p + hist0, it * sizeof(gd_iter_record));
        c.sync();
        for (const auto& rec : recs) {
            ++E.iterations;
            E.info_[r].history.push_back(rec.delta_in);
            E.info_[r].log.push_back(rec);
        }
        return it;
    }

    // ---- peer-memory partitioned loop (gd_device_config.partition_exchange
    // = 0) ------------------------------------------------------
    // Mailbox + inbox of this rank (cudaMalloc bases: CUDA IPC maps them into
    // the other ranks), their peer mappings and the device routing table.
    struct PeerState {
        Transport* t = nullptr;
        PeerMail* mail = nullptr;
        u64* inbox = nullptr;
        u64 inbox_cap = 0;
        std::vector<void*> mails, inboxes;
        // inboxes replaced by a regrow: freed only when the run ends (a
        // cudaFree synchronizes the device, and loopback ranks sharing it
        // may be spinning in a device barrier)
        std::vector<std::pair<u64*, std::vector<void*>>> retired;
        DevBuf<PeerTab> tab;
        ~PeerState() {
            if (t) {
                t->unmap_peers(inboxes);
                t->unmap_peers(mails);
                for (auto& r : retired) t->unmap_peers(r.second);
            }
            for (auto& r : retired) cudaFree(r.first);
            if (inbox) cudaFree(inbox);
            if (mail) cudaFree(mail);
        }
    };

    // Sum (op 0) / max (op 1) of n words over all ranks, through the
    // transport (rare paths only: rollbacks and stalls).  Also a barrier.
    void host_allreduce(Comm& comm, u64* v, u32 n, int op) {
        const u32 R = comm.nranks;
        if (R == 1) return;
        DevBuf<u64> d(c, (u64)n * (R + 1));
        c.h2d(d.p, v, n * sizeof(u64));
        comm.t->group_start();
        for (u32 q = 0; q < R; ++q) {
            if (q == comm.rank) continue;
            comm.t->send(d.p, n, q, c.stream);
            comm.t->recv(d.p + (u64)n * (q + 1), n, q, c.stream);
        }
        comm.t->group_end(c.stream);
        std::vector<u64> all((u64)n * R);
        c.d2h(all.data(), d.p + n, (u64)n * R * sizeof(u64));
        c.sync();
        for (u32 q = 0; q < R; ++q) {
            if (q == comm.rank) continue;
            for (u32 k = 0; k < n; ++k) v[k] = op ? std::max(v[k], all[(u64)q * n + k]) : v[k] + all[(u64)q * n + k];
        }
    }

    void peer_map_inbox(Comm& comm, PeerState& ps, u64 cap) {
        if (ps.inbox) {
            ps.retired.emplace_back(ps.inbox, std::move(ps.inboxes));
            ps.inboxes.clear();
            ps.inbox = nullptr;
        }
        GD_CUDA(cudaMalloc(&ps.inbox, std::max<u64>(cap, 1) * sizeof(u64)));
        ps.inbox_cap = cap;
        comm.t->map_peers(ps.inbox, ps.inboxes, c.stream);
        std::vector<u64> caps(comm.nranks, 0);
        caps[comm.rank] = cap;
        host_allreduce(comm, caps.data(), comm.nranks, 0);
        PeerTab h{};
        h.P = comm.nranks;
        h.rank = comm.rank;
        for (u32 q = 0; q < comm.nranks; ++q) {
            h.inbox[q] = static_cast<u64*>(ps.inboxes[q]);
            h.cap[q] = caps[q];
            h.mail[q] = static_cast<PeerMail*>(ps.mails[q]);
        }
        c.h2d(ps.tab.p, &h, sizeof(PeerTab));
        c.sync();
    }

    // Grows log / index / stamps / history of the single head after a stall
    // (the insert of the received rows did not fit).
    void peer_grow_head(LHead& H, u64 ln, u64 need) {
        PartLoop& P = *pl;
        LoopCtl* hc = P.hc;
        if (need > H.log_cap) {
            const u64 cap = std::max<u64>(2 * need, 1 << 16);
            DevBuf<u64> nl(c, cap);
            if (ln) loop_copy_u64(c, nl.p, H.log.p, ln);
            H.log = std::move(nl);
            H.log_cap = cap;
        }
        if (need > H.tab_limit) {  // load 1/index_growth after the growth when free HBM allows
            const u64 sb = loop_slot_bytes(H.sbits);
            const u64 reserve = 1ull << 30, spill = (ln / 16 + (1u << 20)) * sizeof(u64);
            const u64 avail = c.available_bytes(true);  // exact: other ranks may share this GPU (loopback)
            const u64 fit = avail > reserve + spill ? (avail - reserve - spill) / sb : 0;
            const u64 cap = std::min<u64>((u64)c.cfg.index_growth * need, fit);
            if (cap < need / 3 * 4 + 16)
                throw_budget("index", "device memory cannot hold the full-tuple index of " + std::to_string(need) +
                                          " keys");
            DevBuf<u64> old = std::move(H.tab);
            const u64 old_cap = H.tab_cap;
            H.alloc_tab(c, cap, cap < 2 * need, false);
            loop_table_rehash(c, old.p, old_cap, H.tab.p, H.tab_cap, H.sbits, ln);
        }
        if (hc->iter + 1 - hc->epoch_base > (H.sbits ? (1u << H.sbits) - 1 : 0xfffffffeu)) {
            loop_table_restamp(c, H.tab.p, H.tab_cap, H.sbits);
            hc->epoch_base = hc->iter;
        }
    }

    // The whole partitioned fixpoint as one CUDA graph per rank: per
    // iteration the joins of the local Δ, the final step's rows routed into
    // their owners' inboxes over peer memory, barrier 1 (overflow consensus,
    // received count, capacity gate), the insert of the inbox into this
    // rank's full-tuple index and log, barrier 2 (record, Δ window, |Δ| sum
    // -> the while condition).  No host round trip per iteration; the host
    // steps in only to grow a buffer (every rank rolls back together) or to
    // finish a stalled insert.
    u64 part_peer_run(Comm& comm, u64 max_iters) {
        PartLoop& P = *pl;
        LoopCtl* hc = P.hc;
        const u32 ns = (u32)P.steps.size();
        const u32 R = E.nranks;
        if (comm.nranks != R || comm.rank != E.rank)
            throw_usage("gd_engine_run_partitioned: communicator does not match set_partition");
        LHead& H = P.heads[0];
        const u32 r = H.rel;
        const bool tiny = c.cfg.min_capacities != 0;
        PeerState ps;
        ps.t = comm.t;
        GD_CUDA(cudaMalloc(&ps.mail, sizeof(PeerMail)));
        GD_CUDA(cudaMemsetAsync(ps.mail, 0, sizeof(PeerMail), c.stream));
        ps.tab = DevBuf<PeerTab>(c, 1);
        comm.t->map_peers(ps.mail, ps.mails, c.stream);
        const u64 f0 = hc->h[0].log_n;
        peer_map_inbox(comm, ps, tiny ? 1 : std::max<u64>(2 * f0 / R + 1024, 1 << 20));

        const u64 hist0 = hc->iter;
        auto grow_hist = [&](u64 need) {
            if (need <= P.hist_cap) return;
            const u64 cap = std::max<u64>(need, 2 * P.hist_cap + 256);
            DevBuf<gd_iter_record> h2(c, cap);
            if (P.hist_cap) c.d2d(h2.p, P.hist.p, P.hist_cap * sizeof(gd_iter_record));
            P.hist = std::move(h2);
            P.hist_cap = cap;
        };
        grow_hist(hist0 + (tiny ? 1 : 1024));
        hc->part_epoch = 0;
        hc->part_join = 0;
        hc->part_over = hc->part_stall = hc->part_stall_any = hc->part_inbox_over = hc->part_timeout = 0;
        hc->overflow = hc->done = 0;
        c.h2d(P.ctl.p, hc, sizeof(LoopCtl));

        auto outer_of = [&](const LStep& L) {
            LoopOuter o{};
            o.kind = L.kind;
            o.head = L.src_head;
            o.src_step = L.src_step;
            o.ptr = L.kind == LO_TEMP ? P.steps[L.src_step].temp.p : H.log.p;
            return o;
        };
        auto record_iteration = [&](cudaStream_t s, bool use_cond, unsigned long long cond) {
            PeerSyncDesc d{};
            d.tab = ps.tab.p;
            d.final_step = P.final_step;
            d.nsteps = ns;
            d.log_cap = H.log_cap;
            d.tab_limit = H.tab_limit;
            d.stamp_max = H.sbits ? (1u << H.sbits) - 1 : 0xfffffffeu;
            d.hist = P.hist.p;
            d.hist_cap = P.hist_cap;
            d.cond = cond;
            d.use_cond = use_cond ? 1 : 0;
            d.timeout_ns = (u64)c.cfg.peer_timeout_ms * 1000000ull;
            for (u32 i = 0; i < ns; ++i) {
                LStep& L = P.steps[i];
                const LoopOuter o = outer_of(L);
                if (L.final && L.xp) {
                    loop_count(c, s, P.ctl.p, i, o, L.jd, L.dv, L.bufs(), c.cfg.heavy_rows, nullptr);
                    loop_expand_route(c, s, P.ctl.p, i, o, L.inner, L.jd, L.dv, L.bufs(), c.cfg.heavy_rows,
                                      ps.tab.p);
                    continue;
                }
                loop_probe(c, s, P.ctl.p, i, o, L.jd, L.has_iv ? &L.iv : nullptr, L.dv, L.inner_n, L.bufs(),
                           P.block_sums.p);
                loop_scan(c, s, P.ctl.p, i, o, L.bufs(), P.block_sums.p, nullptr);
                loop_materialize_temp(c, s, P.ctl.p, i, o, L.inner, L.jd, L.bufs(), L.temp.p, L.temp_cap);
                if (L.final) loop_route_keys(c, s, P.ctl.p, i, L.temp.p, ps.tab.p);
            }
            loop_peer_sync1(c, s, P.ctl.p, d);
            loop_insert_keys(c, s, P.ctl.p, P.final_step, 0, ps.inbox, part_bufs(), nullptr);
            loop_peer_sync2(c, s, P.ctl.p, d);
        };

        const bool eager = c.prof.on || c.cfg.loop_mode != GD_LOOP_GRAPH;
        cudaGraphExec_t exec = nullptr;
        cudaGraph_t graph = nullptr;
        cudaStream_t cap_stream = nullptr;
        u64 kernels_per_iter = 0;
        auto destroy_graph = [&]() {
            if (exec) cudaGraphExecDestroy(exec);
            if (graph) cudaGraphDestroy(graph);
            exec = nullptr;
            graph = nullptr;
        };
        auto build_graph = [&]() {
            destroy_graph();
            if (!cap_stream) GD_CUDA(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
            GD_CUDA(cudaGraphCreate(&graph, 0));
            cudaGraphConditionalHandle hdl;
            GD_CUDA(cudaGraphConditionalHandleCreate(&hdl, graph, 1, cudaGraphCondAssignDefault));
            cudaGraphNodeParams np{};
            np.type = cudaGraphNodeTypeConditional;
            np.conditional.handle = hdl;
            np.conditional.type = cudaGraphCondTypeWhile;
            np.conditional.size = 1;
            cudaGraphNode_t node;
            GD_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &np));
            cudaGraph_t body = np.conditional.phGraph_out[0];
            GD_CUDA(cudaStreamBeginCaptureToGraph(cap_stream, body, nullptr, nullptr, 0,
                                                  cudaStreamCaptureModeThreadLocal));
            const u64 l0 = c.launches;
            try {
                record_iteration(cap_stream, true, (unsigned long long)hdl);
            } catch (...) {
                cudaStreamEndCapture(cap_stream, &body);
                throw;
            }
            kernels_per_iter = c.launches - l0;
            c.launches = l0;
            GD_CUDA(cudaStreamEndCapture(cap_stream, &body));
            GD_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        };
        struct Cleanup {
            std::function<void()> f;
            ~Cleanup() { f(); }
        } cleanup{[&] {
            destroy_graph();
            if (cap_stream) cudaStreamDestroy(cap_stream);
        }};

        u32 done_iters = hc->iter;
        const u64 iter_limit = hist0 + max_iters;
        // Every rank has its graph built (and its buffers set) before any
        // rank launches: a rank spinning in a device barrier must never wait
        // on a peer stuck in a host call that synchronizes the device
        // (loopback ranks share one GPU).
        auto ready = [&]() {
            if (!eager && !exec) build_graph();
            u64 bar = 0;
            host_allreduce(comm, &bar, 1, 0);
        };
        ready();
        for (;;) {
            if (eager) {
                record_iteration(c.stream, false, 0);
            } else {
                GD_CUDA(cudaGraphLaunch(exec, c.stream));
            }
            c.d2h(hc, P.ctl.p, sizeof(LoopCtl));
            c.sync();
            if (!eager) c.launches += kernels_per_iter * (hc->iter - done_iters + (hc->part_over ? 1 : 0));
            done_iters = hc->iter;
            if (hc->part_timeout)
                throw Error(GD_ERR_NCCL, "partitioned loop: a peer did not reach the device barrier within " +
                                             std::to_string(c.cfg.peer_timeout_ms) + " ms (rank " +
                                             std::to_string(comm.rank) + ", iteration " + std::to_string(hc->iter) +
                                             ": waiting for epoch " + std::to_string(hc->dbg_epoch) + ", rank " +
                                             std::to_string(hc->dbg_rank) + " at " + std::to_string(hc->dbg_flag) +
                                             "; stall " + std::to_string(hc->part_stall) + " over " +
                                             std::to_string(hc->part_over) + ")");
            if (hc->part_over) {  // every rank rolled the iteration back: grow, remap, rerun
                for (u32 i = 0; i < ns; ++i) {
                    LStep& L = P.steps[i];
                    if (hc->need_rows[i] > L.rows_cap) {
                        L.rows_cap = hc->need_rows[i] + hc->need_rows[i] / 2;
                        L.alloc_rows(c);
                    }
                    if (hc->need_splits[i] > L.splits_cap) {
                        L.splits_cap = hc->need_splits[i] + hc->need_splits[i] / 2;
                        L.splits = DevBuf<u64>(c, L.splits_cap);
                    }
                    if (hc->need_temp[i] > L.temp_cap) {
                        L.temp_cap = hc->need_temp[i] + hc->need_temp[i] / 2;
                        L.temp = DevBuf<u64>(c, L.temp_cap);
                    }
                    hc->need_rows[i] = hc->need_splits[i] = hc->need_temp[i] = 0;
                    hc->step_total[i] = hc->step_cand[i] = hc->heavy_n[i] = 0;
                }
                const u64 demand = hc->part_recv;  // rows routed to this rank (counted past the capacity)
                u64 grow = demand > ps.inbox_cap ? 1 : 0;
                host_allreduce(comm, &grow, 1, 1);
                if (grow) peer_map_inbox(comm, ps, demand > ps.inbox_cap ? demand + demand / 2 : ps.inbox_cap);
                hc->overflow = hc->part_over = hc->part_inbox_over = 0;
                hc->part_recv = 0;
                hc->h[0].J = hc->h[0].N = hc->h[0].D = 0;
                c.h2d(P.ctl.p, hc, sizeof(LoopCtl));
                GD_CUDA(cudaMemsetAsync(&ps.mail->cursor, 0, sizeof(unsigned long long), c.stream));
                c.sync();
                destroy_graph();
                ready();  // every cursor reset and every graph rebuilt before any rank routes again
                continue;
            }
            if (hc->part_stall_any) {
                u64 D = hc->part_last_D;
                if (hc->part_stall) {  // finish this rank's insert under host control
                    const u64 ln = hc->h[0].log_n, recv = hc->part_recv;
                    peer_grow_head(H, ln, ln + recv);
                    grow_hist(hc->iter + 1);
                    hc->step_total[P.final_step] = recv;
                    hc->h[0].J = hc->h[0].N = hc->h[0].D = 0;
                    c.h2d(P.ctl.p, hc, sizeof(LoopCtl));
                    if (recv) loop_insert_keys(c, c.stream, P.ctl.p, P.final_step, 0, ps.inbox, part_bufs(), nullptr);
                    loop_part_advance(c, P.ctl.p, P.final_step, recv, P.hist.p);
                    GD_CUDA(cudaMemsetAsync(&ps.mail->cursor, 0, sizeof(unsigned long long), c.stream));
                    c.d2h(hc, P.ctl.p, sizeof(LoopCtl));
                    c.sync();
                    gd_iter_record rec;
                    c.d2h(&rec, P.hist.p + (hc->iter - 1), sizeof(rec));
                    c.sync();
                    D = rec.delta_out;
                    hc->part_last_D = D;
                }
                // a rank whose graph recorded the iteration keeps its buffers;
                // the next graph run needs this rank's new capacities
                grow_hist(hc->iter + 1);
                hc->part_stall = hc->part_stall_any = 0;
                hc->h[0].J = hc->h[0].N = hc->h[0].D = 0;
                for (u32 i = 0; i < ns; ++i) hc->step_total[i] = hc->step_cand[i] = hc->heavy_n[i] = 0;
                c.h2d(P.ctl.p, hc, sizeof(LoopCtl));
                host_allreduce(comm, &D, 1, 0);
                c.sync();
                destroy_graph();
                if (D == 0) break;
                if (hc->iter >= iter_limit) break;
                ready();
                continue;
            }
            if (hc->done || hc->iter >= iter_limit) break;
            if (eager) continue;
            // a graph that stopped without a reason: cannot happen
            throw_logic("partitioned loop: graph stopped without termination, overflow or stall");
        }
        {  // no rank frees its mailbox / inboxes while a peer may still write them
            u64 bar = 0;
            host_allreduce(comm, &bar, 1, 0);
        }
        const u64 it = hc->iter - hist0;
        E.join_tuples += hc->part_join;
        std::vector<gd_iter_record> recs(it);
        if (it) c.d2h(recs.data(), P.hist.p + hist0, it * sizeof(gd_iter_record));
        c.sync();
        for (const auto& rec : recs) {
            ++E.iterations;
            E.info_[r].history.push_back(rec.delta_in);
            E.info_[r].log.push_back(rec);
        }
        hc->done = 0;
        return it;
    }

    // The canonical local shard: sort the log once (like iterate_loop).
    void part_loop_finish() {
        if (!pl) return;
        PartLoop& P = *pl;
        LHead& H = P.heads[0];
        auto& st = rels[H.rel];
        H.tab.release();
        const u64 f = P.hc->h[0].log_n;
        const u32 ar = E.info_[H.rel].arity;
        DevBuf<u64> scratch(c, std::max<u64>(f, 1));
        u64* sorted = radix_sort<u64>(c, H.log.p, scratch.p, f, ar * bits);
        DevBuf<u64>& res = sorted == H.log.p ? H.log : scratch;
        st.full.release();
        st.full.ctx = res.ctx;
        st.full.p = reinterpret_cast<K*>(res.p);
        st.full.cap = res.cap;
        res.p = nullptr;
        res.cap = 0;
        st.full_n = f;
        st.tail.clear();
        st.delta_n = 0;
        st.new_n = 0;
        pl.reset();
    }

private:
    Engine& E;
    Ctx& c;
    u32 bits;
    std::vector<RelDev<K>> rels;
    std::map<u64, std::pair<bool, u64>> consts;  // value -> (present, encoded)
    // partition-mode state
    DevBuf<K> send_buf;
    DevBuf<u32> owners;

    template <typename F>
    static void for_each_constant(const gd_rule_plan& p, F&& f) {
        auto op = [&](const gd_operand& o) { if (o.kind == GD_CONSTANT) f(o.value); };
        for (u32 v = 0; v < p.nvariants; ++v) {
            const gd_variant& var = p.variants[v];
            for (u32 k = 0; k < var.sel_arity; ++k) op(var.sel_proj[k]);
            for (u32 k = 0; k < var.nsel_filters; ++k) { op(var.sel_filters[k].lhs); op(var.sel_filters[k].rhs); }
            for (u32 s = 0; s < var.nsteps; ++s) {
                const gd_join_step& st = var.steps[s];
                for (u32 k = 0; k < st.proj_arity; ++k) op(st.proj[k]);
                for (u32 k = 0; k < st.nfilters; ++k) { op(st.filters[k].lhs); op(st.filters[k].rhs); }
            }
        }
    }

    void encode_const(u64 v) {
        if (consts.count(v)) return;
        u64 enc = 0;
        const bool ok = encode_value(c, E.enc.e, v, &enc);
        consts[v] = {ok, enc};
    }

    static bool reads(const gd_rule_plan& p, u32 rel) {
        const gd_variant& v = p.variants[0];
        if (v.src_rel == rel) return true;
        for (u32 s = 0; s < v.nsteps; ++s)
            if (v.steps[s].inner_rel == rel) return true;
        return false;
    }

    DevOperand dev_op(const gd_operand& o, bool* never) {
        DevOperand d{o.kind, o.column, 0};
        if (o.kind == GD_CONSTANT) {
            auto it = consts.find(o.value);
            if (it == consts.end()) { encode_const(o.value); it = consts.find(o.value); }
            if (!it->second.first) {
                if (never) *never = true;
                else throw_logic("projection constant missing from the encoding");
            }
            d.value = it->second.second;
        }
        return d;
    }

    DevJoin make_desc(u32 jcc, u32 outer_arity, const u32* outer_perm, u32 inner_arity, u32 proj_arity,
                      const gd_operand* proj, u32 nfilters, const gd_filter* filters) {
        DevJoin jd;
        std::memset(&jd, 0, sizeof(jd));
        jd.jcc = jcc;
        jd.proj_arity = proj_arity;
        jd.nfilters = nfilters;
        jd.bits = bits;
        jd.outer_arity = outer_arity;
        jd.outer_identity = is_identity(outer_perm, outer_arity) ? 1 : 0;
        jd.inner_arity = inner_arity;
        for (u32 i = 0; i < outer_arity; ++i) jd.outer_perm[i] = outer_perm[i];
        for (u32 k = 0; k < proj_arity; ++k) jd.proj[k] = dev_op(proj[k], nullptr);
        for (u32 f = 0; f < nfilters; ++f) {
            bool never = false;
            jd.filters[f].lhs = dev_op(filters[f].lhs, &never);
            jd.filters[f].rhs = dev_op(filters[f].rhs, &never);
            jd.filters[f].require_equal = filters[f].require_equal;
            jd.filters[f].never = never ? 1 : 0;
        }
        return jd;
    }

    void check_temp_watermark() const {  // engine.hpp:544-548
        if (E.acct.current(Accountant::kTemp) != 0)
            throw_logic("temporary storage leaked past a rule boundary");
    }

    // refresh_copies, engine.hpp:365-395
    void refresh_copies(u32 r) {
        PhaseTimer t(E, "index");
        auto& st = rels[r];
        if (!st.copies.empty()) compact(st);
        const u32 ar = E.info_[r].arity;
        for (auto& kv : st.copies) {
            CopyState<K>& cp = kv.second;
            Tracked scratch(E.acct, Accountant::kTemp, 2 * rb(st.full_n, ar) + st.full_n * 8, "index");
            const K* data;
            if (cp.identity) {
                cp.n = st.full_n;
                data = st.full.p;
            } else if (cp.built && st.merge_gen == cp.synced_gen + 1 && st.last_merge_was_delta &&
                       cp.n + st.delta_n == st.full_n) {
                // incremental: copy' = copy U sort(perm(Δ))
                const u64 dn = st.delta_n;
                DevBuf<K> a(c, dn), b(c, dn);
                permute_keys<K>(c, st.delta.p, dn, ar, bits, cp.perm.data(), a.p);
                K* sorted = radix_sort<K>(c, a.p, b.p, dn, ar * bits);
                ensure_discard(c, cp.alt, cp.n + dn);
                merge_disjoint<K>(c, cp.rows.p, cp.n, sorted, dn, cp.alt.p);
                cp.rows.swap(cp.alt);
                cp.n += dn;
                data = cp.rows.p;
            } else {
                const u64 n = st.full_n;
                ensure_discard(c, cp.rows, n);
                ensure_discard(c, cp.alt, n);
                permute_keys<K>(c, st.full.p, n, ar, bits, cp.perm.data(), cp.rows.p);
                K* sorted = radix_sort<K>(c, cp.rows.p, cp.alt.p, n, ar * bits);
                if (sorted != cp.rows.p) cp.rows.swap(cp.alt);
                cp.n = n;
                data = cp.rows.p;
            }
            cp.built = true;
            cp.synced_gen = st.merge_gen;
            if (cp.prefix > 0) build_index<K>(c, data, cp.n, ar, bits, cp.prefix, E.cfg.load_factor, cp.index);
            scratch.reset();
            const u64 bytes = rb(cp.n, ar) + (cp.prefix > 0 ? cp.index.logical_slots * 16ull : 0);
            E.acct.charge(Accountant::kContainer, bytes, "index");
            E.acct.release(Accountant::kContainer, cp.bytes);
            cp.bytes = bytes;
        }
        st.dirty = false;
    }

    // execute_chain, engine.hpp:401-484.  The final step's rows are appended
    // to (sink, sink_n); *produced = rows appended.
    void execute_chain(const gd_variant& v, DevBuf<K>& sink, u64& sink_n, u64* produced) {
        auto& src = rels[v.src_rel];
        const u32 ar = E.info_[v.src_rel].arity;
        const bool use_delta = v.src_version == GD_DELTA;
        if (!use_delta) compact(src);
        const K* cur = use_delta ? src.delta.p : src.full.p;
        u64 cur_n = use_delta ? src.delta_n : src.full_n;
        u32 cur_ar = ar;
        u32 cur_perm[kMaxArity];
        for (u32 i = 0; i < kMaxArity; ++i) cur_perm[i] = i < ar ? v.src_perm[i] : i;

        Tracked permuted_charge;
        if (!is_identity(v.src_perm, ar)) {
            // The permutation is folded into the outer view (no re-sort: the
            // outer order only changes the raw join order, never results).
            PhaseTimer t(E, "join");
            Tracked scratch(E.acct, Accountant::kTemp, 2 * rb(cur_n, ar) + cur_n * 8, "join");
            scratch.reset();
            permuted_charge = Tracked(E.acct, Accountant::kTemp, rb(cur_n, ar), "join");
        }
        if (v.nsteps == 0) {
            PhaseTimer t(E, "join");
            DevJoin jd = make_desc(0, cur_ar, cur_perm, 0, v.sel_arity, v.sel_proj, v.nsel_filters, v.sel_filters);
            ensure_keep(c, sink, sink_n + cur_n, sink_n);
            const u64 m = cur_n ? select_project<K>(c, cur, cur_n, jd, sink.p + sink_n) : 0;
            sink_n += m;
            *produced = m;
            return;
        }
        DevBuf<K> chained;
        Tracked chained_charge;
        for (u32 s = 0; s < v.nsteps; ++s) {
            const gd_join_step& st = v.steps[s];
            auto& in = rels[st.inner_rel];
            const u32 iar = E.info_[st.inner_rel].arity;
            CopyState<K>& cp = in.copies.at(CopyKey{std::vector<u32>(st.inner_perm, st.inner_perm + iar),
                                                    st.join_column_count});
            const K* inner = cp.identity ? in.full.p : cp.rows.p;
            const u64 inner_n = cp.identity ? in.full_n : cp.n;
            const DevJoin jd = make_desc(st.join_column_count, cur_ar, cur_perm, iar, st.proj_arity, st.proj,
                                         st.nfilters, st.filters);
            const bool last = s + 1 == v.nsteps;
            u64 total = 0;
            DevBuf<K> cand;  // filtered path: candidates, then survivors
            DevBuf<u64> row_start, row_off;
            {
                PhaseTimer t(E, "join");
                if (cur_n && inner_n) {
                    row_start = DevBuf<u64>(c, cur_n);
                    row_off = DevBuf<u64>(c, cur_n + 1);
                    IndexView<K> iv{};
                    if (st.join_column_count > 0)
                        iv = IndexView<K>{cp.index.slots.p, cp.index.slot_count, inner, inner_n, iar, bits,
                                          st.join_column_count};
                    const u64 ncand = join_probe<K>(c, cur, cur_n, jd, st.join_column_count ? &iv : nullptr,
                                                    inner_n, row_start.p, row_off.p);
                    if (st.nfilters == 0) {
                        total = ncand;
                    } else if (ncand) {
                        DevBuf<K> raw(c, ncand);
                        DevBuf<uint8_t> flags(c, ncand);
                        join_materialize<K>(c, cur, cur_n, inner, jd, row_start.p, row_off.p, ncand, raw.p,
                                            flags.p);
                        cand = DevBuf<K>(c, ncand);
                        total = compact_flagged<K>(c, raw.p, flags.p, ncand, cand.p);
                    }
                }
            }
            Tracked out_charge(E.acct, Accountant::kTemp, total * st.proj_arity * 8ull, "join");
            if constexpr (std::is_same_v<K, u64>) {
                // output-bounded final step (engine.hpp:401-484,
                // PAPER.md:429-478): a final step whose output would not fit runs in
                // row ranges of bounded output, the sink deduplicated between them
                // (hash set, dedup.cu) so it holds about the distinct rows; the
                // logical counts and charges stay the reference's
                const u64 limit = chain_chunk_rows();
                if (last && st.nfilters == 0 && c.cfg.hash_dedup && total > limit && cur_n > 1) {
                    PhaseTimer t(E, "join");
                    chunked_final_step(cur, cur_n, inner, jd, row_start.p, row_off.p, total, limit, sink, sink_n);
                    E.join_tuples += total;
                    *produced = total;
                    break;
                }
            }
            K* dst;
            DevBuf<K> out;
            if (last) {
                ensure_keep(c, sink, sink_n + total, sink_n);
                dst = sink.p + sink_n;
            } else {
                out = DevBuf<K>(c, total);
                dst = out.p;
            }
            if (total) {
                PhaseTimer t(E, "join");
                if (st.nfilters == 0)
                    join_materialize<K>(c, cur, cur_n, inner, jd, row_start.p, row_off.p, total, dst, nullptr);
                else
                    c.d2d(dst, cand.p, total * sizeof(K));
            }
            E.join_tuples += total;
            if (last) {
                sink_n += total;
                *produced = total;
                break;
            }
            chained = std::move(out);
            chained_charge = std::move(out_charge);
            permuted_charge.reset();
            cur = chained.p;
            cur_n = total;
            cur_ar = st.proj_arity;
            for (u32 i = 0; i < kMaxArity; ++i) cur_perm[i] = i;
        }
    }

    // Output rows one chunk of a chained final step may materialize
    // (gd_device_config.chain_chunk_rows; 0: an eighth of the free HBM).
    u64 chain_chunk_rows() const {
        if (c.cfg.chain_chunk_rows) return c.cfg.chain_chunk_rows;
        return std::max<u64>(1ull << 24, c.available_bytes() / 8 / sizeof(u64));
    }

    // The final step of a chain over outer rows [0, n) in row ranges whose
    // output stays near `limit` rows (range ends from offsets sampled at
    // 64 K points; one sampled interval is the smallest range), appended
    // to the sink, which is hash-deduplicated whenever it passes `limit`.
    void chunked_final_step(const u64* outer, u64 n, const u64* inner, const DevJoin& jd, const u64* row_start,
                            const u64* row_off, u64 total, u64 limit, DevBuf<u64>& sink, u64& sink_n) {
        const u64 S = std::min<u64>(n, 1ull << 16);
        const u64 stride = (n + S - 1) / S;
        const u64 m = (n + stride - 1) / stride;  // samples k * stride < n, plus row_off[n]
        std::vector<u64> off(m + 1);
        {
            DevBuf<u64> d(c, m + 1);
            gather_strided(c, row_off, stride, n, m, d.p);
            c.d2h(off.data(), d.p, (m + 1) * sizeof(u64));
            c.sync();
        }
        auto row_of = [&](u64 k) { return std::min(k * stride, n); };
        std::vector<u64> ends;  // sample indices ending each range
        u64 k0 = 0;
        for (u64 k = 1; k <= m; ++k) {
            if (off[k] - off[k0] > limit && k - 1 > k0) {
                ends.push_back(k - 1);
                k0 = k - 1;
            }
        }
        ends.push_back(m);
        u64 max_rows = 0;
        k0 = 0;
        for (u64 k : ends) {
            max_rows = std::max(max_rows, row_of(k) - row_of(k0));
            k0 = k;
        }
        DevBuf<u64> roff(c, max_rows + 1);
        const bool trace = (c.cfg.trace & 1) != 0;
        k0 = 0;
        for (u64 k : ends) {
            const u64 r0 = row_of(k0), r1 = row_of(k), cnt = off[k] - off[k0];
            k0 = k;
            if (!cnt) continue;
            offsets_rebase(c, row_off, r0, r1 - r0 + 1, roff.p);
            ensure_keep(c, sink, sink_n + cnt, sink_n);
            join_materialize<u64>(c, outer + r0, r1 - r0, inner, jd, row_start + r0, roff.p, cnt, sink.p + sink_n,
                                  nullptr);
            sink_n += cnt;
            if (sink_n > limit) compact_sink(sink, sink_n);
            if (trace)
                fprintf(stderr, "[chain] rows [%llu, %llu): %llu outputs, sink %llu rows\n",
                        (unsigned long long)r0, (unsigned long long)r1, (unsigned long long)cnt,
                        (unsigned long long)sink_n);
        }
        (void)total;
    }

    // Sink rows -> their distinct rows (hash set; the set grows until it fits).
    void compact_sink(DevBuf<u64>& sink, u64& sink_n) {
        for (u64 expect = std::max<u64>(sink_n / 4, 1 << 16);; expect *= 2) {
            DevBuf<u64> uniq(c, std::min<u64>(sink_n, 2 * expect + 1));
            const u64 u = hash_dedup(c, sink.p, sink_n, expect, uniq.p, uniq.cap);
            if (u != ~0ull) {
                sink = std::move(uniq);
                sink_n = u;
                return;
            }
            if (expect >= sink_n) return;  // no set fits: keep the rows as they are
        }
    }

    void append_new(u32 r, u64 m) {  // engine.hpp:486-495
        if (m == 0) return;
        const u64 b = rb(m, E.info_[r].arity);
        E.acct.charge(Accountant::kContainer, b, "join");
        E.info_[r].new_bytes += b;
    }

    void assign_delta(u32 r, u64 rows, const char* phase) {  // engine.hpp:511-517
        RelInfo& ri = E.info_[r];
        const u64 b = rb(rows, ri.arity);
        E.acct.charge(Accountant::kContainer, b, phase);
        E.acct.release(Accountant::kContainer, ri.delta_bytes);
        ri.delta_bytes = b;
    }

    // merge_into_full bookkeeping (engine.hpp:520-533 + merge_buffer.hpp).
    void merge_accounting(u32 r, u64 full_before, u64 gained, const char* phase) {
        RelInfo& ri = E.info_[r];
        E.bufs.acquire(ri.name, full_before, gained, ri.arity);
        E.bufs.release(ri.name);
        const u64 b = rb(full_before + gained, ri.arity);
        E.acct.charge(Accountant::kContainer, b, phase);
        E.acct.release(Accountant::kContainer, ri.full_bytes);
        ri.full_bytes = b;
    }

    // Sorts rows [0, m) of `buf` (scratch `tmp`), returns the sorted pointer.
    K* sort_rows(DevBuf<K>& buf, u64 m, u32 ar) {
        DevBuf<K> tmp(c, m);
        K* s = radix_sort<K>(c, buf.p, tmp.p, m, ar * bits);
        if (s != buf.p) {
            buf.swap(tmp);  // keep the sorted data in buf; old buf freed with tmp
            return buf.p;
        }
        return s;
    }

    void seed_rule(const gd_rule_plan& plan) {  // engine.hpp:141-168
        const gd_variant& v = plan.variants[0];
        for (u32 s = 0; s < v.nsteps; ++s)  // refresh_inputs, engine.hpp:355-360
            if (rels[v.steps[s].inner_rel].dirty) refresh_copies(v.steps[s].inner_rel);
        const u32 h = plan.head_rel;
        const u32 ar = E.info_[h].arity;
        DevBuf<K> rows;
        u64 m = 0, produced = 0;
        execute_chain(v, rows, m, &produced);
        // charges follow the logical rows (a chunked final step leaves them deduplicated)
        const u64 mlog = std::max<u64>(m, produced);
        Tracked rows_charge(E.acct, Accountant::kTemp, rb(mlog, ar), "join");
        if (m == 0) return;
        auto& head = rels[h];
        K* sorted;
        {
            PhaseTimer t(E, "dedup");
            sorted = sort_rows(rows, m, ar);
        }
        MergeResult mr;
        DevBuf<K> gained(c, m);
        {
            PhaseTimer t(E, "difference");
            mr = difference_full(head, sorted, m, gained.p);
        }
        {
            Tracked scratch(E.acct, Accountant::kTemp, mlog * 8 + rb(mlog, ar), "dedup");
        }
        Tracked fresh_charge(E.acct, Accountant::kTemp, rb(mr.unique_new, ar), "dedup");
        rows_charge.reset();
        if (mr.delta_n == 0) return;
        Tracked gained_charge(E.acct, Accountant::kTemp, rb(mr.delta_n, ar), "difference");
        fresh_charge.reset();
        {
            PhaseTimer t(E, "merge");
            merge_accounting(h, total_n(head), mr.delta_n, "merge");
            add_to_full(head, gained.p, mr.delta_n);
        }
        ++head.merge_gen;
        head.last_merge_was_delta = false;
        head.dirty = true;
    }

    // Steps (3)-(5) of one iteration for relation r (engine.hpp:228-251).
    void dedup_diff_merge(u32 r, gd_iter_record& log) {
        auto& st = rels[r];
        RelInfo& ri = E.info_[r];
        const u32 ar = ri.arity;
        const u64 m = st.new_n;
        // the reference's charges follow the logical join rows (a chunked final
        // step leaves fewer, deduplicated rows in new_acc)
        const u64 mlog = std::max<u64>(m, (u64)log.join);
        MergeResult mr;
        if (m > 0) {
            K* sorted;
            u64 ms = m;  // rows that reach the sort
            {
                PhaseTimer t(E, "dedup");
                bool done = false;
                if constexpr (std::is_same_v<K, u64>) {
                    // mostly-duplicate join output: hash pre-dedup, then sort
                    // only the distinct rows (dedup.cu); the set is sized from
                    // the previous iteration's distinct count
                    const u64 expect = std::max<u64>(2 * st.last_unique + 4096, m / 64);
                    if (c.cfg.hash_dedup && m >= c.cfg.hash_dedup_min_rows && 4 * expect < m) {
                        DevBuf<u64> uniq(c, std::min<u64>(m, 2 * expect + 1));
                        const u64 u = hash_dedup(c, reinterpret_cast<const u64*>(st.new_acc.p), m, expect, uniq.p,
                                                 uniq.cap);
                        if (u != ~0ull) {
                            DevBuf<K> tmp(c, std::max<u64>(u, 1));
                            sorted = reinterpret_cast<K*>(radix_sort<u64>(c, uniq.p, reinterpret_cast<u64*>(tmp.p), u,
                                                                          ar * bits));
                            // keep the sorted rows alive in new_acc
                            if (u) c.d2d(st.new_acc.p, sorted, u * sizeof(K));
                            sorted = st.new_acc.p;
                            ms = u;
                            done = true;
                        }
                    }
                }
                if (!done) sorted = sort_rows(st.new_acc, m, ar);
            }
            PhaseTimer t(E, "difference");
            ensure_discard(c, st.delta_alt, ms);
            mr = difference_full(st, sorted, ms, st.delta_alt.p);
            st.last_unique = mr.unique_new;
            Tracked scratch(E.acct, Accountant::kTemp, mlog * 8 + rb(mlog, ar), "dedup");
        }
        Tracked fresh_charge(E.acct, Accountant::kTemp, rb(mr.unique_new, ar), "dedup");
        // clear_new, engine.hpp:497-501
        E.acct.release(Accountant::kContainer, ri.new_bytes);
        ri.new_bytes = 0;
        st.new_n = 0;
        fresh_charge.reset();
        assign_delta(r, mr.delta_n, "difference");
        st.delta.swap(st.delta_alt);
        st.delta_n = mr.delta_n;
        if (mr.delta_n > 0) {
            PhaseTimer t(E, "merge");
            merge_accounting(r, total_n(st), mr.delta_n, "merge");
            add_to_full(st, st.delta.p, mr.delta_n);
            ++st.merge_gen;
            st.last_merge_was_delta = true;
            st.dirty = true;
        }
        log.new_unique = mr.unique_new;
        log.delta_out = mr.delta_n;
        log.full_after = total_n(st);
    }
};

// ---- partition mode -------------------------------------------------
// begin: run every recursive variant on the local Δ into new_acc, sort it
// with the owner rank as the most significant digit (so the send buffer
// is grouped by destination, each group sorted), drop local duplicates.
template <typename K>
void Impl<K>::partition_begin(u64* send_counts, const void** d_send) {
    u32 rec_rel = UINT32_MAX;
    for (const auto& p : E.plans_)
        if (p.recursive) rec_rel = p.head_rel;
    if constexpr (std::is_same_v<K, u64>) {
        if (pl || part_loop_eligible(rec_rel)) {
            if (!pl) part_loop_setup(rec_rel);
            part_loop_begin(send_counts, d_send);
            return;
        }
    }
    auto& head = rels[rec_rel];
    const u32 ar = E.info_[rec_rel].arity;
    for (u32 r = 0; r < rels.size(); ++r)
        if (rels[r].dirty && !rels[r].copies.empty()) refresh_copies(r);
    for (const auto& p : E.plans_) {
        if (!p.recursive) continue;
        for (u32 v = 0; v < p.nvariants; ++v) {
            const gd_variant& var = p.variants[v];
            if (rels[var.src_rel].delta_n == 0) continue;
            u64 m = 0;
            execute_chain(var, head.new_acc, head.new_n, &m);
        }
    }
    const u64 m = head.new_n;
    for (u32 k = 0; k < E.nranks; ++k) send_counts[k] = 0;
    if (m == 0) {
        *d_send = nullptr;
        return;
    }
    PhaseTimer t(E, "dedup");
    K* sorted = sort_rows(head.new_acc, m, ar);
    ensure_discard(c, send_buf, m);
    const u64 u = unique_sorted<K>(c, sorted, m, send_buf.p);
    // group by owner: stable counting split on the owner (keys stay sorted
    // inside each destination group)
    ensure_discard(c, owners, u);
    owner_of<K>(c, send_buf.p, u, E.nranks, owners.p);
    std::vector<unsigned long long> cnt(E.nranks, 0);
    {
        // one stable partition pass per destination via flag compaction
        DevBuf<K> grouped(c, u);
        DevBuf<uint8_t> flags(c, u);
        u64 off = 0;
        for (u32 k = 0; k < E.nranks; ++k) {
            owner_flags(c, owners.p, u, k, flags.p);
            const u64 got = compact_flagged<K>(c, send_buf.p, flags.p, u, grouped.p + off);
            cnt[k] = got;
            off += got;
        }
        send_buf.swap(grouped);
    }
    head.new_n = 0;
    for (u32 k = 0; k < E.nranks; ++k) send_counts[k] = cnt[k];
    *d_send = send_buf.p;
}

template <typename K>
u64 Impl<K>::partition_run(Comm& comm, u64 max_iters) {
    if constexpr (std::is_same_v<K, u64>) {
        u32 rec_rel = UINT32_MAX;
        for (const auto& p : E.plans_)
            if (p.recursive) rec_rel = p.head_rel;
        if (pl || part_loop_eligible(rec_rel)) {
            if (!pl) part_loop_setup(rec_rel);
            // peer-memory exchange inside the graph loop unless the NCCL
            // send/recv driver (one host round trip per iteration) is asked for
            if (c.cfg.partition_exchange == GD_EXCHANGE_PEER) return part_peer_run(comm, max_iters);
            return part_loop_run(comm, max_iters);
        }
    }
    throw_unsupported("gd_engine_run_partitioned: the native driver runs the loop-kernel partition path "
                      "(one recursive relation, 64-bit keys); drive other programs with partition_begin/end");
}

template <typename K>
void Impl<K>::partition_end(const void* d_recv, u64 recv_rows, u64* local_delta) {
    if constexpr (std::is_same_v<K, u64>) {
        if (pl) {
            part_loop_end(d_recv, recv_rows, local_delta);
            return;
        }
    }
    u32 rec_rel = UINT32_MAX;
    for (const auto& p : E.plans_)
        if (p.recursive) rec_rel = p.head_rel;
    auto& st = rels[rec_rel];
    const u32 ar = E.info_[rec_rel].arity;
    ++E.iterations;
    E.info_[rec_rel].history.push_back(st.delta_n);
    gd_iter_record log{st.delta_n, recv_rows, 0, 0, 0};
    MergeResult mr;
    if (recv_rows) {
        DevBuf<K> buf(c, recv_rows);
        c.d2d(buf.p, d_recv, recv_rows * sizeof(K));
        K* sorted;
        {
            PhaseTimer t(E, "dedup");
            sorted = sort_rows(buf, recv_rows, ar);
        }
        PhaseTimer t(E, "difference");
        ensure_discard(c, st.delta_alt, recv_rows);
        mr = difference_full(st, sorted, recv_rows, st.delta_alt.p);
    }
    st.delta.swap(st.delta_alt);
    st.delta_n = mr.delta_n;
    if (mr.delta_n) {
        PhaseTimer t(E, "merge");
        add_to_full(st, st.delta.p, mr.delta_n);
    }
    log.new_unique = mr.unique_new;
    log.delta_out = mr.delta_n;
    log.full_after = total_n(st);
    E.info_[rec_rel].log.push_back(log);
    *local_delta = mr.delta_n;
}

}  // namespace

// ---- shared helpers used above ---------------------------------------

u64 canonicalize_rows(Ctx& c, const u64* d_rows, u64 n, u32 arity, DevBuf<u64>& out) {
    out.reserve_discard(c, std::max<u64>(n * arity, 1));
    if (n == 0) return 0;
    EncodingOwner eo;
    choose_encoding(c, {{d_rows, n * arity}}, {}, arity, eo);
    auto run = [&](auto tag) -> u64 {
        using K = decltype(tag);
        DevBuf<K> a(c, n), b(c, n);
        pack_rows<K>(c, d_rows, n, arity, eo.e, a.p);
        K* s = radix_sort<K>(c, a.p, b.p, n, arity * eo.e.bits);
        K* u = s == a.p ? b.p : a.p;
        const u64 m = unique_sorted<K>(c, s, n, u);
        unpack_rows<K>(c, u, m, arity, eo.e, out.p);
        return m;
    };
    return eo.e.key_words == 1 ? run(u64{}) : run(u128{});
}

// ---- Engine ----------------------------------------------------------

Engine::Engine(Ctx& ctx, const gd_engine_config& cf, u32 nrels, const u32* arities, const u32* is_edb,
               const char* const* names)
    : c(ctx), cfg(cf), acct(cf.memory_budget_bytes), bufs(acct, cf.ebm_enabled != 0, cf.alpha) {
    if (!(cfg.load_factor > 0.0) || cfg.load_factor >= 1.0)
        throw_config("engine: load factor must be in (0, 1)");
    info_.resize(nrels);
    raw.resize(nrels);
    raw_n.assign(nrels, 0);
    for (u32 r = 0; r < nrels; ++r) {
        if (arities[r] == 0 || arities[r] > kMaxArity)
            throw_unsupported("relation arity must be in [1, " + std::to_string(kMaxArity) + "]");
        info_[r].arity = arities[r];
        info_[r].is_edb = is_edb[r] != 0;
        info_[r].name = names && names[r] ? std::string(names[r]) : "r" + std::to_string(r);
    }
}

Engine::~Engine() = default;

void Engine::set_plans(const gd_rule_plan* plans, u32 n) {  // engine.hpp:97-101, 300-310
    if (seeded || impl) throw_logic("override_plans: engine already seeded");
    for (u32 i = 0; i < n; ++i) {
        const gd_rule_plan& p = plans[i];
        check_rel(p.head_rel);
        if (p.nvariants == 0 || p.nvariants > GD_MAX_VARIANTS) throw_plan_error("rule plan has no/too many variants");
        for (u32 v = 0; v < p.nvariants; ++v) {
            const gd_variant& var = p.variants[v];
            check_rel(var.src_rel);
            if (var.nsteps > GD_MAX_STEPS) throw_unsupported("too many join steps");
            u32 out_ar = var.nsteps ? var.steps[var.nsteps - 1].proj_arity : var.sel_arity;
            if (out_ar != info_[p.head_rel].arity) throw_logic("append_new: arity mismatch");
            for (u32 s = 0; s < var.nsteps; ++s) {
                const gd_join_step& st = var.steps[s];
                check_rel(st.inner_rel);
                if (st.proj_arity == 0 || st.proj_arity > kMaxArity)
                    throw_config("join: projection must produce at least one column");
            }
        }
    }
    plans_.assign(plans, plans + n);
}

void Engine::load_edb(u32 r, const u64* rows, u64 n, bool canonical, bool device) {  // engine.hpp:107-128
    if (seeded || impl) throw_logic("load_edb: engine already running");
    if (r >= info_.size() || !info_[r].is_edb)
        throw_load("load_edb: '" + (r < info_.size() ? info_[r].name : std::to_string(r)) +
                   "' is not a declared EDB relation");
    const u32 ar = info_[r].arity;
    DevBuf<u64> up(c, std::max<u64>(n * ar, 1));
    if (device) {
        c.d2d(up.p, rows, n * ar * sizeof(u64));
        if (n && max_value(c, up.p, n * ar) == kEmptySlot)
            throw_load("load_edb: '" + info_[r].name + "' contains the reserved sentinel value");
    } else {
        c.h2d(up.p, rows, n * ar * sizeof(u64));
        // sentinel check on the device (one pass over the uploaded rows)
        if (n && max_value(c, up.p, n * ar) == kEmptySlot)
            throw_load("load_edb: '" + info_[r].name + "' contains the reserved sentinel value");
    }
    u64 m = n;
    if (canonical) {
        raw[r] = std::move(up);
    } else {
        PhaseTimer t(*this, "other");
        Tracked scratch(acct, Accountant::kTemp, n * 8 + rb(n, ar), "other");
        m = canonicalize_rows(c, up.p, n, ar, raw[r]);
    }
    raw_n[r] = m;
    // assign_full, engine.hpp:503-509
    const u64 b = rb(m, ar);
    acct.charge(Accountant::kContainer, b, "other");
    acct.release(Accountant::kContainer, info_[r].full_bytes);
    info_[r].full_bytes = b;
}

void Engine::seed() {  // engine.hpp:137-179
    if (seeded) throw_logic("seed: called twice");
    const auto t0 = std::chrono::steady_clock::now();
    if (!impl) {
        // Encoding over every EDB value and every rule constant.
        std::vector<std::pair<const u64*, u64>> arrays;
        u32 max_ar = 1;
        for (u32 r = 0; r < info_.size(); ++r) {
            max_ar = std::max(max_ar, info_[r].arity);
            if (info_[r].is_edb && raw_n[r]) arrays.push_back({raw[r].p, raw_n[r] * info_[r].arity});
        }
        std::vector<u64> constants;
        for (const auto& p : plans_)
            for (u32 v = 0; v < p.nvariants; ++v) {
                const gd_variant& var = p.variants[v];
                auto op = [&](const gd_operand& o) { if (o.kind == GD_CONSTANT) constants.push_back(o.value); };
                for (u32 k = 0; k < var.sel_arity; ++k) op(var.sel_proj[k]);
                for (u32 k = 0; k < var.nsel_filters; ++k) { op(var.sel_filters[k].lhs); op(var.sel_filters[k].rhs); }
                for (u32 s = 0; s < var.nsteps; ++s) {
                    const gd_join_step& st = var.steps[s];
                    max_ar = std::max(max_ar, st.proj_arity);
                    for (u32 k = 0; k < st.proj_arity; ++k) op(st.proj[k]);
                    for (u32 k = 0; k < st.nfilters; ++k) { op(st.filters[k].lhs); op(st.filters[k].rhs); }
                }
            }
        choose_encoding(c, arrays, constants, max_ar, enc);
        if (enc.e.key_words == 1) impl.reset(new Impl<u64>(*this));
        else impl.reset(new Impl<u128>(*this));
    }
    impl->seed();
    seeded = true;
    total_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void Engine::iterate() {  // engine.hpp:181-257
    if (!seeded) seed();
    const auto t0 = std::chrono::steady_clock::now();
    impl->iterate();
    if (c.cfg.trace & 4) fprintf(stderr, "[segsort] iterate returns (pending %d)\n", (int)impl->output_pending());
    if (!impl->output_pending()) c.sync();
    total_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

u64 Engine::relation_count(u32 r) {
    check_rel(r);
    if (!impl) return info_[r].is_edb ? raw_n[r] : 0;
    return impl->count(r);
}

void Engine::relation_download(u32 r, u64* out, u64 capacity_rows, bool device) {
    check_rel(r);
    const u64 n = relation_count(r);
    if (n > capacity_rows) throw_logic("relation download: buffer too small");
    if (!impl) {
        if (n == 0) return;
        if (device) c.d2d(out, raw[r].p, n * info_[r].arity * sizeof(u64));
        else c.d2h(out, raw[r].p, n * info_[r].arity * sizeof(u64));
        c.sync();
        return;
    }
    impl->download(r, out, device);
}

u64 Engine::relation_digest(u32 r) {
    check_rel(r);
    if (!impl) throw_logic("relation_digest: engine not seeded");
    return impl->digest(r);
}

void Engine::fill_stats(gd_run_stats* out) const {  // engine.hpp:270-277, stats.hpp:21-46
    std::memset(out, 0, sizeof(*out));
    static const char* kPhases[6] = {"index", "join", "dedup", "difference", "merge", "other"};
    double categorized = 0;
    for (int p = 0; p < 5; ++p) {
        auto it = phase_seconds_.find(kPhases[p]);
        out->phase_seconds[p] = it == phase_seconds_.end() ? 0.0 : it->second;
        categorized += out->phase_seconds[p];
    }
    out->phase_seconds[5] = std::max(0.0, total_seconds - categorized);
    out->total_seconds = total_seconds;
    out->iterations = iterations;
    out->buffer_allocations = bufs.allocations();
    out->charge_events = acct.events();
    out->peak_tracked_bytes = acct.peak();
    out->peak_temp_bytes = acct.peak_temp();
    out->join_tuples = join_tuples;
    out->device_bytes_peak = c.bytes_peak;
    for (int p = 0; p < 6; ++p) {
        out->kernel_seconds[p] = kernel_seconds[p];
        out->algo_bytes[p] = algo_bytes[p];
    }
}

void Engine::encoding(u32* bits, u32* key_words, u32* dict) const {
    *bits = enc.e.bits;
    *key_words = enc.e.key_words;
    *dict = enc.e.dict ? 1 : 0;
}

void Engine::set_partition(u32 rk, u32 nr) {
    if (seeded) throw_logic("set_partition: engine already seeded");
    if (nr == 0 || rk >= nr) throw_config("set_partition: rank must be < nranks");
    u32 nrec = 0;
    std::set<u32> heads;
    for (const auto& p : plans_) {
        if (!p.recursive) continue;
        heads.insert(p.head_rel);
        for (u32 v = 0; v < p.nvariants; ++v)
            for (u32 s = 0; s < p.variants[v].nsteps; ++s)
                if (!info_[p.variants[v].steps[s].inner_rel].is_edb)
                    throw_unsupported("partitioned mode needs EDB-only inner relations (SURVEY §8e); "
                                      "run IDB-inner programs as replicas");
    }
    nrec = (u32)heads.size();
    if (nrec != 1) throw_unsupported("partitioned mode supports exactly one recursive relation");
    rank = rk;
    nranks = nr;
}

u32 Engine::exchange_words() const { return enc.e.key_words; }

void Engine::partition_begin(u64* send_counts, const void** d_send) {
    if (!seeded) throw_logic("partition_begin: seed first");
    impl->partition_begin(send_counts, d_send);
}
void Engine::partition_end(const void* d_recv, u64 recv_rows, u64* local_delta) {
    impl->partition_end(d_recv, recv_rows, local_delta);
}
void Engine::partition_finish() { impl->partition_finish(); }
u64 Engine::partition_run(Comm& comm, u64 max_iters) {
    if (!seeded) throw_logic("gd_engine_run_partitioned: seed first");
    if (nranks == 0) throw_usage("gd_engine_run_partitioned: set_partition first");
    return impl->partition_run(comm, max_iters);
}

}  // namespace gd
