// loop.cu — kernels of the resident fixpoint loop (loop.h): one iteration of
// engine::iterate_to_fixpoint (engine.hpp:181-257) for loop heads as a fixed
// kernel sequence whose sizes live in device memory (LoopCtl), so the
// sequence can be captured once into a CUDA graph and repeated on the
// device.
//
// Per variant-step:  loop_probe   one HISA probe per outer row (join_count,
//                                 ra.hpp:141-182) + per-CTA count sums;
//                    loop_scan    exclusive scan of the counts (the
//                                 sequential prefix sum of join_materialize,
//                                 ra.hpp:235-238), CTA prefixes from the sums;
//                    loop_materialize_temp  intermediate chain steps
//                                 (execute_chain temps, engine.hpp:401-484).
// Then loop_gate (capacity check of every insertion before any side effect),
// loop_materialize_insert — the final step's load-balanced expansion fused
// with canonicalize's dedup, difference and the append of Δ
// (tuple_array.hpp:73-133, ra.hpp:386-422): every join row probes the
// head's full-tuple hash index once — and loop_end (records the iteration,
// advances Δ, detects the fixpoint, sets the graph's while condition).
//
// Grids are fixed at capture (multiples of the SM count); every kernel
// reads its sizes from LoopCtl and returns at once when the loop is done or
// an overflow rolled the iteration back.
#include "index.cuh"
#include "join.cuh"
#include "loop.h"

namespace gd {

namespace {

constexpr int kLT = 256;              // threads per CTA
constexpr int kLItems = 4;            // probe rows per thread per tile
constexpr u64 kLTile = (u64)kLT * kLItems;
constexpr u64 kHashSeed = 0x9e3779b97f4a7c15ull;
constexpr int kScan = 4;  // slots read per collision step (one 32-byte sector when aligned)

__device__ __forceinline__ bool loop_stopped(const LoopCtl* ctl) {
    return (ctl->overflow | ctl->done) != 0;
}

__device__ __forceinline__ void resolve(const LoopOuter& o, const LoopCtl* ctl, const u64*& p, u64& n) {
    switch (o.kind) {
        case LO_DELTA:
            p = o.ptr + ctl->h[o.head].dlo;
            n = ctl->h[o.head].dhi - ctl->h[o.head].dlo;
            break;
        case LO_FULL:
            p = o.ptr;
            n = ctl->h[o.head].dhi;
            break;
        case LO_TEMP:
            p = o.ptr;
            n = ctl->step_total[o.src_step];
            break;
        default:
            p = o.ptr;
            n = o.n;
    }
}

// Home slot of a key; homes are monotone in the hash (the zone growth pass
// relies on it).  (4-slot aligned buckets read whole were measured slower on
// C2: 118 ms with 2-slot and 129 ms with 4-slot first reads vs 104 ms for
// exact homes — keys crowd the bucket starts and the wider reads spill.)
__device__ __forceinline__ u64 hs_home(u64 key, u64 cap) { return __umul64hi(fmix64(key ^ kHashSeed), cap); }

// Rare paths of a packed-slot insertion, out of line (register pressure of
// the batched fast path): the key was seen in an earlier iteration (stamp
// update), or its home slot holds another key (linear probing, kScan slots
// read per round trip).  p = the slot reached, o = its current value (a
// CAS's return or the bucket read: another key, or this key with an older
// stamp).  Returns bit 0 = new key, bit 1 = first occurrence this iteration.
__device__ __noinline__ u32 insert_slow_packed(u64* __restrict__ tab, u64 cap, u32 sb, u64 st, u64 key, u64 p,
                                               u64 o) {
    const u64 smask = (1ull << sb) - 1;
    const u64 want = key << sb | st;
    while (true) {
        if (o == kEmptySlot) return 3;
        if ((o >> sb) == key) {
            while ((o & smask) != st) {  // seen before, not yet this iteration
                const u64 o2 = atomicCAS(&tab[p], o, want);
                if (o2 == o) return 2;
                o = o2;
            }
            return 0;
        }
        // collision: read the next kScan slots together (one round trip,
        // mostly one sector) and CAS only the first candidate
        u64 w[kScan];
#pragma unroll
        for (int q = 0; q < kScan; ++q) {
            u64 pq = p + 1 + q;
            pq = pq >= cap ? pq - cap : pq;
            w[q] = __ldcg(&tab[pq]);
        }
        int hit = kScan;
        u64 wv = w[kScan - 1];
#pragma unroll
        for (int q = kScan - 1; q >= 0; --q)
            if (w[q] == kEmptySlot || (w[q] >> sb) == key) {
                hit = q;
                wv = w[q];
            }
        p = p + 1 + (hit == kScan ? kScan - 1 : hit);
        p = p >= cap ? p - cap : p;
        o = (hit < kScan && wv == kEmptySlot) ? atomicCAS(&tab[p], kEmptySlot, want) : wv;
    }
}

// The same from the home slot (the caller's home-slot read or CAS returned o).
__device__ __noinline__ u32 insert_slow_home(u64* __restrict__ tab, u64 cap, u32 sb, u64 st, u64 key, u64 o) {
    return insert_slow_packed(tab, cap, sb, st, key, hs_home(key, cap), o);
}

__device__ __noinline__ u32 insert_slow_wide(HSlot* __restrict__ tab, u64 cap, u32 st, u64 key, u64 o) {
    u64 p = hs_home(key, cap);
    while (o != kEmptySlot && o != key) {
        p = p + 1 == cap ? 0 : p + 1;
        o = atomicCAS(&tab[p].key, kEmptySlot, key);
    }
    const u32 fresh = o == kEmptySlot;
    const u32 first = __ldcg(&tab[p].stamp) != st && atomicExch(&tab[p].stamp, st) != st;
    return fresh | first << 1;
}

// Membership + insertion of PER keys in the head's full-tuple index: the
// home-slot CAS of every key is issued together (independent L2 round trips
// in flight); a CAS that finds an empty slot (new key) or this key already
// stamped with this iteration settles it; anything else takes the slow path.
// fresh: bit k = key k is new (appended by the caller); first: bit k = first
// occurrence of key k in this iteration (stamp st) — the distinct count of
// the join output.
template <int PER, int NSLOT = 1>
__device__ __forceinline__ void hs_insert(const LoopHeadBufs& hb, u32 st, const u64 (&key)[PER], u32 ok,
                                          u32& fresh, u32& first) {
    static_assert(NSLOT == 0 || NSLOT == 1 || NSLOT == 2, "insert mode 0 (CAS first), 1 (load first), 2 (batched)");
    fresh = first = 0;
    u64 old[PER];
    if constexpr (NSLOT <= 1) {
      if (hb.sbits) {
        u64* tab = static_cast<u64*>(hb.tab);
        const u32 sb = hb.sbits;
        // NSLOT = 1 (default): load the home slots first, then CAS only the
        // empty ones — the CAS hits the line the load brought into L2.
        // NSLOT = 0: CAS first (one round trip, the CAS misses to DRAM).
        u64 home[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            home[k] = hs_home(key[k], hb.tab_cap);
            if (NSLOT) old[k] = (ok >> k & 1) ? __ldcg(&tab[home[k]]) : 0ull;
            else old[k] = (ok >> k & 1) ? atomicCAS(&tab[home[k]], kEmptySlot, key[k] << sb | st) : 0ull;
        }
        if (NSLOT) {
#pragma unroll
            for (int k = 0; k < PER; ++k)
                if ((ok >> k & 1) && old[k] == kEmptySlot)
                    old[k] = atomicCAS(&tab[home[k]], kEmptySlot, key[k] << sb | st);
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            if (!(ok >> k & 1)) continue;
            u32 r;
            if (old[k] == kEmptySlot) r = 3;
            else if (old[k] == (key[k] << sb | st)) r = 0;
            else r = insert_slow_home(tab, hb.tab_cap, sb, st, key[k], old[k]);
            fresh |= (r & 1u) << k;
            first |= (r >> 1) << k;
        }
        return;
      }
    } else if (hb.sbits) {
        // NSLOT = 2: load-first with BATCHED probing.  Every unresolved key
        // of the thread advances one step per pass — a claiming CAS on an
        // empty slot, a stamp CAS on its own slot, or the load of the next
        // slot after another key — and a pass issues all of them before
        // consuming any, so a thread (and its warp) pays the longest probe
        // chain among its keys instead of the sum of its collisions.
        u64* tab = static_cast<u64*>(hb.tab);
        const u32 sb = hb.sbits;
        const u64 smask = (1ull << sb) - 1;
        u64 pos[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            pos[k] = hs_home(key[k], hb.tab_cap);
            old[k] = (ok >> k & 1) ? __ldcg(&tab[pos[k]]) : 0ull;
        }
        u32 pend = ok;
        while (pend) {
            u32 cas = 0;
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                if (!(pend >> k & 1)) continue;
                if (old[k] == kEmptySlot) {
                    cas |= 1u << k;
                } else if ((old[k] >> sb) == key[k]) {
                    if ((old[k] & smask) == st) pend &= ~(1u << k);  // seen this iteration already
                    else cas |= 1u << k;                               // stamp update
                } else {  // another key: the next slot
                    pos[k] = pos[k] + 1 == hb.tab_cap ? 0 : pos[k] + 1;
                    old[k] = __ldcg(&tab[pos[k]]);
                }
            }
            u64 res[PER];
#pragma unroll
            for (int k = 0; k < PER; ++k)
                if (cas >> k & 1) res[k] = atomicCAS(&tab[pos[k]], old[k], key[k] << sb | st);
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                if (!(cas >> k & 1)) continue;
                if (res[k] == old[k]) {  // claimed: a new key (was empty) or this iteration's first sight
                    fresh |= (u32)(old[k] == kEmptySlot) << k;
                    first |= 1u << k;
                    pend &= ~(1u << k);
                } else {
                    old[k] = res[k];  // lost a race: look at what is there now
                }
            }
        }
        return;
    }
    {  // wide slots
        HSlot* tab = static_cast<HSlot*>(hb.tab);
#pragma unroll
        for (int k = 0; k < PER; ++k)
            old[k] = (ok >> k & 1) ? atomicCAS(&tab[hs_home(key[k], hb.tab_cap)].key, kEmptySlot, key[k]) : 0ull;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            if (!(ok >> k & 1)) continue;
            const u32 r = insert_slow_wide(tab, hb.tab_cap, st, key[k], old[k]);
            fresh |= (r & 1u) << k;
            first |= (r >> 1) << k;
        }
    }
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
    v = warp_sum(v);
    if (lane_id() == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    T t = 0;
#pragma unroll
    for (int w = 0; w < kLT / 32; ++w) t += red[w];
    __syncthreads();
    return t;
}

// Uniform per-CTA view of the stop flags (another CTA may raise overflow
// while this one starts).
__device__ __forceinline__ bool cta_stopped(const LoopCtl* ctl, u32* s) {
    if (threadIdx.x == 0) {
        const volatile LoopCtl* v = ctl;
        *s = (v->overflow | v->done) != 0;
    }
    __syncthreads();
    return *s != 0;
}

// True in every thread of the grid's last CTA to get here; that CTA sees
// every other CTA's writes (fence before the count).
__device__ __forceinline__ bool last_cta(LoopCtl* ctl, u32* s) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const u32 t = atomicAdd(&ctl->ctas_done, 1u);
        *s = t == gridDim.x - 1;
        if (*s) {
            ctl->ctas_done = 0;
            __threadfence();
        }
    }
    __syncthreads();
    return *s != 0;
}

// Each CTA of a fixed grid owns a contiguous chunk of outer rows (a whole
// number of tiles), so per-CTA sums + the scan give row offsets without
// look-back or workspace resets.
__device__ __forceinline__ void chunk_of(u64 n, u64& begin, u64& end) {
    const u64 tiles = (n + kLTile - 1) / kLTile;
    const u64 per = (tiles + gridDim.x - 1) / gridDim.x;
    begin = min(n, (u64)blockIdx.x * per * kLTile);
    end = min(n, begin + per * kLTile);
}

// ---- gate / end bodies (one thread) --------------------------------------

// One thread; every control-block load is issued up front (__ldcg: L2,
// coherent after the caller's fence) so the body costs a few round trips.
__device__ void gate_body(LoopCtl* ctl, const LoopGateDesc& g) {
    const u32 overflow = __ldcg(&ctl->overflow), done = __ldcg(&ctl->done), iter = __ldcg(&ctl->iter);
    const u32 nh = __ldcg(&ctl->nheads), epoch = __ldcg(&ctl->epoch_base);
    const u64 hist_cap = __ldcg(&ctl->hist_cap);
    u64 log_n0 = nh ? __ldcg(&ctl->h[0].log_n) : 0;
    if (overflow | done) return;
    if (iter >= hist_cap) {
        ctl->need_hist = hist_cap * 2;
        ctl->overflow = 1;
        return;
    }
    if (iter + 1 - epoch > g.stamp_max) {
        ctl->need_restamp = 1;
        ctl->overflow = 1;
        return;
    }
    bool over = false;
    for (u32 h = 0; h < nh; ++h) {
        u64 add = 0;
        for (u32 f = 0; f < g.nfinal; ++f)
            if (g.final_head[f] == h) add += __ldcg(&ctl->step_cand[g.final_step[f]]);
        ctl->h[h].cand = add;
        const u64 need = (h ? __ldcg(&ctl->h[h].log_n) : log_n0) + add;
        if (need > g.log_cap[h]) {
            ctl->need_log[h] = need;
            over = true;
        }
        if (need > g.tab_limit[h]) {
            ctl->need_tab[h] = need;
            over = true;
        }
    }
    if (over) ctl->overflow = 1;
}

// The gate evaluated by every CTA of the insert kernel itself (gate in the
// insert, gd_device_config.gate_in_insert): the same decision as gate_body
// from fields that stay fixed while the iteration inserts — the log size
// before any insert is the Δ window's end (log_n == dhi until the first
// append) — so every CTA reaches the same answer without a barrier; the
// caller's CTA 0 also writes the capacities it asks for (write = true).
// Returns true when the iteration must not insert.
__device__ bool gate_eval(LoopCtl* ctl, const LoopGateDesc& g, bool write) {
    const u32 overflow = __ldcg(&ctl->overflow), done = __ldcg(&ctl->done), iter = __ldcg(&ctl->iter);
    const u32 nh = __ldcg(&ctl->nheads), epoch = __ldcg(&ctl->epoch_base);
    const u64 hist_cap = __ldcg(&ctl->hist_cap);
    if (overflow | done) return true;
    if (iter >= hist_cap) {
        if (write) {
            ctl->need_hist = hist_cap * 2;
            ctl->overflow = 1;
        }
        return true;
    }
    if (iter + 1 - epoch > g.stamp_max) {
        if (write) {
            ctl->need_restamp = 1;
            ctl->overflow = 1;
        }
        return true;
    }
    bool over = false;
    for (u32 h = 0; h < nh; ++h) {
        u64 add = 0;
        for (u32 f = 0; f < g.nfinal; ++f)
            if (g.final_head[f] == h) add += __ldcg(&ctl->step_cand[g.final_step[f]]);
        const u64 need = __ldcg(&ctl->h[h].dhi) + add;
        if (write) ctl->h[h].cand = add;
        if (need > g.log_cap[h]) {
            if (write) ctl->need_log[h] = need;
            over = true;
        }
        if (need > g.tab_limit[h]) {
            if (write) ctl->need_tab[h] = need;
            over = true;
        }
    }
    if (over && write) ctl->overflow = 1;
    return over;
}

__device__ void end_body(LoopCtl* ctl, const LoopEndDesc& e) {
    const cudaGraphConditionalHandle cond = (cudaGraphConditionalHandle)e.cond;
    const u32 overflow = __ldcg(&ctl->overflow), done = __ldcg(&ctl->done), iter = __ldcg(&ctl->iter);
    const u32 nh = __ldcg(&ctl->nheads);
    const u32 ns = e.hist.nsteps;
    if (done) {
        if (e.use_cond) cudaGraphSetConditional(cond, 0);
        return;
    }
    if (overflow) {  // roll back: nothing was inserted (gate)
        for (u32 h = 0; h < nh; ++h) ctl->h[h].cand = ctl->h[h].J = ctl->h[h].N = ctl->h[h].D = 0;
        for (u32 s = 0; s < ns; ++s) ctl->step_total[s] = ctl->step_cand[s] = ctl->heavy_n[s] = 0;
        ctl->pre_valid = ctl->pre_bad = 0;  // the rerun counts its rows itself
        ctl->pre_cand = ctl->pre_heavy_n = 0;
        if (e.use_cond) cudaGraphSetConditional(cond, 0);
        return;
    }
    const u64 i = iter;
    bool active = false;
    for (u32 h = 0; h < nh; ++h) {  // a head's fields are loaded together
        LoopHeadState& st = ctl->h[h];
        const u64 dlo = __ldcg(&st.dlo), dhi = __ldcg(&st.dhi), J = __ldcg(&st.J), N = __ldcg(&st.N),
                  D = __ldcg(&st.D), ln = __ldcg(&st.log_n);
        gd_iter_record r;
        r.delta_in = dhi - dlo;
        r.join = J;
        r.new_unique = N;
        r.delta_out = D;
        r.full_after = ln;
        e.hist.rec[i * nh + h] = r;
        st.dlo = dhi;
        st.dhi = ln;
        active |= ln > dhi;
        st.cand = st.J = st.N = st.D = 0;
    }
    for (u32 s = 0; s < ns; ++s) {
        e.hist.steps[i * ns + s] = __ldcg(&ctl->step_total[s]);
        ctl->last_cand[s] = __ldcg(&ctl->step_cand[s]);
        ctl->step_total[s] = ctl->step_cand[s] = ctl->heavy_n[s] = 0;
    }
    if (e.pre_step != ~0u) {  // the next iteration's counts, from this iteration's insert
        const u32 bad = __ldcg(&ctl->pre_bad);
        if (!bad) {
            ctl->step_cand[e.pre_step] = __ldcg(&ctl->pre_cand);
            ctl->heavy_n[e.pre_step] = __ldcg(&ctl->pre_heavy_n);
            ctl->pre_sel ^= 1;
        }
        ctl->pre_valid = bad ? 0 : 1;
        ctl->pre_bad = 0;
        ctl->pre_cand = ctl->pre_heavy_n = 0;
    }
    ctl->iter = iter + 1;
    ctl->done = active ? 0 : 1;
    __threadfence();
    if (e.use_cond) cudaGraphSetConditional(cond, active ? 1 : 0);
}

// ---- kernels ----------------------------------------------------------------

__global__ void __launch_bounds__(kLT) loop_probe_kernel(LoopCtl* ctl, u32 step, LoopOuter o, DevJoin jd,
                                                         IndexView<u64> ix, LoopDense dense, u64 inner_n,
                                                         LoopStepBufs sb, u64* __restrict__ block_sums) {
    __shared__ u64 red[kLT / 32];
    __shared__ u32 s_flag;
    if (cta_stopped(ctl, &s_flag)) return;
    const u64* outer;
    u64 n;
    resolve(o, ctl, outer, n);
    if (n + 1 > sb.rows_cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            ctl->need_rows[step] = n + 1;
            ctl->overflow = 1;
        }
        return;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->step_n[step] = n;
    u64* __restrict__ row_start = sb.row_start;
    u64* __restrict__ row_cnt = sb.row_off;
    u64 begin, end;
    chunk_of(n, begin, end);
    u64 sum = 0;
    for (u64 t0 = begin; t0 < end; t0 += kLTile) {
        const u64 base = t0 + threadIdx.x;
        if (jd.jcc == 0 || inner_n == 0) {  // Cartesian step / empty inner
#pragma unroll
            for (int j = 0; j < kLItems; ++j) {
                const u64 r = base + (u64)j * kLT;
                if (r < end) {
                    const u64 c = jd.jcc == 0 ? inner_n : 0;
                    row_start[r] = 0;
                    row_cnt[r] = c;
                    sum += c;
                }
            }
            continue;
        }
        u64 pre[kLItems];
#pragma unroll
        for (int j = 0; j < kLItems; ++j) {
            const u64 r = base + (u64)j * kLT;
            pre[j] = r < end ? outer_prefix(jd, outer[r]) : 0ull;
        }
        if (dense.off) {
            u32 a[kLItems], b[kLItems];
#pragma unroll
            for (int j = 0; j < kLItems; ++j) {
                const u64 q = pre[j] - dense.lo;
                const bool in = q < dense.span;
                a[j] = in ? __ldg(dense.off + q) : 0u;
                b[j] = in ? __ldg(dense.off + q + 1) : 0u;
            }
#pragma unroll
            for (int j = 0; j < kLItems; ++j) {
                const u64 r = base + (u64)j * kLT;
                if (r >= end) continue;
                row_start[r] = a[j];
                row_cnt[r] = b[j] - a[j];
                sum += b[j] - a[j];
            }
            continue;
        }
        Slot s[kLItems];
#pragma unroll
        for (int j = 0; j < kLItems; ++j) s[j] = ix.slots[slot_home(pre[j], ix.slot_count)];
#pragma unroll
        for (int j = 0; j < kLItems; ++j) {
            const u64 r = base + (u64)j * kLT;
            if (r >= end) continue;
            u64 st = 0, ln = 0;
            if (s[j].tag == pre[j]) {
                st = s[j].val & kStartMask;
                const u64 l = s[j].val >> 40;
                ln = l == kLenSat ? run_end(ix, pre[j], st) - st : l;
            } else if (s[j].tag != kEmptySlot) {
                index_probe(ix, pre[j], st, ln);  // collision chain (rare)
            }
            row_start[r] = st;
            row_cnt[r] = ln;
            sum += ln;
        }
    }
    sum = block_sum(sum, red);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = sum;
}

// Row r's outputs occupy merge-path items [off_r + r, off_r + c_r + r]
// (outputs, then its row end E_r = off_{r+1} + r); the split of a tile
// boundary D (number of row ends before D) is r for E_{r-1} < D <= E_r.
__global__ void __launch_bounds__(kLT) loop_scan_kernel(LoopCtl* ctl, u32 step, LoopOuter o, LoopStepBufs sb,
                                                        const u64* __restrict__ block_sums, LoopGateDesc g,
                                                        int do_gate) {
    __shared__ u64 red[kLT / 32];
    __shared__ u64 s_scan[kLT / 32 + 1];
    __shared__ u32 s_flag;
    if (!cta_stopped(ctl, &s_flag)) {
        const u64* outer;
        u64 n;
        resolve(o, ctl, outer, n);
        u64 pre = 0, all = 0;
        for (u32 b = threadIdx.x; b < gridDim.x; b += kLT) {
            const u64 v = block_sums[b];
            all += v;
            if (b < blockIdx.x) pre += v;
        }
        pre = block_sum(pre, red);
        all = block_sum(all, red);
        const u64 ntiles = all ? (n + all + kLoopMatTile - 1) / kLoopMatTile : 0;
        const bool fits = ntiles + 1 <= sb.splits_cap;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            sb.row_off[n] = all;
            ctl->step_cand[step] = all;
            if (!fits) {
                ctl->need_splits[step] = ntiles + 1;
                ctl->overflow = 1;
            } else if (ntiles) {
                sb.splits[ntiles] = n;
            }
        }
        u64* __restrict__ row_off = sb.row_off;
        u64 begin, end;
        chunk_of(n, begin, end);
        u64 carry = pre;
        for (u64 t0 = begin; t0 < end; t0 += kLTile) {
            const u64 first = t0 + (u64)threadIdx.x * kLItems;
            u64 c[kLItems];
            u64 sum = 0;
#pragma unroll
            for (int j = 0; j < kLItems; ++j) {
                c[j] = first + j < end ? row_off[first + j] : 0;
                sum += c[j];
            }
            u64 tot;
            u64 off = carry + block_exclusive_scan<u64, kLT>(sum, tot, s_scan);
#pragma unroll
            for (int j = 0; j < kLItems; ++j) {
                const u64 r = first + j;
                if (r < end) {
                    row_off[r] = off;
                    if (fits) {
                        const u64 e_r = off + c[j] + r;
                        for (u64 d = (off + r + kLoopMatTile - 1) / kLoopMatTile * kLoopMatTile; d <= e_r;
                             d += kLoopMatTile)
                            sb.splits[d / kLoopMatTile] = r;
                    }
                }
                off += c[j];
            }
            carry += tot;
        }
    }
    if (do_gate && last_cta(ctl, &s_flag) && threadIdx.x == 0) gate_body(ctl, g);
}

struct MatSmem {
    u64 off[kLoopMatTile + 1];
    u64 start[kLoopMatTile + 1];
    u64 outer[kLoopMatTile + 1];
};

// Stages tile `tile`'s rows; returns false when the tile has no output.
__device__ __forceinline__ bool stage_tile(MatSmem& sm, u64 tile, const u64* outer, u64 n, u64 total,
                                           const LoopStepBufs& sb, u64& b0, u64& b1, u32& rcount) {
    const u64 diag0 = tile * kLoopMatTile;
    const u64 diag1 = min(diag0 + kLoopMatTile, n + total);
    const u64 a0 = sb.splits[tile], a1 = sb.splits[tile + 1];
    b0 = diag0 - a0;
    b1 = diag1 - a1;
    __syncthreads();  // previous tile's readers are done with sm
    if (b1 <= b0) return false;
    const u64 rlast = min(a1, n - 1);
    rcount = (u32)(rlast - a0 + 1);
    for (u32 i = threadIdx.x; i < rcount; i += kLT) {
        sm.off[i] = sb.row_off[a0 + i];
        sm.start[i] = sb.row_start[a0 + i];
        sm.outer[i] = outer[a0 + i];
    }
    __syncthreads();
    return true;
}

__device__ __forceinline__ u32 row_of(const MatSmem& sm, u32 rcount, u64 j) {
    u32 lo = 0, hi = rcount;
    while (hi - lo > 1) {
        const u32 mid = (lo + hi) >> 1;
        if (sm.off[mid] <= j) lo = mid;
        else hi = mid;
    }
    return lo;
}

constexpr int kPer = (int)(kLoopMatTile / kLT);  // outputs per thread per tile

__global__ void __launch_bounds__(kLT) loop_materialize_temp_kernel(LoopCtl* ctl, u32 step, LoopOuter o,
                                                                    const u64* __restrict__ inner, DevJoin jd,
                                                                    LoopStepBufs sb, u64* __restrict__ temp,
                                                                    u64 temp_cap) {
    __shared__ MatSmem sm;
    __shared__ u64 s_scan[kLT / 32 + 1];
    __shared__ u64 s_base;
    __shared__ u32 s_flag;
    if (cta_stopped(ctl, &s_flag)) return;
    const u64* outer;
    u64 n;
    resolve(o, ctl, outer, n);
    const u64 total = ctl->step_cand[step];
    // output window [wlo, whi) (windowed iteration) or everything
    const bool win = ctl->win_hi != 0 && ctl->win_step == step;
    const u64 wlo = win ? ctl->win_lo : 0, whi = win ? min(ctl->win_hi, total) : total;
    if (whi - wlo > temp_cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            ctl->need_temp[step] = whi - wlo;
            ctl->overflow = 1;
        }
        return;
    }
    if (jd.nfilters == 0 && blockIdx.x == 0 && threadIdx.x == 0) ctl->step_total[step] = whi - wlo;
    if (whi <= wlo) return;
    // tiles holding the window's outputs: output j lies on merge-path
    // diagonal j + (rows ended before it) = j + #{r : off[r+1] <= j}
    u64 t_lo = 0, t_hi = (n + total + kLoopMatTile - 1) / kLoopMatTile;
    if (win) {
        auto rows_before = [&](u64 j) {  // #{r < n : row_off[r+1] <= j}
            u64 lo = 0, hi = n;
            while (lo < hi) {
                const u64 mid = (lo + hi) >> 1;
                if (sb.row_off[mid + 1] <= j) lo = mid + 1;
                else hi = mid;
            }
            return lo;
        };
        t_lo = (wlo + rows_before(wlo)) / kLoopMatTile;
        t_hi = min(t_hi, (whi - 1 + rows_before(whi - 1)) / kLoopMatTile + 1);
    }
    for (u64 tile = t_lo + blockIdx.x; tile < t_hi; tile += gridDim.x) {
        u64 b0, b1;
        u32 rcount;
        if (!stage_tile(sm, tile, outer, n, total, sb, b0, b1, rcount)) continue;
        b0 = max(b0, wlo);
        b1 = min(b1, whi);
        if (jd.nfilters == 0) {
            for (u64 j = b0 + threadIdx.x; j < b1; j += kLT) {
                const u32 r = row_of(sm, rcount, j);
                const u64 i = inner[sm.start[r] + (j - sm.off[r])];
                temp[j - wlo] = project(jd, sm.outer[r], i);
            }
            continue;
        }
        // filtered: survivors compacted through one atomic per tile
        u64 key[kPer];
        bool keep[kPer];
        u64 cnt = 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const u64 j = b0 + threadIdx.x + (u64)k * kLT;
            keep[k] = false;
            if (j < b1) {
                const u32 r = row_of(sm, rcount, j);
                const u64 ov = sm.outer[r];
                const u64 i = inner[sm.start[r] + (j - sm.off[r])];
                keep[k] = passes(jd, ov, i);
                key[k] = project(jd, ov, i);
                cnt += keep[k];
            }
        }
        u64 tot;
        const u64 ex = block_exclusive_scan<u64, kLT>(cnt, tot, s_scan);
        if (threadIdx.x == 0) s_base = tot ? atomicAdd(&ctl->step_total[step], tot) : 0;
        __syncthreads();
        u64 p = s_base + ex;
#pragma unroll
        for (int k = 0; k < kPer; ++k)
            if (keep[k]) temp[p++] = key[k];
    }
}

__global__ void loop_gate_kernel(LoopCtl* ctl, LoopGateDesc g) {
    if (threadIdx.x == 0 && blockIdx.x == 0) gate_body(ctl, g);
}

__global__ void loop_end_kernel(LoopCtl* ctl, LoopEndDesc e) {
    if (threadIdx.x == 0 && blockIdx.x == 0) end_body(ctl, e);
}

__global__ void loop_select_cand_kernel(LoopCtl* ctl, u32 step, LoopOuter o) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (loop_stopped(ctl)) return;
    const u64* p;
    u64 n;
    resolve(o, ctl, p, n);
    ctl->step_n[step] = n;
    ctl->step_cand[step] = n;
}

// Appends the CTA's new keys of one tile to the log: one atomic per CTA and
// tile on the shared counter (per-warp atomics contend on it), warp ballots
// + an 8-entry scan for the positions.
template <int PER>
__device__ __forceinline__ void append_cta(u64* __restrict__ log, unsigned long long* log_n, const u64 (&key)[PER],
                                           u32 fresh, u32* s_warp, u64* s_base) {
    constexpr int W = kLT / 32;
    u32 m[PER];
    u32 tot = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        m[k] = __ballot_sync(0xffffffffu, fresh >> k & 1);
        tot += __popc(m[k]);
    }
    const u32 warp = threadIdx.x >> 5;
    if (lane_id() == 0) s_warp[warp] = tot;
    __syncthreads();
    if (threadIdx.x == 0) {
        u32 all = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const u32 c = s_warp[w];
            s_warp[w] = all;
            all += c;
        }
        *s_base = all ? atomicAdd(log_n, (unsigned long long)all) : 0;
    }
    __syncthreads();
    u64 base = *s_base + s_warp[warp];
    const u32 lt = lanemask_lt();
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        if (fresh >> k & 1) log[base + __popc(m[k] & lt)] = key[k];
        base += __popc(m[k]);
    }
}

// Appends the warp's new keys to the log with one atomic per warp: no CTA
// barrier, so a warp's next keys do not wait for the slowest warp's probes.
template <int PER>
__device__ __forceinline__ void append_warp(u64* __restrict__ log, unsigned long long* log_n, const u64 (&key)[PER],
                                            u32 fresh) {
    u32 m[PER];
    u32 tot = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        m[k] = __ballot_sync(0xffffffffu, fresh >> k & 1);
        tot += __popc(m[k]);
    }
    unsigned long long base = 0;
    if (lane_id() == 0 && tot) base = atomicAdd(log_n, (unsigned long long)tot);
    base = __shfl_sync(0xffffffffu, base, 0);
    const u32 lt = lanemask_lt();
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        if (fresh >> k & 1) log[base + __popc(m[k] & lt)] = key[k];
        base += __popc(m[k]);
    }
}

// Flushes per-thread J / N / D counts of a CTA (once, at exit).
__device__ __forceinline__ void flush_counts(LoopCtl* ctl, u32 head, u32 step, u64 J, u64 N, u64 D, u64* red,
                                             bool step_total = true) {
    const u64 j = block_sum(J, red);
    const u64 nn = block_sum(N, red);
    const u64 d = block_sum(D, red);
    if (threadIdx.x == 0) {
        if (j) {
            atomicAdd(&ctl->h[head].J, j);
            if (step_total) atomicAdd(&ctl->step_total[step], j);
        }
        if (nn) atomicAdd(&ctl->h[head].N, nn);
        if (d) atomicAdd(&ctl->h[head].D, d);
    }
}

// Final step: load-balanced expansion fused with dedup + difference + append
// (the join rows are never written to HBM).  Each random slot CAS costs a
// 64-byte line read and write-back, so this kernel runs at the random
// read-modify-write rate of HBM.
// 6 CTAs/SM (40 registers, a few spills) measured fastest on C2: 94 ms vs
// 100 ms at 5 CTAs (48 registers) and 120 ms at 8 CTAs (32 registers).
template <int NS>
__global__ void __launch_bounds__(kLT, 6) loop_materialize_insert_kernel(
    LoopCtl* ctl, u32 step, u32 head, LoopOuter o, const u64* __restrict__ inner, DevJoin jd, LoopStepBufs sb,
    LoopHeadBufs hb, LoopEndDesc e, int do_end) {
    __shared__ MatSmem sm;
    __shared__ u64 red[kLT / 32];
    __shared__ u32 s_warp[kLT / 32];
    __shared__ u64 s_base;
    __shared__ u32 s_flag;
    if (!cta_stopped(ctl, &s_flag)) {
        const u64* outer;
        u64 n;
        resolve(o, ctl, outer, n);
        const u64 total = ctl->step_cand[step];
        const u32 it = ctl->iter + 1 - ctl->epoch_base;
        const u64 ntiles = total ? (n + total + kLoopMatTile - 1) / kLoopMatTile : 0;
        u64 J = 0, N = 0, D = 0;
        for (u64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            u64 b0, b1;
            u32 rcount;
            if (!stage_tile(sm, tile, outer, n, total, sb, b0, b1, rcount)) continue;
            u64 key[kPer];
            u32 ok = 0;
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const u64 j = b0 + threadIdx.x + (u64)k * kLT;
                key[k] = 0;
                if (j < b1) {
                    const u32 r = row_of(sm, rcount, j);
                    const u64 ov = sm.outer[r];
                    const u64 i = inner[sm.start[r] + (j - sm.off[r])];
                    if (passes(jd, ov, i)) ok |= 1u << k;
                    key[k] = project(jd, ov, i);
                }
            }
            u32 fresh, first;
            hs_insert<kPer, NS>(hb, it, key, ok, fresh, first);
            J += __popc(ok);
            N += __popc(first);
            D += __popc(fresh);
            if (hb.warp_append) append_warp<kPer>(hb.log, &ctl->h[head].log_n, key, fresh);
            else append_cta<kPer>(hb.log, &ctl->h[head].log_n, key, fresh, s_warp, &s_base);
        }
        flush_counts(ctl, head, step, J, N, D, red);
    }
    if (do_end && last_cta(ctl, &s_flag) && threadIdx.x == 0) end_body(ctl, e);
}

// Dedup + difference + append of a final step's join rows (materialized in
// `keys` by loop_materialize_temp): each thread keeps kInsPer CASes in flight
// (the random-CAS rate needs ~8 K in flight per SM; a fused materialize
// kernel holds too many registers to get there).
template <int NS, int kInsPer = 8, int kMinCta = 4>
__global__ void __launch_bounds__(kLT, kMinCta) loop_insert_keys_kernel(LoopCtl* ctl, u32 step, u32 head,
                                                                  const u64* __restrict__ keys, LoopHeadBufs hb,
                                                                  LoopEndDesc e, int do_end) {
    __shared__ u64 red[kLT / 32];
    __shared__ u32 s_flag;
    if (!cta_stopped(ctl, &s_flag)) {
        const u64 n = ctl->step_total[step];
        const u32 it = ctl->iter + 1 - ctl->epoch_base;
        constexpr u64 kChunk = (u64)kLT * kInsPer;
        u64 J = 0, N = 0, D = 0;
        for (u64 base = (u64)blockIdx.x * kChunk; base < n; base += (u64)gridDim.x * kChunk) {
            u64 key[kInsPer];
            u32 ok = 0;
#pragma unroll
            for (int k = 0; k < kInsPer; ++k) {
                const u64 j = base + (u64)k * kLT + threadIdx.x;
                key[k] = j < n ? __ldcs(keys + j) : 0ull;
                ok |= (u32)(j < n) << k;
            }
            u32 fresh, first;
            hs_insert<kInsPer, NS>(hb, it, key, ok, fresh, first);
            J += __popc(ok);
            N += __popc(first);
            D += __popc(fresh);
            append_warp<kInsPer>(hb.log, &ctl->h[head].log_n, key, fresh);
        }
        flush_counts(ctl, head, step, J, N, D, red, false);
    }
    if (do_end && last_cta(ctl, &s_flag) && threadIdx.x == 0) end_body(ctl, e);
}

// Pipelined insert of materialized keys (packed slots; split final steps and
// the partitioned inbox): each thread keeps two batches of kPP keys — the
// next batch's key reads and home-slot reads are issued before the current
// batch's CASes, probes and log append run, so DRAM latency overlaps the
// L2 round trips instead of adding to them.  Probing is batched (every
// unresolved key advances one step per pass) and the append is one atomic
// per warp.
constexpr int kPP = 4;
struct PipeBatch {
    u64 key[kPP];
    u64 old[kPP];
    u32 ok;
};

__device__ __forceinline__ void pipe_issue(PipeBatch& b, const u64* __restrict__ keys, u64 base, u64 n,
                                           const u64* tab, u64 cap) {
    b.ok = 0;
#pragma unroll
    for (int k = 0; k < kPP; ++k) {
        const u64 j = base + (u64)k * kLT + threadIdx.x;
        b.key[k] = j < n ? __ldcs(keys + j) : 0ull;
        b.ok |= (u32)(j < n) << k;
    }
#pragma unroll
    for (int k = 0; k < kPP; ++k) b.old[k] = (b.ok >> k & 1) ? __ldcg(tab + hs_home(b.key[k], cap)) : 0ull;
}

// Settles batch b (its home slots already read) and appends its new keys.
__device__ __forceinline__ void pipe_resolve(PipeBatch& b, u64* tab, u64 cap, u32 sb, u32 st, u64* __restrict__ log,
                                             unsigned long long* log_n, u64& J, u64& N, u64& D) {
    const u64 smask = (1ull << sb) - 1;
    u64 pos[kPP];
#pragma unroll
    for (int k = 0; k < kPP; ++k) pos[k] = hs_home(b.key[k], cap);
    u32 pend = b.ok, fresh = 0, first = 0;
    while (pend) {
        u32 cas = 0;
#pragma unroll
        for (int k = 0; k < kPP; ++k) {
            if (!(pend >> k & 1)) continue;
            if (b.old[k] == kEmptySlot) {
                cas |= 1u << k;
            } else if ((b.old[k] >> sb) == b.key[k]) {
                if ((b.old[k] & smask) == st) pend &= ~(1u << k);
                else cas |= 1u << k;
            } else {
                pos[k] = pos[k] + 1 == cap ? 0 : pos[k] + 1;
                b.old[k] = __ldcg(tab + pos[k]);
            }
        }
        u64 res[kPP];
#pragma unroll
        for (int k = 0; k < kPP; ++k)
            if (cas >> k & 1) res[k] = atomicCAS(tab + pos[k], b.old[k], b.key[k] << sb | st);
#pragma unroll
        for (int k = 0; k < kPP; ++k) {
            if (!(cas >> k & 1)) continue;
            if (res[k] == b.old[k]) {
                fresh |= (u32)(b.old[k] == kEmptySlot) << k;
                first |= 1u << k;
                pend &= ~(1u << k);
            } else {
                b.old[k] = res[k];
            }
        }
    }
    J += __popc(b.ok);
    N += __popc(first);
    D += __popc(fresh);
    append_warp<kPP>(log, log_n, b.key, fresh);
}

__global__ void __launch_bounds__(kLT, 3) loop_insert_keys_pipe_kernel(LoopCtl* ctl, u32 step, u32 head,
                                                                       const u64* __restrict__ keys, LoopHeadBufs hb,
                                                                       LoopEndDesc e, int do_end) {
    __shared__ u64 red[kLT / 32];
    __shared__ u32 s_flag;
    if (!cta_stopped(ctl, &s_flag)) {
        const u64 n = ctl->step_total[step];
        const u32 st = ctl->iter + 1 - ctl->epoch_base;
        u64* tab = static_cast<u64*>(hb.tab);
        unsigned long long* log_n = reinterpret_cast<unsigned long long*>(&ctl->h[head].log_n);
        constexpr u64 kChunk = (u64)kLT * kPP;
        const u64 stride = (u64)gridDim.x * kChunk;
        u64 J = 0, N = 0, D = 0;
        u64 base = (u64)blockIdx.x * kChunk;
        PipeBatch a, b;
        pipe_issue(a, keys, base, n, tab, hb.tab_cap);
        while (base < n) {
            const u64 next = base + stride;
            pipe_issue(b, keys, next, n, tab, hb.tab_cap);  // in flight while a settles
            pipe_resolve(a, tab, hb.tab_cap, hb.sbits, st, hb.log, log_n, J, N, D);
            a = b;
            base = next;
        }
        flush_counts(ctl, head, step, J, N, D, red, false);
    }
    if (do_end && last_cta(ctl, &s_flag) && threadIdx.x == 0) end_body(ctl, e);
}

template <int NS>
__global__ void __launch_bounds__(kLT) loop_select_insert_kernel(LoopCtl* ctl, u32 step, u32 head, LoopOuter o,
                                                                 DevJoin jd, LoopHeadBufs hb, LoopEndDesc e,
                                                                 int do_end) {
    __shared__ u64 red[kLT / 32];
    __shared__ u32 s_warp[kLT / 32];
    __shared__ u64 s_base;
    __shared__ u32 s_flag;
    if (!cta_stopped(ctl, &s_flag)) {
        const u64* outer;
        u64 n;
        resolve(o, ctl, outer, n);
        const u32 it = ctl->iter + 1 - ctl->epoch_base;
        const u64 ntiles = (n + kLT - 1) / kLT;
        u64 J = 0, N = 0, D = 0;
        for (u64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const u64 r = tile * kLT + threadIdx.x;
            u64 key[1] = {0};
            const u32 ok = r < n && passes(jd, outer[r], 0ull) ? 1u : 0u;
            if (ok) key[0] = project(jd, outer[r], 0ull);
            u32 fresh, first;
            hs_insert<1, NS>(hb, it, key, ok, fresh, first);
            J += ok;
            N += first;
            D += fresh;
            append_cta<1>(hb.log, &ctl->h[head].log_n, key, fresh, s_warp, &s_base);
        }
        flush_counts(ctl, head, step, J, N, D, red);
    }
    if (do_end && last_cta(ctl, &s_flag) && threadIdx.x == 0) end_body(ctl, e);
}

// ---- warp-expanded final step over a dense inner ---------------------------
// (DESIGN.md §4b.)  loop_count reads each outer row's range from the
// L2-resident dense offsets, sums the candidates (one atomic per CTA) and
// queues rows with more than heavy_rows outputs as (row, segment) items;
// its last CTA runs the gate.  loop_expand_insert: every warp takes 32
// outer rows at a time (grid-stride), scans their counts with shuffles and
// expands the outputs — source row found by a 5-step shuffle search,
// filters applied, survivors compacted by ballot — into its own shared
// buffer; each full round of 256 keys is inserted with 8 keys per lane
// (home slots loaded together, hs_insert) and appended with one atomic per
// warp.  Then the heavy items, one warp each.  No CTA barrier in the loops,
// no per-row arrays, no merge-path splits.
constexpr int kXBuf = 512;    // keys per warp buffer (4 KB)
constexpr int kXRound = 256;  // keys per insert round (8 per lane)
constexpr int kXPer = kXRound / 32;

__device__ __forceinline__ void dense_range(const LoopDense& dv, u64 p, u64& a, u64& c) {
    const u64 q = p - dv.lo;
    if (q < dv.span) {
        const u32 x = __ldg(dv.off + q), y = __ldg(dv.off + q + 1);
        a = x;
        c = y - x;
    } else {
        a = c = 0;
    }
}

// The step buffers of this iteration / of the next one (precounted steps
// alternate two sets; pre_sel names the current one).
__device__ __forceinline__ LoopStepBufs bufs_of_iter(const LoopStepBufs& sb, const LoopCtl* ctl, bool next) {
    LoopStepBufs b = sb;
    if (sb.rc2 && (((ctl->pre_sel & 1) != 0) != next)) {
        b.rc = sb.rc2;
        b.row_start = sb.row_start2;
        b.row_off = sb.row_off2;
    }
    return b;
}

__global__ void __launch_bounds__(kLT) loop_count_kernel(LoopCtl* ctl, u32 step, LoopOuter o, DevJoin jd,
                                                         LoopDense dv, LoopStepBufs sb, u64 heavy_min,
                                                         LoopGateDesc g, int do_gate) {
    __shared__ u64 red[kLT / 32];
    __shared__ u32 s_flag;
    // the insert launched behind this kernel (programmatic dependent launch,
    // gd_device_config.pdl) may take SM slots as this grid's CTAs retire; it
    // waits for this grid's completion before reading anything
    asm volatile("griddepcontrol.launch_dependents;");
    if (!cta_stopped(ctl, &s_flag)) {
        const u64* outer;
        u64 n;
        resolve(o, ctl, outer, n);
        if (blockIdx.x == 0 && threadIdx.x == 0) ctl->step_n[step] = n;
        const LoopStepBufs sb0 = sb;
        LoopStepBufs sb = bufs_of_iter(sb0, ctl, false);
        if (sb0.rc2 && ctl->pre_valid) n = 0;  // the last insert counted these rows already
        if (sb.rc && n > sb.rows_cap) {  // the row ranges need n entries
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                atomicMax((unsigned long long*)&ctl->need_rows[step], (unsigned long long)(n + 1));
                ctl->overflow = 1;
            }
            n = 0;
        }
        u64 sum = 0;
        for (u64 base = (u64)blockIdx.x * kLTile; base < n; base += (u64)gridDim.x * kLTile) {
            u64 pre[kLItems];
#pragma unroll
            for (int j = 0; j < kLItems; ++j) {
                const u64 r = base + threadIdx.x + (u64)j * kLT;
                pre[j] = r < n ? outer_prefix(jd, outer[r]) : 0ull;
            }
            u64 a[kLItems], c[kLItems];
#pragma unroll
            for (int j = 0; j < kLItems; ++j) dense_range(dv, pre[j], a[j], c[j]);
#pragma unroll
            for (int j = 0; j < kLItems; ++j) {
                const u64 r = base + threadIdx.x + (u64)j * kLT;
                if (r >= n) continue;
                if (sb.rc) sb.rc[r] = a[j] << 32 | c[j];  // the expansion reads it instead of re-probing
                sum += c[j];
                if (c[j] > heavy_min) {
                    const u64 segs = (c[j] + heavy_min - 1) / heavy_min;
                    const u64 pos = atomicAdd((unsigned long long*)&ctl->heavy_n[step], (unsigned long long)segs);
                    if (pos + segs <= sb.rows_cap) {
                        for (u64 q = 0; q < segs; ++q) {
                            sb.row_start[pos + q] = r;
                            sb.row_off[pos + q] = q;
                        }
                    } else {
                        atomicMax((unsigned long long*)&ctl->need_rows[step], (unsigned long long)(pos + segs));
                        ctl->overflow = 1;
                    }
                }
            }
        }
        sum = block_sum(sum, red);
        if (threadIdx.x == 0 && sum) atomicAdd((unsigned long long*)&ctl->step_cand[step], (unsigned long long)sum);
    }
    if (do_gate && last_cta(ctl, &s_flag) && threadIdx.x == 0) gate_body(ctl, g);
}

struct XWarp {
    u64* buf;  // this warp's shared buffer
    u32 fill;  // keys in buf (warp-uniform)
    u64 J, N, D;
};

// Sink of the warp expansion: inserts buf[0, m) (m <= kXRound) into the
// head's index and appends the new keys to the log.
template <int NS, int PER = kXPer>
struct InsertSink {
    static constexpr int kRound = 32 * PER;
    const LoopHeadBufs& hb;  // the kernel parameter itself (a copy would take registers)
    u32 it;
    unsigned long long* log_n;
    // precount (LoopCtl.pre_*): each appended row's next-iteration range
    bool pre = false;
    LoopCtl* ctl = nullptr;
    const DevJoin* jd = nullptr;
    const LoopDense* dv = nullptr;
    LoopStepBufs nb = LoopStepBufs();
    u64 heavy_min = 0, d0 = 0;
    bool cand_only = false;  // count ahead: only the next iteration's candidate total
    // Row r of the next iteration (an appended key): its inner range and
    // heavy items, as loop_count would write them; returns its candidates.
    __device__ __forceinline__ u64 precount(u64 r, u64 key) {
        u64 a, c;
        dense_range(*dv, outer_prefix(*jd, key), a, c);
        if (cand_only) return c;
        if (r >= nb.rows_cap) {
            ctl->pre_bad = 1;
            return c;
        }
        nb.rc[r] = a << 32 | c;
        if (c > heavy_min) {
            const u64 segs = (c + heavy_min - 1) / heavy_min;
            const u64 hp = atomicAdd((unsigned long long*)&ctl->pre_heavy_n, (unsigned long long)segs);
            if (hp + segs <= nb.rows_cap) {
                for (u64 q = 0; q < segs; ++q) {
                    nb.row_start[hp + q] = r;
                    nb.row_off[hp + q] = q;
                }
            } else {
                ctl->pre_bad = 1;
            }
        }
        return c;
    }
    __device__ __forceinline__ void round(XWarp& w, u32 m) {
        __syncwarp();
        const u32 lane = lane_id();
        u64 key[PER];
        u32 ok = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const u32 idx = lane + 32u * k;
            key[k] = idx < m ? w.buf[idx] : 0ull;
            ok |= (u32)(idx < m) << k;
        }
        u32 fresh, first;
        hs_insert<PER, NS>(hb, it, key, ok, fresh, first);
        w.N += __popc(first);
        w.D += __popc(fresh);
        u32 mk[PER];
        u32 tot = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            mk[k] = __ballot_sync(0xffffffffu, fresh >> k & 1);
            tot += __popc(mk[k]);
        }
        unsigned long long base = 0;
        if (lane == 0 && tot) base = atomicAdd(log_n, (unsigned long long)tot);
        base = __shfl_sync(0xffffffffu, base, 0);
        const u32 lt = lanemask_lt();
        u64 csum = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const u64 p = base + __popc(mk[k] & lt);
            if (fresh >> k & 1) {
                hb.log[p] = key[k];
                if (pre) csum += precount(p - d0, key[k]);
            }
            base += __popc(mk[k]);
        }
        if (pre) {
            csum = warp_sum(csum);
            if (lane == 0 && csum) atomicAdd((unsigned long long*)&ctl->pre_cand, (unsigned long long)csum);
        }
        __syncwarp();
    }
};

// Sink of the split final step: buf[0, m) is appended to the step's temp
// (one atomic per round on the step's row count, coalesced stores); the
// insert runs as its own kernel (loop_insert_keys) over the temp.
struct TempSink {
    static constexpr int kRound = kXRound;
    u64* temp;
    unsigned long long* total;
    __device__ __forceinline__ void round(XWarp& w, u32 m) {
        __syncwarp();
        const u32 lane = lane_id();
        unsigned long long base = 0;
        if (lane == 0 && m) base = atomicAdd(total, (unsigned long long)m);
        base = __shfl_sync(0xffffffffu, base, 0);
        for (u32 i = lane; i < m; i += 32) temp[base + i] = w.buf[i];
        __syncwarp();
    }
};

// Sink of the partitioned loop: buf[0, m) goes to the owners' inboxes —
// per destination one system-scope atomic on the owner's cursor (counted
// even past the capacity, so the owner learns its demand), then coalesced
// (peer) stores.  Keys that do not fit raise part_inbox_over; the iteration
// is rolled back on every rank at the next barrier.
struct RouteSink {
    static constexpr int kRound = kXRound;
    const PeerTab* tab;
    LoopCtl* ctl;
    __device__ __forceinline__ void round(XWarp& w, u32 m) {
        __syncwarp();
        const u32 lane = lane_id();
        u64 key[kXPer];
        u32 own[kXPer];
        const u32 P = tab->P;
#pragma unroll
        for (int k = 0; k < kXPer; ++k) {
            const u32 idx = lane + 32u * k;
            key[k] = idx < m ? w.buf[idx] : 0ull;
            own[k] = idx < m ? (u32)(key_hash64<u64>(key[k]) % P) : kLoopMaxRanks;
        }
        const u32 lt = lanemask_lt();
        for (u32 q = 0; q < P; ++q) {
            u32 mk[kXPer];
            u32 tot = 0;
#pragma unroll
            for (int k = 0; k < kXPer; ++k) {
                mk[k] = __ballot_sync(0xffffffffu, own[k] == q);
                tot += __popc(mk[k]);
            }
            if (!tot) continue;
            PeerMail* mq = tab->mail[q];
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd_system(&mq->cursor, (unsigned long long)tot);
            base = __shfl_sync(0xffffffffu, base, 0);
            if (base + tot > tab->cap[q]) {
                if (lane == 0) ctl->part_inbox_over = 1;
                continue;
            }
            u64* dst = tab->inbox[q];
#pragma unroll
            for (int k = 0; k < kXPer; ++k) {
                if (own[k] == q) dst[base + __popc(mk[k] & lt)] = key[k];
                base += __popc(mk[k]);
            }
        }
        __syncwarp();
    }
};

// Adds one key per lane (`have`) to the warp buffer, compacted; a full
// round goes to the sink at once and the (< 32) keys past it move to the
// front.
template <class Sink>
__device__ __forceinline__ void x_emit(XWarp& w, bool have, u64 key, Sink& sink) {
    const u32 mask = __ballot_sync(0xffffffffu, have);
    if (have) w.buf[w.fill + __popc(mask & lanemask_lt())] = key;
    w.fill += __popc(mask);
    if (w.fill >= (u32)Sink::kRound) {
        sink.round(w, Sink::kRound);
        const u32 rest = w.fill - Sink::kRound;
        const u32 lane = lane_id();
        const u64 t = lane < rest ? w.buf[Sink::kRound + lane] : 0ull;
        __syncwarp();
        if (lane < rest) w.buf[lane] = t;
        w.fill = rest;
    }
}

// The expansion itself (both sinks): light rows 32 at a time per warp,
// then the heavy (row, segment) items queued by loop_count.
template <class Sink, int kXB = 4>
__device__ __forceinline__ void expand_rows(const LoopCtl* ctl, u32 step, const u64* outer, u64 n,
                                            const u64* __restrict__ inner, const DevJoin& jd, const LoopDense& dv,
                                            const LoopStepBufs& sb, u64 heavy_min, XWarp& w, Sink& sink) {
    const u64 nheavy = min(__ldcg(&ctl->heavy_n[step]), sb.rows_cap);
    const u32 lane = lane_id(), warp = threadIdx.x >> 5;
    const u64 gw = (u64)blockIdx.x * (kLT / 32) + warp, nw = (u64)gridDim.x * (kLT / 32);
    for (u64 base = gw * 32; base < n; base += nw * 32) {
        const u64 r = base + lane;
        u64 ov = 0, a = 0, c = 0;
        if (r < n) {
            if (sb.rc) {  // the row's range from loop_count: both loads independent
                ov = outer[r];
                const u64 v = __ldcg(sb.rc + r);
                a = v >> 32;
                c = v & 0xffffffffull;
            } else {
                ov = outer[r];
                dense_range(dv, outer_prefix(jd, ov), a, c);
            }
            if (c > heavy_min) c = 0;  // a heavy item (loop_count queued it)
        }
        const u64 incl = warp_inclusive_scan(c);
        const u64 T = __shfl_sync(0xffffffffu, incl, 31);
        const u64 excl = incl - c;
        // kXB outputs per lane at a time: their inner loads in flight together
        for (u64 j0 = 0; j0 < T; j0 += 32 * kXB) {
            u64 iv[kXB], so[kXB];
#pragma unroll
            for (int q = 0; q < kXB; ++q) {
                const u64 j = j0 + 32 * q + lane;
                // source lane: the last s with excl_s <= j (rows without
                // output share the next row's excl and are never last)
                u32 s = 0;
#pragma unroll
                for (u32 d = 16; d; d >>= 1) {
                    const u64 ex = __shfl_sync(0xffffffffu, excl, s + d);
                    if (ex <= j) s += d;
                }
                const u64 sa = __shfl_sync(0xffffffffu, a, s);
                const u64 se = __shfl_sync(0xffffffffu, excl, s);
                so[q] = __shfl_sync(0xffffffffu, ov, s);
                iv[q] = j < T ? inner[sa + (j - se)] : 0ull;
            }
#pragma unroll
            for (int q = 0; q < kXB; ++q) {
                if (j0 + 32 * q >= T) break;  // warp-uniform
                const u64 j = j0 + 32 * q + lane;
                bool have = false;
                u64 key = 0;
                if (j < T) {
                    have = passes(jd, so[q], iv[q]);
                    key = project(jd, so[q], iv[q]);
                }
                w.J += have;
                x_emit(w, have, key, sink);
            }
        }
    }
    for (u64 i = gw; i < nheavy; i += nw) {  // heavy items: one segment of heavy_min outputs per warp
        const u64 r = sb.row_start[i], sg = sb.row_off[i];
        const u64 ov = outer[r];
        u64 a, c;
        dense_range(dv, outer_prefix(jd, ov), a, c);
        const u64 b0 = sg * heavy_min, b1 = min(c, b0 + heavy_min);
        for (u64 j0 = b0; j0 < b1; j0 += 32) {
            const u64 j = j0 + lane;
            bool have = false;
            u64 key = 0;
            if (j < b1) {
                const u64 iv = inner[a + j];
                have = passes(jd, ov, iv);
                key = project(jd, ov, iv);
            }
            w.J += have;
            x_emit(w, have, key, sink);
        }
    }
    if (w.fill) sink.round(w, w.fill);
}

template <int NS, int PER = kXPer, int XB = 1>
__global__ void __launch_bounds__(kLT, PER >= 8 ? 3 : 5) loop_expand_insert_kernel(
    LoopCtl* ctl, u32 step, u32 head, LoopOuter o, const u64* __restrict__ inner, DevJoin jd, LoopDense dv,
    LoopStepBufs sb, u64 heavy_min, LoopHeadBufs hb, LoopEndDesc e, int do_end, LoopGateDesc g, int do_gate,
    int count_ahead) {
    __shared__ u64 sbuf[kLT / 32][PER >= 8 ? kXBuf : kXBuf / 2];
    __shared__ u64 red[kLT / 32];
    __shared__ u32 s_flag;
    // launched as a programmatic dependent of loop_count (pdl): wait for its
    // completion and memory (a no-op under a plain launch)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    bool stopped;
    if (do_gate) {  // the iteration's gate, evaluated here instead of in loop_count's last CTA
        if (threadIdx.x == 0) s_flag = gate_eval(ctl, g, blockIdx.x == 0) ? 1u : 0u;
        __syncthreads();
        stopped = s_flag != 0;
    } else {
        stopped = cta_stopped(ctl, &s_flag);
    }
    if (!stopped) {
        const u64* outer;
        u64 n;
        resolve(o, ctl, outer, n);
        const LoopStepBufs cur = bufs_of_iter(sb, ctl, false);
        InsertSink<NS, PER> sink{hb, ctl->iter + 1 - ctl->epoch_base,
                                 reinterpret_cast<unsigned long long*>(&ctl->h[head].log_n)};
        if (count_ahead) {  // the next iteration's candidate total, summed as its rows are appended
            sink.pre = true;
            sink.cand_only = true;
            sink.ctl = ctl;
            sink.jd = &jd;
            sink.dv = &dv;
            sink.d0 = ctl->h[head].dhi;
        } else if (sb.rc2) {  // precount the next iteration's rows as they are appended
            sink.pre = true;
            sink.ctl = ctl;
            sink.jd = &jd;
            sink.dv = &dv;
            sink.nb = bufs_of_iter(sb, ctl, true);
            sink.heavy_min = heavy_min;
            sink.d0 = ctl->h[head].dhi;
        }
        XWarp w{sbuf[threadIdx.x >> 5], 0, 0, 0, 0};
        expand_rows<InsertSink<NS, PER>, (PER >= 8 ? 4 : XB)>(ctl, step, outer, n, inner, jd, dv, cur, heavy_min, w, sink);
        flush_counts(ctl, head, step, w.J, w.N, w.D, red);
    }
    if (do_end && last_cta(ctl, &s_flag) && threadIdx.x == 0) end_body(ctl, e);
}

// Warp expansion into the step's temp (split final step): the capacity is
// checked against the exact candidate count first (outputs <= candidates).
__global__ void __launch_bounds__(kLT, 3) loop_expand_temp_kernel(LoopCtl* ctl, u32 step, LoopOuter o,
                                                                  const u64* __restrict__ inner, DevJoin jd,
                                                                  LoopDense dv, LoopStepBufs sb, u64 heavy_min,
                                                                  u64* __restrict__ temp, u64 temp_cap) {
    __shared__ u64 sbuf[kLT / 32][kXBuf];
    __shared__ u32 s_flag;
    if (cta_stopped(ctl, &s_flag)) return;
    const u64 cand = ctl->step_cand[step];
    if (cand > temp_cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            ctl->need_temp[step] = cand;
            ctl->overflow = 1;
        }
        return;
    }
    const u64* outer;
    u64 n;
    resolve(o, ctl, outer, n);
    TempSink sink{temp, reinterpret_cast<unsigned long long*>(&ctl->step_total[step])};
    XWarp w{sbuf[threadIdx.x >> 5], 0, 0, 0, 0};
    expand_rows(ctl, step, outer, n, inner, jd, dv, sb, heavy_min, w, sink);
}

__global__ void __launch_bounds__(kLT, 3) loop_expand_route_kernel(LoopCtl* ctl, u32 step, LoopOuter o,
                                                                   const u64* __restrict__ inner, DevJoin jd,
                                                                   LoopDense dv, LoopStepBufs sb, u64 heavy_min,
                                                                   const PeerTab* tab) {
    __shared__ u64 sbuf[kLT / 32][kXBuf];
    __shared__ u64 red[kLT / 32];
    __shared__ u32 s_flag;
    if (cta_stopped(ctl, &s_flag)) return;
    const u64* outer;
    u64 n;
    resolve(o, ctl, outer, n);
    RouteSink sink{tab, ctl};
    XWarp w{sbuf[threadIdx.x >> 5], 0, 0, 0, 0};
    expand_rows(ctl, step, outer, n, inner, jd, dv, sb, heavy_min, w, sink);
    const u64 j = block_sum(w.J, red);
    if (threadIdx.x == 0 && j) atomicAdd((unsigned long long*)&ctl->step_total[step], (unsigned long long)j);
    __threadfence_system();  // peer stores before the barrier's flag (loop_peer_sync1)
}

// Routes materialized rows (a chain's final temp) to their owners.
__global__ void __launch_bounds__(kLT) loop_route_keys_kernel(LoopCtl* ctl, u32 step, const u64* __restrict__ keys,
                                                              const PeerTab* tab) {
    __shared__ u64 sbuf[kLT / 32][kXRound];
    __shared__ u32 s_flag;
    if (cta_stopped(ctl, &s_flag)) return;
    const u64 n = ctl->step_total[step];
    RouteSink sink{tab, ctl};
    const u32 lane = lane_id(), warp = threadIdx.x >> 5;
    XWarp w{sbuf[warp], 0, 0, 0, 0};
    const u64 gw = (u64)blockIdx.x * (kLT / 32) + warp, nw = (u64)gridDim.x * (kLT / 32);
    for (u64 b = gw * kXRound; b < n; b += nw * kXRound) {
        const u32 m = (u32)min((u64)kXRound, n - b);
        for (u32 i = lane; i < m; i += 32) w.buf[i] = __ldcs(keys + b + i);
        sink.round(w, m);
    }
    __threadfence_system();
}

// ---- device-side barrier of the peer loop (one thread) --------------------
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ u64 global_ns() {
    u64 t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Publishes `val` to every rank's mailbox slot of this rank, then waits
// until every rank reached the same epoch; out[s] = rank s's payload.
// Returns false when a rank did not arrive within timeout_ns (a dead peer
// must not hang the GPU: the caller stops the graph, the host reports it).
__device__ bool peer_barrier(LoopCtl* ctl, const PeerTab* tab, u64 epoch, const u64 (&val)[kPeerVals],
                             u64 (&out)[kLoopMaxRanks][kPeerVals], u64 timeout_ns) {
    const u32 P = tab->P, me = tab->rank;
    for (u32 q = 0; q < P; ++q) {
        PeerMail* m = tab->mail[q];
#pragma unroll
        for (u32 k = 0; k < kPeerVals; ++k) m->val[me][k] = val[k];
    }
    __threadfence_system();
    for (u32 q = 0; q < P; ++q) st_release_sys(&tab->mail[q]->flag[me], epoch);
    PeerMail* mine = tab->mail[me];
    const u64 t0 = global_ns();
    for (u32 s = 0; s < P; ++s) {
        u64 f;
        while ((f = ld_acquire_sys(&mine->flag[s])) < epoch) {
            __nanosleep(64);
            if (global_ns() - t0 > timeout_ns) {
                ctl->dbg_rank = s;
                ctl->dbg_flag = f;
                ctl->dbg_epoch = epoch;
                return false;
            }
        }
#pragma unroll
        for (u32 k = 0; k < kPeerVals; ++k) out[s][k] = __ldcv(&mine->val[s][k]);
    }
    return true;
}

__global__ void loop_peer_sync1_kernel(LoopCtl* ctl, PeerSyncDesc d) {
    if (threadIdx.x || blockIdx.x) return;
    const cudaGraphConditionalHandle cond = (cudaGraphConditionalHandle)d.cond;
    if (ctl->done) {
        if (d.use_cond) cudaGraphSetConditional(cond, 0);
        return;
    }
    const PeerTab* tab = d.tab;
    const u64 epoch = ctl->part_epoch + 1;
    ctl->part_epoch = epoch;
    const u64 mine[kPeerVals] = {(u64)(ctl->overflow | ctl->part_inbox_over), 0, 0, 0};
    __shared__ u64 got[kLoopMaxRanks][kPeerVals];
    if (!peer_barrier(ctl, tab, epoch, mine, got, d.timeout_ns)) {
        ctl->part_timeout = 1;
        ctl->overflow = 1;
        if (d.use_cond) cudaGraphSetConditional(cond, 0);
        return;
    }
    u64 any = 0;
    for (u32 s = 0; s < tab->P; ++s) any |= got[s][0];
    const u64 recv = ld_acquire_sys(&tab->mail[tab->rank]->cursor);
    ctl->part_recv = recv;
    if (any) {  // roll back on every rank: nothing was inserted anywhere
        ctl->overflow = 1;
        ctl->part_over = 1;
        if (d.use_cond) cudaGraphSetConditional(cond, 0);
        return;
    }
    u64 j = 0;
    for (u32 s = 0; s < d.nsteps; ++s) j += ctl->step_total[s];
    ctl->part_join += j;
    // capacity gate of this rank's insert (no rollback past this point)
    const u64 need = ctl->h[0].log_n + recv;
    const bool stamp_over = ctl->iter + 1 - ctl->epoch_base > d.stamp_max;
    const bool hist_over = ctl->iter >= d.hist_cap;
    if (need > d.log_cap || need > d.tab_limit || stamp_over || hist_over) {
        ctl->part_stall = 1;
        ctl->need_log[0] = need;
        ctl->need_tab[0] = need;
        ctl->need_restamp = stamp_over;
        ctl->need_hist = hist_over ? ctl->iter + 1 : 0;
        ctl->step_total[d.final_step] = 0;  // the insert kernel does nothing
    } else {
        ctl->step_total[d.final_step] = recv;
    }
    ctl->h[0].J = ctl->h[0].N = ctl->h[0].D = 0;
    __threadfence();
}

__global__ void loop_peer_sync2_kernel(LoopCtl* ctl, PeerSyncDesc d) {
    if (threadIdx.x || blockIdx.x) return;
    const cudaGraphConditionalHandle cond = (cudaGraphConditionalHandle)d.cond;
    if (ctl->done || ctl->overflow) {
        if (d.use_cond) cudaGraphSetConditional(cond, 0);
        return;
    }
    const PeerTab* tab = d.tab;
    const u32 stall = ctl->part_stall;
    LoopHeadState& st = ctl->h[0];
    const u64 D = stall ? 0 : st.D;
    if (!stall) tab->mail[tab->rank]->cursor = 0;  // inbox consumed (peers route again only after this barrier)
    const u64 epoch = ctl->part_epoch + 1;
    ctl->part_epoch = epoch;
    const u64 mine[kPeerVals] = {D, (u64)stall, 0, 0};
    __shared__ u64 got[kLoopMaxRanks][kPeerVals];
    if (!peer_barrier(ctl, tab, epoch, mine, got, d.timeout_ns)) {
        ctl->part_timeout = 1;
        if (d.use_cond) cudaGraphSetConditional(cond, 0);
        return;
    }
    u64 gD = 0, any_stall = 0;
    for (u32 s = 0; s < tab->P; ++s) {
        gD += got[s][0];
        any_stall |= got[s][1];
    }
    if (!stall) {
        const u32 i = ctl->iter;
        gd_iter_record r;
        r.delta_in = st.dhi - st.dlo;
        r.join = ctl->part_recv;
        r.new_unique = st.N;
        r.delta_out = st.D;
        r.full_after = st.log_n;
        d.hist[i] = r;
        st.dlo = st.dhi;
        st.dhi = st.log_n;
        ctl->iter = i + 1;
        ctl->part_last_D = st.D;
        st.J = st.N = st.D = 0;
    }
    for (u32 s = 0; s < d.nsteps; ++s) ctl->step_total[s] = ctl->step_cand[s] = ctl->heavy_n[s] = 0;
    if (stall) ctl->step_total[d.final_step] = 0;
    __threadfence();
    if (any_stall) {
        ctl->part_stall_any = 1;
        if (d.use_cond) cudaGraphSetConditional(cond, 0);
        return;
    }
    if (gD == 0) {
        ctl->done = 1;
        if (d.use_cond) cudaGraphSetConditional(cond, 0);
        return;
    }
    if (d.use_cond) cudaGraphSetConditional(cond, 1);
}

// Rebuild of a table from the log (keys unique): stamp 0 = "before the
// current epoch".
__global__ void table_fill_kernel(void* tab, u64 cap, u32 sb, const u64* __restrict__ keys, u64 n) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 key = keys[i];
        u64 pos = hs_home(key, cap);
        while (true) {
            u64* w = sb ? static_cast<u64*>(tab) + pos : &static_cast<HSlot*>(tab)[pos].key;
            const u64 want = sb ? key << sb : key;
            const u64 old = atomicCAS(w, kEmptySlot, want);
            if (old == kEmptySlot) {
                if (!sb) static_cast<HSlot*>(tab)[pos].stamp = 0;
                break;
            }
            pos = pos + 1 == cap ? 0 : pos + 1;
        }
    }
}

// Growth: re-spread the old table into a larger one.  Home positions are
// umul64hi(hash, cap), monotone in the hash, and linear probing keeps each
// run in home order, so a contiguous run of old slots lands on a nearly
// contiguous run of new slots.  Each thread moves its own run of kRun old
// slots, so the CASes of a warp do not pile onto the same lines and every
// thread streams through both tables.  Stamps restart at 0 (growth happens
// between iterations).
constexpr u64 kRun = 32;
__global__ void table_rehash_kernel(const void* old_tab, u64 old_cap, void* tab, u64 cap, u32 sb) {
    const u64 runs = (old_cap + kRun - 1) / kRun;
    for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < runs; r += (u64)gridDim.x * blockDim.x) {
        const u64 end = min(old_cap, (r + 1) * kRun);
        // [blk, pos) is a range of slots known to be occupied (this thread's
        // placements and the occupied slots its probes stepped over): a key
        // whose home falls inside it may start probing at pos — no empty
        // slot lies between its home and its placement, so lookups find it.
        u64 blk = 0, pos = 0;
        for (u64 i = r * kRun; i < end; ++i) {
            const u64 w = sb ? __ldcs(static_cast<const u64*>(old_tab) + i)
                             : __ldcs(&static_cast<const HSlot*>(old_tab)[i].key);
            if (w == kEmptySlot) continue;
            const u64 key = sb ? w >> sb : w;
            const u64 home = hs_home(key, cap);
            const bool inside = blk <= home && home < pos;
            const u64 start = inside ? pos : home;
            u64 p = start;
            while (true) {
                u64* t = sb ? static_cast<u64*>(tab) + p : &static_cast<HSlot*>(tab)[p].key;
                if (atomicCAS(t, kEmptySlot, sb ? key << sb : key) == kEmptySlot) {
                    if (!sb) static_cast<HSlot*>(tab)[p].stamp = 0;
                    break;
                }
                p = p + 1 == cap ? 0 : p + 1;
            }
            if (p + 1 == cap || p < start) {  // wrapped: forget the range
                blk = pos = 0;
            } else {
                if (!inside) blk = home;  // [home, p] occupied now
                pos = p + 1;
            }
        }
    }
}

// Growth as a streaming pass (supersedes table_place for ratios it fits):
// CTA b owns old slots [i0, i1) and the new-table zone [zlo, zhi) they map
// to (i·cap/old_cap, zones partition the new table).  The zone is built in
// shared memory — cleared, keys placed by linear probing with shared CAS
// from their new home — then written out whole, EMPTY slots included, so
// the new table needs no separate clear and both tables are streamed
// once.  Keys whose new home lies outside the zone (displaced across the
// range start, or wrapped) or whose probe runs off the zone end are
// spilled and CAS-inserted afterwards.  Insertion order within a zone does
// not matter for linear probing (nothing is deleted).
constexpr u32 kZoneThreads = 256;
constexpr u32 kZoneSlotsMax = 8192;  // zone_slots upper bound
constexpr u32 kZoneBatch = 8;
__global__ void __launch_bounds__(kZoneThreads) table_zone_kernel(const void* old_tab, u64 old_cap, void* tab,
                                                                  u64 cap, u32 sb, u32 T, u64* __restrict__ spill,
                                                                  unsigned long long* nspill, u64 spill_cap) {
    extern __shared__ __align__(16) unsigned long long zone_raw[];
    const u64 i0 = (u64)blockIdx.x * T, i1 = min(old_cap, i0 + T);
    const u64 zlo = (u64)((u128)i0 * cap / old_cap);
    // zone[j] <-> new slot zlo + j, placed so shared and global addresses
    // agree mod 16 (the write-out is one bulk copy of the aligned run)
    unsigned long long* zone = zone_raw + (zlo & 1);
    const u64 zhi = i1 == old_cap ? cap : (u64)((u128)i1 * cap / old_cap);
    const u32 width = (u32)(zhi - zlo);  // <= the zone's shared slots (host sizes T)
    for (u32 j = threadIdx.x; j < width; j += kZoneThreads) zone[j] = kEmptySlot;
    __syncthreads();
    // kZoneBatch independent loads per thread in flight (the pass is
    // latency-bound with one)
    for (u64 base = i0; base < i1; base += (u64)kZoneThreads * kZoneBatch) {
        u64 w[kZoneBatch];
#pragma unroll
        for (u32 q = 0; q < kZoneBatch; ++q) {
            const u64 i = base + q * kZoneThreads + threadIdx.x;
            w[q] = i >= i1 ? kEmptySlot
                   : sb    ? __ldcs(static_cast<const u64*>(old_tab) + i)
                           : __ldcs(&static_cast<const HSlot*>(old_tab)[i].key);
        }
#pragma unroll
        for (u32 q = 0; q < kZoneBatch; ++q) {
            if (w[q] == kEmptySlot) continue;
            const u64 key = sb ? w[q] >> sb : w[q];
            const u64 want = sb ? key << sb : key;
            const u64 h = hs_home(key, cap);
            bool placed = false;
            if (h >= zlo && h < zhi) {
                for (u32 p = (u32)(h - zlo); p < width; ++p) {
                    if (zone[p] != kEmptySlot) continue;
                    if (atomicCAS(&zone[p], kEmptySlot, want) == kEmptySlot) {
                        placed = true;
                        break;
                    }
                }
            }
            if (!placed) {
                const u64 at = atomicAdd(nspill, 1ull);
                if (at < spill_cap) spill[at] = key;  // else: the host redoes the growth with CAS
            }
        }
    }
    __syncthreads();
    if (sb) {
        // The zone leaves shared memory as one bulk async copy (cp.async.bulk
        // shared -> global, UBLKCP): one instruction instead of width / 256
        // store rounds per thread; the (at most two) 8-byte slots outside
        // the 16-byte-aligned run are stored directly.
        u64* out = static_cast<u64*>(tab) + zlo;
        const u32 j0 = (u32)(zlo & 1), j1 = width > j0 ? j0 + ((width - j0) & ~1u) : j0;
        if (threadIdx.x == 0 && j1 > j0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + j0),
                         "r"((u32)__cvta_generic_to_shared(zone + j0)), "r"((j1 - j0) * 8u)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (threadIdx.x == 1 && j0 == 1) __stcs(out, (u64)zone[0]);
        if (threadIdx.x == 2 && j1 < width) __stcs(out + j1, (u64)zone[j1]);
        if (threadIdx.x == 0 && j1 > j0)  // shared memory stays until the copy has read it
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    } else {
        HSlot* out = static_cast<HSlot*>(tab) + zlo;
        for (u32 j = threadIdx.x; j < width; j += kZoneThreads) {
            const u64 k = zone[j];
            __stcs(reinterpret_cast<ulonglong2*>(out + j), make_ulonglong2(k, k == kEmptySlot ? kEmptySlot : 0ull));
        }
    }
}

// CAS insertion of the spilled keys (count in device memory).
__global__ void table_fill_dev_kernel(void* tab, u64 cap, u32 sb, const u64* __restrict__ keys,
                                      const unsigned long long* n_ptr) {
    const u64 n = *n_ptr;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 key = keys[i];
        u64 pos = hs_home(key, cap);
        while (true) {
            u64* w = sb ? static_cast<u64*>(tab) + pos : &static_cast<HSlot*>(tab)[pos].key;
            if (atomicCAS(w, kEmptySlot, sb ? key << sb : key) == kEmptySlot) {
                if (!sb) static_cast<HSlot*>(tab)[pos].stamp = 0;
                break;
            }
            pos = pos + 1 == cap ? 0 : pos + 1;
        }
    }
}

// New stamp epoch in place: every stamp back to 0.
__global__ void table_restamp_kernel(void* tab, u64 cap, u32 sb) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += (u64)gridDim.x * blockDim.x) {
        if (sb) {
            u64* t = static_cast<u64*>(tab) + i;
            const u64 w = *t;
            if (w != kEmptySlot) *t = w >> sb << sb;
        } else {
            HSlot& h = static_cast<HSlot*>(tab)[i];
            if (h.key != kEmptySlot) h.stamp = 0;
        }
    }
}

// ---- partitioned mode: group a step's join rows by owner rank -----------
// owner(key) = key_hash64(key) mod P, the function keep_owned partitions
// the seeded relation with (engine.cu).  Pass 1 counts per destination;
// pass 2 reserves one range per (CTA tile, destination) and scatters every
// row to offsets[dst] + range + its rank in the tile (shared atomics).
constexpr u32 kOwnTile = 2048;
constexpr u32 kMaxRanks = 64;

__global__ void owner_count_kernel(const u64* __restrict__ keys, const u64* __restrict__ n_ptr, u64 cap, u32 P,
                                   unsigned long long* __restrict__ counts) {
    __shared__ u32 sc[kMaxRanks];
    for (u32 i = threadIdx.x; i < P; i += blockDim.x) sc[i] = 0;
    __syncthreads();
    const u64 n = min(*n_ptr, cap);  // an overflowed step: bounded, and redone by the host
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        atomicAdd(&sc[key_hash64<u64>(keys[i]) % P], 1u);
    __syncthreads();
    for (u32 i = threadIdx.x; i < P; i += blockDim.x)
        if (sc[i]) atomicAdd(&counts[i], (unsigned long long)sc[i]);
}

__global__ void owner_scatter_kernel(const u64* __restrict__ keys, const u64* __restrict__ n_ptr, u32 P,
                                     const unsigned long long* __restrict__ offsets,
                                     unsigned long long* __restrict__ cursors, u64* __restrict__ out) {
    __shared__ u32 sc[kMaxRanks];
    __shared__ unsigned long long sb[kMaxRanks];
    const u64 n = *n_ptr;
    for (u64 t0 = (u64)blockIdx.x * kOwnTile; t0 < n; t0 += (u64)gridDim.x * kOwnTile) {
        for (u32 i = threadIdx.x; i < P; i += blockDim.x) sc[i] = 0;
        __syncthreads();
        constexpr u32 kPerT = kOwnTile / 256;
        u64 k[kPerT];
        u32 dst[kPerT], rank[kPerT];
#pragma unroll
        for (u32 q = 0; q < kPerT; ++q) {
            const u64 i = t0 + q * 256 + threadIdx.x;
            dst[q] = kMaxRanks;
            if (i < n) {
                k[q] = keys[i];
                dst[q] = (u32)(key_hash64<u64>(k[q]) % P);
                rank[q] = atomicAdd(&sc[dst[q]], 1u);
            }
        }
        __syncthreads();
        for (u32 i = threadIdx.x; i < P; i += blockDim.x)
            sb[i] = sc[i] ? offsets[i] + atomicAdd(&cursors[i], (unsigned long long)sc[i]) : 0;
        __syncthreads();
#pragma unroll
        for (u32 q = 0; q < kPerT; ++q)
            if (dst[q] < kMaxRanks) out[sb[dst[q]] + rank[q]] = k[q];
        __syncthreads();
    }
}

__global__ void part_meta_kernel(const unsigned long long* __restrict__ counts, const LoopCtl* ctl, u32 P,
                                 u64 min_delta, u64* __restrict__ meta) {
    const u32 p = threadIdx.x;
    if (p >= P) return;
    const u64 d = ctl->h[0].dhi - ctl->h[0].dlo;
    meta[3 * p] = counts[p];
    meta[3 * p + 1] = d > min_delta ? d : min_delta;
    meta[3 * p + 2] = ctl->overflow;
}

__global__ void part_advance_kernel(LoopCtl* ctl, u32 final_step, u64 recv_rows, gd_iter_record* hist) {
    if (threadIdx.x || blockIdx.x) return;
    LoopHeadState& st = ctl->h[0];
    const u32 i = ctl->iter;
    gd_iter_record r;
    r.delta_in = st.dhi - st.dlo;
    r.join = recv_rows;
    r.new_unique = st.N;
    r.delta_out = st.D;
    r.full_after = st.log_n;
    hist[i] = r;
    st.dlo = st.dhi;
    st.dhi = st.log_n;
    ctl->iter = i + 1;
    ctl->step_total[final_step] = 0;
}

// Streaming fill / copy for the growth path (16-byte vectors; the driver's
// memset / device-to-device memcpy showed 3-146 ms for the same sizes).
__global__ void fill_u64_kernel(ulonglong2* __restrict__ p, u64 n2, u64 v) {
    const ulonglong2 w = make_ulonglong2(v, v);
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (u64)gridDim.x * blockDim.x) p[i] = w;
}
// Streaming copy (log growth): four 16-byte loads in flight per thread
// before their stores (one load per thread measured 1.6 TB/s on a 2 GB log).
__global__ void copy_u64_kernel(ulonglong2* __restrict__ d, const ulonglong2* __restrict__ s, u64 n2) {
    constexpr int kU = 4;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i0 = (u64)blockIdx.x * blockDim.x + threadIdx.x; i0 < n2; i0 += kU * stride) {
        ulonglong2 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (i0 + u * stride < n2) v[u] = __ldcs(s + i0 + u * stride);
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (i0 + u * stride < n2) __stcs(d + i0 + u * stride, v[u]);
    }
}

template <typename Kern>
int occupancy(Kern k, size_t smem = 0) {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, kLT, smem);
    return b > 0 ? b : 1;
}

int g_occ_temp = 0, g_occ_insert = 0, g_occ_select = 0, g_occ_keys = 0, g_occ_expand = 0, g_occ_xroute = 0,
    g_occ_route = 0, g_occ_xtemp = 0, g_occ_keys_pipe = 0, g_occ_keys4 = 0, g_occ_keys2 = 0, g_occ_expand4 = 0;
// Insert grid = waves x resident CTAs: CTAs beyond the resident set start as
// others finish, so the hardware balances the iteration's tiles.  Large
// relations (log capacity >= kWideLog rows) run 3 waves (C2 -2.8%, SG
// W=4000 -4.3%); small ones 1, where the idle CTAs' launch cost shows
// (C1 +5% at 3).  gd_device_config.insert_waves overrides.
constexpr u64 kWideLog = 64ull << 20;

}  // namespace

int loop_grid(const Ctx& c) { return c.num_sms * 4; }

// Insert mode (gd_device_config.insert_slots): 0 CAS first, 1 load first,
// 2 load first with batched probing.
#define SLOT_DISPATCH(c, kern, ...)                                      \
    do {                                                                 \
        if ((c).cfg.insert_slots == 2) kern<2> __VA_ARGS__;              \
        else if ((c).cfg.insert_slots == 0) kern<0> __VA_ARGS__;         \
        else kern<1> __VA_ARGS__;                                        \
    } while (0)

void loop_prepare() {
    if (g_occ_temp) return;
    g_occ_temp = occupancy(loop_materialize_temp_kernel);
    g_occ_insert = occupancy(loop_materialize_insert_kernel<1>);
    g_occ_keys = occupancy(loop_insert_keys_kernel<1>);
    g_occ_keys4 = occupancy(loop_insert_keys_kernel<1, 4, 6>);
    g_occ_keys2 = occupancy(loop_insert_keys_kernel<1, 2, 8>);
    g_occ_select = occupancy(loop_select_insert_kernel<1>);
    g_occ_expand = occupancy(loop_expand_insert_kernel<1>);
    g_occ_expand4 = occupancy(loop_expand_insert_kernel<1, 4>);
    g_occ_xroute = occupancy(loop_expand_route_kernel);
    g_occ_route = occupancy(loop_route_keys_kernel);
    g_occ_xtemp = occupancy(loop_expand_temp_kernel);
    g_occ_keys_pipe = occupancy(loop_insert_keys_pipe_kernel);
}

void loop_fill_u64(Ctx& c, u64* p, u64 n, u64 v) {
    if (n == 0) return;
    if ((reinterpret_cast<uintptr_t>(p) & 15) || (n & 1)) {  // allocator blocks are 256-aligned; odd tails only
        c.memset(p, (int)(v & 0xff), n * sizeof(u64));
        if (v != (v & 0xff) * 0x0101010101010101ull) throw_logic("loop_fill_u64: unaligned non-byte fill");
        return;
    }
    const u64 n2 = n / 2;
    fill_u64_kernel<<<(int)std::min<u64>((n2 + 255) / 256, (u64)c.num_sms * 16), 256, 0, c.stream>>>(
        reinterpret_cast<ulonglong2*>(p), n2, v);
    c.check_launch();
}

void loop_copy_u64(Ctx& c, u64* d, const u64* s, u64 n) {
    if (n == 0) return;
    const u64 n2 = n / 2;
    if (n2 && !(reinterpret_cast<uintptr_t>(d) & 15) && !(reinterpret_cast<uintptr_t>(s) & 15)) {
        copy_u64_kernel<<<(int)std::min<u64>((n2 + 1023) / 1024, (u64)c.num_sms * 8), 256, 0, c.stream>>>(
            reinterpret_cast<ulonglong2*>(d), reinterpret_cast<const ulonglong2*>(s), n2);
        c.check_launch();
        if (n & 1) c.d2d(d + n - 1, s + n - 1, sizeof(u64));
        return;
    }
    c.d2d(d, s, n * sizeof(u64));
}

void loop_table_clear(Ctx& c, void* tab, u64 cap, u32 sbits) {
    const u64 words = cap * loop_slot_bytes(sbits) / 8;
    if (words & 1) c.memset(tab, 0xff, words * 8);
    else loop_fill_u64(c, static_cast<u64*>(tab), words, kEmptySlot);
}

void loop_table_fill(Ctx& c, void* tab, u64 cap, u32 sbits, const u64* keys, u64 n) {
    if (n == 0) return;
    const int grid = (int)std::max<u64>(1, std::min<u64>((n + 255) / 256, (u64)c.num_sms * 16));
    table_fill_kernel<<<grid, 256, 0, c.stream>>>(tab, cap, sbits, keys, n);
    c.check_launch();
}

void loop_table_rehash(Ctx& c, const void* old_tab, u64 old_cap, void* tab, u64 cap, u32 sbits, u64 nkeys) {
    // `tab` is uninitialised: the zone pass writes every slot; the CAS
    // fallbacks clear it first.
    if (old_cap == 0) {
        loop_table_clear(c, tab, cap, sbits);
        return;
    }
    const bool cas_only = c.cfg.rehash_cas_only != 0;
    const u32 zslots = std::min<u32>(kZoneSlotsMax, std::max<u32>(1024, c.cfg.zone_slots));
    const u64 T = (u64)((double)(zslots - 2) * (double)old_cap / (double)cap) / 32 * 32;
    const u64 nzones = T ? (old_cap + T - 1) / T : 0;
    if (!cas_only && T >= 256 && nzones < (1u << 31)) {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(table_zone_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)((kZoneSlotsMax + 2) * sizeof(u64)));
            attr = true;
        }
        const u64 spill_cap = nkeys / 16 + (1u << 20);
        DevBuf<u64> spill(c, spill_cap);
        DevBuf<unsigned long long> ns(c, 1);
        c.memset(ns.p, 0, sizeof(unsigned long long));
        table_zone_kernel<<<(unsigned)nzones, kZoneThreads, (zslots + 2) * sizeof(u64), c.stream>>>(
            old_tab, old_cap, tab, cap, sbits, (u32)T, spill.p, ns.p, spill_cap);
        c.check_launch();
        unsigned long long spilled;
        c.read_words(&spilled, ns.p, 1);
        if (spilled <= spill_cap) {
            if (spilled) {
                table_fill_dev_kernel<<<c.num_sms * 4, 256, 0, c.stream>>>(tab, cap, sbits, spill.p, ns.p);
                c.check_launch();
            }
            return;
        }
    }
    loop_table_clear(c, tab, cap, sbits);  // CAS re-spread (spill list overflowed, or a very large ratio)
    const u64 runs = (old_cap + kRun - 1) / kRun;
    const int grid = (int)std::max<u64>(1, std::min<u64>((runs + 255) / 256, (u64)c.num_sms * 16));
    table_rehash_kernel<<<grid, 256, 0, c.stream>>>(old_tab, old_cap, tab, cap, sbits);
    c.check_launch();
}

void loop_table_restamp(Ctx& c, void* tab, u64 cap, u32 sbits) {
    const int grid = (int)std::max<u64>(1, std::min<u64>((cap + 255) / 256, (u64)c.num_sms * 16));
    table_restamp_kernel<<<grid, 256, 0, c.stream>>>(tab, cap, sbits);
    c.check_launch();
}

void loop_probe(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, const LoopOuter& o, const DevJoin& jd,
                const IndexView<u64>* ix, const LoopDense& dense, u64 inner_n, const LoopStepBufs& sb,
                u64* block_sums) {
    IndexView<u64> v{};
    if (ix) v = *ix;
    loop_probe_kernel<<<loop_grid(c), kLT, 0, s>>>(ctl, step, o, jd, v, dense, inner_n, sb, block_sums);
    c.check_launch();
}

namespace {
// off[q] = lower_bound of prefix lo + q among the sorted rows (q in [0, span]).
__global__ void dense_offsets_kernel(const u64* __restrict__ rows, u64 n, u32 arity, u32 bits, u64 lo, u64 span,
                                     u32* __restrict__ off) {
    for (u64 q = (u64)blockIdx.x * blockDim.x + threadIdx.x; q <= span; q += (u64)gridDim.x * blockDim.x) {
        const u64 p = lo + q;
        u64 a = 0, b = n;
        while (a < b) {
            const u64 m = (a + b) >> 1;
            if (prefix_of(rows[m], arity, bits, 1) < p) a = m + 1;
            else b = m;
        }
        off[q] = (u32)a;
    }
}
}  // namespace

__global__ void dense_max_group_kernel(const u32* __restrict__ off, u64 span, unsigned long long* out) {
    u32 m = 0;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < span; i += (u64)gridDim.x * blockDim.x)
        m = max(m, off[i + 1] - off[i]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, (unsigned long long)m);
}

u64 loop_dense_max_group(Ctx& c, const LoopDense& dv) {
    if (!dv.off || !dv.span) return 0;
    DevBuf<unsigned long long> m(c, 1);
    c.memset(m.p, 0, sizeof(unsigned long long));
    const int grid = (int)std::max<u64>(1, std::min<u64>((dv.span + 255) / 256, (u64)c.num_sms * 8));
    dense_max_group_kernel<<<grid, 256, 0, c.stream>>>(dv.off, dv.span, m.p);
    c.check_launch();
    unsigned long long v = 0;
    c.read_words(&v, m.p, 1);
    return v;
}

bool loop_dense_build(Ctx& c, const u64* rows, u64 n, u32 arity, u32 bits, DevBuf<u32>& off, u64& lo, u64& span) {
    if (n == 0 || n >= (1ull << 32)) return false;
    unsigned long long first = 0, last = 0;
    c.read2(&first, rows, &last, rows + (n - 1));
    lo = prefix_of(first, arity, bits, 1);
    const u64 hi = prefix_of(last, arity, bits, 1);
    span = hi - lo + 1;
    if (span > 4 * n + 4096) return false;
    off = DevBuf<u32>(c, span + 1);
    const int grid = (int)std::max<u64>(1, std::min<u64>((span + 256) / 256, (u64)c.num_sms * 16));
    dense_offsets_kernel<<<grid, 256, 0, c.stream>>>(rows, n, arity, bits, lo, span, off.p);
    c.check_launch();
    return true;
}

void loop_scan(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, const LoopOuter& o, const LoopStepBufs& sb,
               const u64* block_sums, const LoopGateDesc* gate) {
    LoopGateDesc g{};
    if (gate) g = *gate;
    loop_scan_kernel<<<loop_grid(c), kLT, 0, s>>>(ctl, step, o, sb, block_sums, g, gate ? 1 : 0);
    c.check_launch();
}

void loop_gate(Ctx& c, cudaStream_t s, LoopCtl* ctl, const LoopGateDesc& g) {
    loop_gate_kernel<<<1, 32, 0, s>>>(ctl, g);
    c.check_launch();
}

void loop_materialize_temp(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, const LoopOuter& o, const u64* inner,
                           const DevJoin& jd, const LoopStepBufs& sb, u64* temp, u64 temp_cap) {
    loop_materialize_temp_kernel<<<c.num_sms * g_occ_temp, kLT, 0, s>>>(ctl, step, o, inner, jd, sb, temp,
                                                                         temp_cap);
    c.check_launch();
}

void loop_select_cand(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, const LoopOuter& o) {
    loop_select_cand_kernel<<<1, 32, 0, s>>>(ctl, step, o);
    c.check_launch();
}

void loop_insert_keys(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, u32 head, const u64* keys,
                      const LoopHeadBufs& hb, const LoopEndDesc* end) {
    LoopEndDesc e{};
    if (end) e = *end;
    if (hb.sbits && c.cfg.insert_pipeline)
        loop_insert_keys_pipe_kernel<<<c.num_sms * g_occ_keys_pipe, kLT, 0, s>>>(ctl, step, head, keys, hb, e,
                                                                                end ? 1 : 0);
    else if (c.cfg.insert_per_thread == 4)
        loop_insert_keys_kernel<1, 4, 6><<<c.num_sms * g_occ_keys4, kLT, 0, s>>>(ctl, step, head, keys, hb, e,
                                                                                end ? 1 : 0);
    else if (c.cfg.insert_per_thread == 2)
        loop_insert_keys_kernel<1, 2, 8><<<c.num_sms * g_occ_keys2, kLT, 0, s>>>(ctl, step, head, keys, hb, e,
                                                                                end ? 1 : 0);
    else
        SLOT_DISPATCH(c, loop_insert_keys_kernel, <<<c.num_sms * g_occ_keys, kLT, 0, s>>>(ctl, step, head, keys, hb,
                                                                                          e, end ? 1 : 0));
    c.check_launch();
}

void loop_materialize_insert(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, u32 head, const LoopOuter& o,
                             const u64* inner, const DevJoin& jd, const LoopStepBufs& sb,
                             const LoopHeadBufs& hb, const LoopEndDesc* end) {
    LoopEndDesc e{};
    if (end) e = *end;
    const int waves = c.cfg.insert_waves ? (int)c.cfg.insert_waves : (hb.log_cap >= kWideLog ? 3 : 1);
    SLOT_DISPATCH(c, loop_materialize_insert_kernel, <<<c.num_sms * g_occ_insert * waves, kLT, 0, s>>>(ctl, step, head, o, inner, jd,
                                                                                    sb, hb, e, end ? 1 : 0));
    c.check_launch();
}

void loop_select_insert(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, u32 head, const LoopOuter& o,
                        const DevJoin& jd, const LoopHeadBufs& hb, const LoopEndDesc* end) {
    LoopEndDesc e{};
    if (end) e = *end;
    SLOT_DISPATCH(c, loop_select_insert_kernel, <<<c.num_sms * g_occ_select, kLT, 0, s>>>(ctl, step, head, o, jd, hb, e,
                                                                        end ? 1 : 0));
    c.check_launch();
}

void loop_owner_count(Ctx& c, const u64* keys, const u64* n_ptr, u64 cap, u32 P, unsigned long long* counts) {
    owner_count_kernel<<<c.num_sms * 4, 256, 0, c.stream>>>(keys, n_ptr, cap, P, counts);
    c.check_launch();
}

void loop_part_meta(Ctx& c, const unsigned long long* counts, const LoopCtl* ctl, u32 P, u64 min_delta, u64* meta) {
    part_meta_kernel<<<1, 64, 0, c.stream>>>(counts, ctl, P, min_delta, meta);
    c.check_launch();
}

void loop_part_advance(Ctx& c, LoopCtl* ctl, u32 final_step, u64 recv_rows, gd_iter_record* hist) {
    part_advance_kernel<<<1, 32, 0, c.stream>>>(ctl, final_step, recv_rows, hist);
    c.check_launch();
}

void loop_owner_scatter(Ctx& c, const u64* keys, const u64* n_ptr, u32 P, const unsigned long long* offsets,
                        unsigned long long* cursors, u64* out) {
    owner_scatter_kernel<<<c.num_sms * 4, 256, 0, c.stream>>>(keys, n_ptr, P, offsets, cursors, out);
    c.check_launch();
}

void loop_count(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, const LoopOuter& o, const DevJoin& jd,
                const LoopDense& dense, const LoopStepBufs& sb, u64 heavy_rows, const LoopGateDesc* gate) {
    LoopGateDesc g{};
    if (gate) g = *gate;
    const int grid = c.cfg.count_ctas_per_sm ? c.num_sms * (int)c.cfg.count_ctas_per_sm : loop_grid(c);
    loop_count_kernel<<<grid, kLT, 0, s>>>(ctl, step, o, jd, dense, sb, heavy_rows, g, gate ? 1 : 0);
    c.check_launch();
}

void loop_expand_insert(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, u32 head, const LoopOuter& o,
                        const u64* inner, const DevJoin& jd, const LoopDense& dense, const LoopStepBufs& sb,
                        u64 heavy_rows, const LoopHeadBufs& hb, const LoopEndDesc* end, const LoopGateDesc* gate,
                        bool count_ahead) {
    LoopEndDesc e{};
    if (end) e = *end;
    LoopGateDesc g{};
    if (gate) g = *gate;
    const int waves = c.cfg.insert_waves ? (int)c.cfg.insert_waves : 1;
    if (c.cfg.expand_keys_per_lane == 4 && c.cfg.pdl) {
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3((unsigned)(c.num_sms * g_occ_expand4 * waves));
        lc.blockDim = dim3(kLT);
        lc.dynamicSmemBytes = 0;
        lc.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        GD_CUDA(cudaLaunchKernelEx(&lc, loop_expand_insert_kernel<1, 4>, ctl, step, head, o, inner, jd, dense, sb,
                                   heavy_rows, hb, e, end ? 1 : 0, g, gate ? 1 : 0, count_ahead ? 1 : 0));
    } else if (c.cfg.expand_keys_per_lane == 4)
        loop_expand_insert_kernel<1, 4><<<c.num_sms * g_occ_expand4 * waves, kLT, 0, s>>>(
            ctl, step, head, o, inner, jd, dense, sb, heavy_rows, hb, e, end ? 1 : 0, g, gate ? 1 : 0,
            count_ahead ? 1 : 0);
    else
        SLOT_DISPATCH(c, loop_expand_insert_kernel, <<<c.num_sms * g_occ_expand * waves, kLT, 0, s>>>(
        ctl, step, head, o, inner, jd, dense, sb, heavy_rows, hb, e, end ? 1 : 0, g, gate ? 1 : 0,
        count_ahead ? 1 : 0));
    c.check_launch();
}

void loop_expand_route(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, const LoopOuter& o, const u64* inner,
                       const DevJoin& jd, const LoopDense& dense, const LoopStepBufs& sb, u64 heavy_rows,
                       const PeerTab* tab) {
    loop_expand_route_kernel<<<c.num_sms * g_occ_xroute, kLT, 0, s>>>(ctl, step, o, inner, jd, dense, sb,
                                                                      heavy_rows, tab);
    c.check_launch();
}

void loop_expand_temp(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, const LoopOuter& o, const u64* inner,
                      const DevJoin& jd, const LoopDense& dense, const LoopStepBufs& sb, u64 heavy_rows, u64* temp,
                      u64 temp_cap) {
    loop_expand_temp_kernel<<<c.num_sms * g_occ_xtemp, kLT, 0, s>>>(ctl, step, o, inner, jd, dense, sb, heavy_rows,
                                                                    temp, temp_cap);
    c.check_launch();
}

void loop_route_keys(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, const u64* keys, const PeerTab* tab) {
    loop_route_keys_kernel<<<c.num_sms * g_occ_route, kLT, 0, s>>>(ctl, step, keys, tab);
    c.check_launch();
}

void loop_peer_sync1(Ctx& c, cudaStream_t s, LoopCtl* ctl, const PeerSyncDesc& d) {
    loop_peer_sync1_kernel<<<1, 32, 0, s>>>(ctl, d);
    c.check_launch();
}

void loop_peer_sync2(Ctx& c, cudaStream_t s, LoopCtl* ctl, const PeerSyncDesc& d) {
    loop_peer_sync2_kernel<<<1, 32, 0, s>>>(ctl, d);
    c.check_launch();
}

void loop_end(Ctx& c, cudaStream_t s, LoopCtl* ctl, const LoopEndDesc& end) {
    loop_end_kernel<<<1, 32, 0, s>>>(ctl, end);
    c.check_launch();
}

}  // namespace gd
