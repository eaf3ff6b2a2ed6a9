// radix_sort.cu — LSD onesweep radix sort of bit-packed tuple keys (the HISA
// sort of canonicalize, tuple_array.hpp:73-133, and of permute_columns,
// ra.hpp:426-454).
//
// One pass per 8-bit digit over only the significant low `nbits` bits of the
// packed keys.  A single histogram kernel counts every pass's digits in one
// read of the keys; each pass is then ONE kernel: a CTA claims a tile, ranks
// its keys with warp-level multi-split (__match_any_sync + per-warp digit
// counters in shared memory, stable), publishes its per-digit counts,
// resolves its global per-digit offsets by decoupled look-back (one thread
// per digit), stages the keys digit-sorted in shared memory and writes them
// out so consecutive threads write consecutive addresses of a digit run.
// HBM traffic per pass: read 8·n + write 8·n bytes (u64 keys).
#include "dev_common.cuh"
#include "ops.h"

namespace gd {

namespace {

constexpr int kRadixBits = 8;
constexpr int kRadix = 256;
constexpr int kSortThreads = 256;
constexpr int kWarps = kSortThreads / 32;
constexpr u64 kPortion = 1ull << 28;  // keys per look-back portion (30-bit status values)

template <typename K>
__device__ __forceinline__ u32 digit_of(K k, u32 shift) {
    return (u32)(k >> shift) & (kRadix - 1);
}

// Counts the digits of every pass for keys [begin, begin+n).  Warps
// increment privatized copies (`copies` per CTA, dynamic shared memory of
// npass * 256 words each, at most 32 KB): the top digits of packed keys are
// few and skewed, and one shared copy serialises the CTA on them.
template <typename K>
__global__ void __launch_bounds__(256) radix_hist_kernel(const K* __restrict__ keys, u64 begin, u64 n,
                                                         int npass, int copies, u64* __restrict__ hist) {
    extern __shared__ u32 sh[];
    const int words = npass * kRadix;
    for (int i = threadIdx.x; i < copies * words; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    u32* mine = sh + ((threadIdx.x >> 5) % copies) * words;
    // four independent loads in flight per thread (the pass is otherwise
    // latency-bound on the key stream)
    constexpr int kU = 4;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i0 = (u64)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += kU * stride) {
        K k[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const u64 i = i0 + u * stride;
            if (i < n) k[u] = keys[begin + i];
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (i0 + u * stride < n)
                for (int p = 0; p < npass; ++p) atomicAdd(&mine[p * kRadix + digit_of(k[u], p * kRadixBits)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < words; i += blockDim.x) {
        u32 t = 0;
        for (int c = 0; c < copies; ++c) t += sh[c * words + i];
        if (t) atomicAdd(&hist[i], (u64)t);
    }
}

// bases[pass][d] = number of keys whose pass-digit is smaller than d.
__global__ void radix_bases_kernel(const u64* __restrict__ hist, u64* __restrict__ bases) {
    __shared__ u64 scan_tmp[kRadix / 32 + 1];
    const int pass = blockIdx.x;
    const int d = threadIdx.x;
    u64 all;
    bases[pass * kRadix + d] =
        block_exclusive_scan<u64, kRadix>(hist[pass * kRadix + d], all, scan_tmp);
}

constexpr u32 kSFlagA = 1u << 30;
constexpr u32 kSFlagP = 2u << 30;
constexpr u32 kSMask = (1u << 30) - 1;

template <typename K, int I, bool BALLOT = false, int MINB = 3>
__global__ void __launch_bounds__(kSortThreads, MINB) onesweep_kernel(
    const K* __restrict__ in, K* __restrict__ out, u64 portion_begin, u64 portion_n, u32 shift,
    const u64* __restrict__ digit_base, u64* __restrict__ next_base, u32* __restrict__ ws,
    u32 ntiles) {
    constexpr int TILE = kSortThreads * I;
    __shared__ K s_keys[TILE];
    __shared__ u32 s_whist[kWarps][kRadix + 1];
    __shared__ u32 s_dstart[kRadix];
    __shared__ u64 s_gbase[kRadix];
    __shared__ u32 s_scan[kSortThreads / 32 + 1];
    __shared__ u32 s_tile;

    u32* counter = ws;
    u32* status = ws + 1;

    if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
    const u32 warp = threadIdx.x >> 5, lane = lane_id();
    for (int i = threadIdx.x; i < kWarps * (kRadix + 1); i += kSortThreads) (&s_whist[0][0])[i] = 0;
    __syncthreads();
    const u64 tile = s_tile;
    const u64 tile_begin = tile * TILE;
    const u32 tile_n = (u32)min((u64)TILE, portion_n - tile_begin);

    // Digits are recomputed from the keys where needed (fewer registers);
    // invalid (past-the-end) items use digit kRadix, a group never counted.
    K k[I];
#pragma unroll
    for (int i = 0; i < I; ++i) {
        const u32 idx = warp * (I * 32) + i * 32 + lane;
        k[i] = idx < tile_n ? in[portion_begin + tile_begin + idx] : K(0);
    }
    auto dig = [&](int i) -> u32 {
        const u32 idx = warp * (I * 32) + i * 32 + lane;
        return idx < tile_n ? digit_of(k[i], shift) : (u32)kRadix;
    };

    // Warp-level multi-split ranking, stable in (item, lane) = input order:
    // peers share a digit; the group leader bumps the warp's digit counter
    // with one shared atomic and broadcasts the old value.  Ranks (< 2^16)
    // are packed two per register.
    u32 rank2[(I + 1) / 2];
    // all match masks first: independent MATCH instructions pipeline
    u32 pm[I];
#pragma unroll
    for (int i = 0; i < I; ++i) {
        if constexpr (BALLOT) {  // peers by one ballot per digit bit (+ validity), no MATCH.ANY
            const u32 d = dig(i);
            const bool valid = d < (u32)kRadix;
            const u32 vb = __ballot_sync(0xffffffffu, valid);
            u32 peers = valid ? vb : ~vb;
#pragma unroll
            for (int b = 0; b < kRadixBits; ++b) {
                const bool bit = (d >> b) & 1;
                const u32 bb = __ballot_sync(0xffffffffu, bit);
                peers &= bit ? bb : ~bb;
            }
            pm[i] = peers;
        } else {
            pm[i] = __match_any_sync(0xffffffffu, dig(i));
        }
    }
#pragma unroll
    for (int i = 0; i < I; ++i) {
        const u32 d = dig(i);
        const u32 peers = pm[i];
        const u32 leader = 31 - __clz(peers);  // highest lane: no bit reversal
        u32 base = 0;
        if (lane == leader) base = atomicAdd(&s_whist[warp][d], (u32)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        const u32 r = base + __popc(peers & lanemask_lt());
        if (i & 1) rank2[i >> 1] |= r << 16;
        else rank2[i >> 1] = r;
    }
    __syncthreads();

    // Thread t owns digit t: per-warp exclusive offsets and the tile count.
    const u32 t = threadIdx.x;
    u32 cnt = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const u32 c = s_whist[w][t];
        s_whist[w][t] = cnt;
        cnt += c;
    }
    // Publish the tile aggregate early so successors can proceed.
    u32* my_status = status + tile * kRadix + t;
    if (tile == 0) st_relaxed32(my_status, kSFlagP | cnt);
    else st_relaxed32(my_status, kSFlagA | cnt);

    u32 total;
    const u32 dstart = block_exclusive_scan<u32, kSortThreads>(cnt, total, s_scan);
    s_dstart[t] = dstart;

    // Look-back for digit t across previous tiles of this portion, a window
    // of kLookWindow predecessors per step (independent loads), so the walk
    // back to the nearest inclusive prefix takes ~tiles/kLookWindow round
    // trips instead of one per tile.
    u32 excl = 0;
    if (tile > 0) {
        // Window of kLookWindow predecessors loaded together, consumed in
        // order; an unpublished predecessor is waited on alone (one status
        // word per retry — re-reading the whole window while spinning tripled
        // the L2 reads of a pass, profiles/r2_ncu_captures.md).
        constexpr int kLookWindow = 8;
        long long pred = (long long)tile - 1;
        bool found = false;
        while (!found) {
            u32 sv[kLookWindow];
#pragma unroll
            for (int w = 0; w < kLookWindow; ++w)
                sv[w] = pred - w >= 0 ? ld_relaxed32(status + (u64)(pred - w) * kRadix + t) : kSFlagP;
#pragma unroll
            for (int w = 0; w < kLookWindow; ++w) {
                if (found) break;
                u32 v = sv[w];
                while ((v >> 30) == 0) v = ld_relaxed32(status + (u64)(pred - w) * kRadix + t);
                excl += v & kSMask;
                found = (v >> 30) == 2;
            }
            pred -= kLookWindow;
        }
        st_relaxed32(my_status, kSFlagP | (excl + cnt));
    }
    const u64 base_t = digit_base[t];
    s_gbase[t] = base_t + excl - dstart;
    // The last tile of a portion hands the next portion its digit bases.
    if (tile == ntiles - 1 && next_base) next_base[t] = base_t + excl + cnt;
    __syncthreads();

    // Scatter into shared memory in digit-sorted (stable) order.
#pragma unroll
    for (int i = 0; i < I; ++i) {
        const u32 d = dig(i);
        const u32 r = (rank2[i >> 1] >> ((i & 1) * 16)) & 0xffffu;
        if (d < kRadix) s_keys[s_dstart[d] + s_whist[warp][d] + r] = k[i];
    }
    __syncthreads();

    for (u32 j = threadIdx.x; j < tile_n; j += kSortThreads) {
        const K key = s_keys[j];
        out[s_gbase[digit_of(key, shift)] + j] = key;
    }
}

// ---- pipelined onesweep (u64 keys) -------------------------------------------
// Persistent CTAs (as many as are co-resident), each claiming tiles in
// order: while a tile is ranked, looked back and written out, the CTA's
// NEXT tile is already streaming into a second shared-memory buffer through
// one bulk async copy (cp.async.bulk → UBLKCP, completion on an mbarrier),
// so every CTA keeps 32 KB of reads in flight through its whole compute
// phase instead of stalling on the load at the start of each tile.  Digits
// are RB (8..10) bits wide: 46-bit C2 keys sort in 5 passes of ≤ 10 bits
// instead of 6 of 8.  Per-warp digit counters are u16 pairs in one u32
// word (a warp ranks ≤ 512 keys), so 8 warps × 1024 digits take 16 KB.
// Thread t owns the DPT consecutive digits [t·DPT, (t+1)·DPT) for the
// per-digit work (counts, scan, look-back: one DPT-wide vector load per
// predecessor tile).  Stable in input order, as LSD requires.
constexpr int kPT = 256;         // threads
constexpr int kPI = 16;          // keys per thread
constexpr int kPTile = kPT * kPI;  // 4096 keys, 32 KB
constexpr int kPW = kPT / 32;

// IP (in place): the tile's keys are held in registers after ranking and
// the digit-sorted staging reuses the tile's own buffer (64 KB less shared
// memory per CTA: 2 CTAs per SM at 10-bit digits, 3 at 8-bit).
template <int RB, bool IP>
struct PipeSmem {
    static constexpr int R = 1 << RB;
    u64 buf[2][kPTile];
    u64 stage[IP ? 2 : kPTile];
    u32 wh[kPW][R / 2];  // per-warp digit counters / offsets, u16 pairs
    u32 dstart[R];
    u64 gbase[R];
    u32 scan[kPT / 32 + 1];
    unsigned long long mbar[2];
    u32 tile[2];
};

__device__ __forceinline__ u32 smem_addr(const void* p) { return (u32)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* m) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(m)) : "memory");
}

// One thread: order this CTA's earlier generic-proxy accesses of the
// buffer before the async copy overwrites it, arm the barrier with the
// byte count and issue the bulk copy (bytes % 16 == 0, 16-byte aligned).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, u32 bytes, unsigned long long* m) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(m)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(m))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* m, u32 parity) {
    const u32 a = smem_addr(m);
    u32 done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}

template <int DPT>
struct DigitVec {
    u32 v[DPT];
};

template <int DPT>
__device__ __forceinline__ DigitVec<DPT> ld_status_vec(const u32* p) {
    DigitVec<DPT> r;
    if constexpr (DPT == 2) {
        asm volatile("ld.relaxed.gpu.global.v2.u32 {%0, %1}, [%2];" : "=r"(r.v[0]), "=r"(r.v[1]) : "l"(p) : "memory");
    } else {
        asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3])
                     : "l"(p)
                     : "memory");
    }
    return r;
}

template <int DPT>
__device__ __forceinline__ void st_status_vec(u32* p, const DigitVec<DPT>& r) {
    if constexpr (DPT == 2) {
        asm volatile("st.relaxed.gpu.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(r.v[0]), "r"(r.v[1]) : "memory");
    } else {
        asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(r.v[0]), "r"(r.v[1]),
                     "r"(r.v[2]), "r"(r.v[3])
                     : "memory");
    }
}

template <int RB, bool IP, bool BALLOT>
__global__ void __launch_bounds__(kPT, IP ? 2 : 1) onesweep_pipe_kernel(const u64* __restrict__ in, u64* __restrict__ out,
                                                            u64 portion_begin, u64 portion_n, u32 shift, u32 width,
                                                            const u64* __restrict__ digit_base,
                                                            u64* __restrict__ next_base, u32* __restrict__ ws,
                                                            u32 ntiles) {
    constexpr int R = 1 << RB;
    constexpr int DPT = R >= 1024 ? 4 : 2;  // digits per owner thread
    constexpr int OWN = R / DPT;            // owner threads (128 / 256)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    PipeSmem<RB, IP>& sm = *reinterpret_cast<PipeSmem<RB, IP>*>(smem_raw);
    u32* counter = ws;
    u32* status = ws + 4;  // 16-byte aligned statuses
    const u32 t = threadIdx.x, warp = t >> 5, lane = lane_id();
    const u32 dmask = (1u << width) - 1;
    const u64* src = in + portion_begin;

    auto issue = [&](u32 b, u32 tile) {
        const u64 first = (u64)tile * kPTile;
        const u32 n = (u32)min((u64)kPTile, portion_n - first);
        const u32 bytes = (n * 8u) & ~15u;
        if (bytes) bulk_load(sm.buf[b], src + first, bytes, &sm.mbar[b]);
        else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&sm.mbar[b])) : "memory");
    };

    if (t == 0) {
        mbar_init(&sm.mbar[0]);
        mbar_init(&sm.mbar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // static round-robin tiles (b, b + G, ...): every CTA of the grid is
        // co-resident (sized from the occupancy), so a tile's predecessors
        // are always being processed in the same round and the prefetched
        // next tile never holds up another CTA's look-back (an atomic claim
        // made at prefetch time did: measured 2x slower)
        (void)counter;
        const u32 first = blockIdx.x;
        sm.tile[0] = first;
        if (first < ntiles) issue(0, first);
    }
    u32 cur = 0, ph0 = 0, ph1 = 0;
    while (true) {
        __syncthreads();  // (A) previous tile fully written out; tile ids visible
        const u32 tile = sm.tile[cur];
        if (tile >= ntiles) break;
        if (t == 0) {  // prefetch this CTA's next tile into the other buffer
            const u32 nx = tile + gridDim.x;
            sm.tile[cur ^ 1] = nx;
            if (nx < ntiles) issue(cur ^ 1, nx);
        }
        for (int i = t; i < kPW * (R / 2); i += kPT) (&sm.wh[0][0])[i] = 0;
        const u64 tile_begin = (u64)tile * kPTile;
        const u32 tile_n = (u32)min((u64)kPTile, portion_n - tile_begin);
        mbar_wait(&sm.mbar[cur], cur ? ph1 : ph0);
        if (cur) ph1 ^= 1;
        else ph0 ^= 1;
        u64* keys = sm.buf[cur];
        if (t == 0 && (tile_n & 1)) keys[tile_n - 1] = src[tile_begin + tile_n - 1];
        __syncthreads();  // (B) keys (incl. the odd tail key) and zeroed counters visible

        // warp multi-split ranking, stable in (item, lane) order
        u32 rank2[kPI / 2];
        u64 kr[IP ? kPI : 1];
#pragma unroll
        for (int i = 0; i < kPI; ++i) {
            const u32 idx = warp * (kPI * 32) + i * 32 + lane;
            const u64 kv = keys[idx];
            if constexpr (IP) kr[i] = kv;
            const u32 d = idx < tile_n ? (u32)(kv >> shift) & dmask : (u32)R;
            u32 peers;
            if constexpr (BALLOT) {
                // lanes with the same digit: one ballot per digit bit (plus
                // validity) instead of MATCH.ANY, whose latency dominated
                // the ranking (ncu: short-scoreboard stalls on its results)
                const bool valid = idx < tile_n;
                const u32 vb = __ballot_sync(0xffffffffu, valid);
                peers = valid ? vb : ~vb;
#pragma unroll
                for (int b = 0; b < RB; ++b) {
                    const bool bit = (d >> b) & 1;
                    const u32 bb = __ballot_sync(0xffffffffu, bit);
                    peers &= bit ? bb : ~bb;
                }
            } else {
                peers = __match_any_sync(0xffffffffu, d);
            }
            const u32 leader = 31 - __clz(peers);
            u32 base = 0;
            if (lane == leader && d < (u32)R) {
                const u32 sh = (d & 1) * 16;
                base = (atomicAdd(&sm.wh[warp][d >> 1], (u32)__popc(peers) << sh) >> sh) & 0xffffu;
            }
            base = __shfl_sync(0xffffffffu, base, leader);
            const u32 r = base + __popc(peers & lanemask_lt());
            if (i & 1) rank2[i >> 1] |= r << 16;
            else rank2[i >> 1] = r;
        }
        __syncthreads();  // (C)

        // per-digit work: thread t < OWN owns digits [t*DPT, t*DPT + DPT)
        DigitVec<DPT> cnt{};
        u32 own_sum = 0;
        if (t < (u32)OWN) {
#pragma unroll
            for (int q = 0; q < DPT; q += 2) {
                const u32 w = (t * DPT + q) >> 1;
                u32 c0 = 0, c1 = 0;
#pragma unroll
                for (int wp = 0; wp < kPW; ++wp) {
                    const u32 v = sm.wh[wp][w];
                    sm.wh[wp][w] = c0 | c1 << 16;
                    c0 += v & 0xffffu;
                    c1 += v >> 16;
                }
                cnt.v[q] = c0;
                cnt.v[q + 1] = c1;
                own_sum += c0 + c1;
            }
            DigitVec<DPT> pub;
#pragma unroll
            for (int q = 0; q < DPT; ++q) pub.v[q] = (tile == 0 ? kSFlagP : kSFlagA) | cnt.v[q];
            st_status_vec<DPT>(status + (u64)tile * R + t * DPT, pub);
        }
        u32 total;
        u32 dst0 = block_exclusive_scan<u32, kPT>(own_sum, total, sm.scan);
        if (t < (u32)OWN) {
            DigitVec<DPT> excl{};
            if (tile > 0) {
                constexpr int kWin = 8;
                long long pred = (long long)tile - 1;
                u32 pend = (1u << DPT) - 1;  // digits still looking back
                while (pend) {
                    DigitVec<DPT> s[kWin];
#pragma unroll
                    for (int w = 0; w < kWin; ++w) {
                        if (pred - w >= 0) s[w] = ld_status_vec<DPT>(status + (u64)(pred - w) * R + t * DPT);
                        else {
#pragma unroll
                            for (int q = 0; q < DPT; ++q) s[w].v[q] = kSFlagP;
                        }
                    }
                    bool wait = false;
#pragma unroll
                    for (int q = 0; q < DPT; ++q) {
                        if (!(pend >> q & 1)) continue;
                        int first_inv = kWin, first_p = kWin;
#pragma unroll
                        for (int w = kWin - 1; w >= 0; --w) {
                            const u32 f = s[w].v[q] >> 30;
                            if (f == 0) first_inv = w;
                            if (f == 2) first_p = w;
                        }
                        if (first_inv < first_p) {
                            wait = true;
                            break;
                        }
                    }
                    if (wait) continue;  // an unpublished predecessor inside the window: reload
#pragma unroll
                    for (int q = 0; q < DPT; ++q) {
                        if (!(pend >> q & 1)) continue;
                        int first_p = kWin;
#pragma unroll
                        for (int w = kWin - 1; w >= 0; --w)
                            if ((s[w].v[q] >> 30) == 2) first_p = w;
#pragma unroll
                        for (int w = 0; w < kWin; ++w)
                            if (w <= first_p) excl.v[q] += s[w].v[q] & kSMask;
                        if (first_p < kWin) pend &= ~(1u << q);
                    }
                    pred -= kWin;
                }
                DigitVec<DPT> pub;
#pragma unroll
                for (int q = 0; q < DPT; ++q) pub.v[q] = kSFlagP | (excl.v[q] + cnt.v[q]);
                st_status_vec<DPT>(status + (u64)tile * R + t * DPT, pub);
            }
#pragma unroll
            for (int q = 0; q < DPT; ++q) {
                const u32 d = t * DPT + q;
                const u64 b = digit_base[d];
                sm.dstart[d] = dst0;
                sm.gbase[d] = b + excl.v[q] - dst0;
                if (tile == ntiles - 1 && next_base) next_base[d] = b + excl.v[q] + cnt.v[q];
                dst0 += cnt.v[q];
            }
        }
        __syncthreads();  // (D)

        // scatter into shared memory in digit-sorted (stable) order
        u64* stage = IP ? keys : sm.stage;
#pragma unroll
        for (int i = 0; i < kPI; ++i) {
            const u32 idx = warp * (kPI * 32) + i * 32 + lane;
            if (idx < tile_n) {
                u64 k;
                if constexpr (IP) k = kr[i];
                else k = keys[idx];
                const u32 d = (u32)(k >> shift) & dmask;
                const u32 r = (rank2[i >> 1] >> ((i & 1) * 16)) & 0xffffu;
                const u32 wo = (sm.wh[warp][d >> 1] >> ((d & 1) * 16)) & 0xffffu;
                stage[sm.dstart[d] + wo + r] = k;
            }
        }
        __syncthreads();  // (E)
        for (u32 j = t; j < tile_n; j += kPT) {
            const u64 k = stage[j];
            out[sm.gbase[(u32)(k >> shift) & dmask] + j] = k;
        }
        cur ^= 1;
    }
}

}  // namespace

// Keys per thread of a onesweep tile (4/8/16 are compiled;
// gd_device_config.sort_items, 16 by default: measured on B200 fastest from
// 64K to 16M keys).
template <typename K>
int sort_items(const Ctx& c) {
    int i = (int)c.cfg.sort_items;
    if (sizeof(K) > 8) i = std::min(i, 8);
    return i == 16 || i == 8 ? i : 4;
}

// Mean distinct pass digits per 32 consecutive keys, over warps spread
// evenly across the array: out += the number of peer groups of each warp.
template <typename K>
__global__ void digit_diversity_kernel(const K* __restrict__ keys, u64 n, u32 shift,
                                       unsigned long long* __restrict__ out) {
    const u64 warp = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const u64 nw = ((u64)gridDim.x * blockDim.x) >> 5;
    const u64 base = n > 32 ? (n - 32) * warp / nw : 0;
    const u64 i = base + lane_id();
    const u32 d = i < n ? digit_of(keys[i], shift) : (u32)kRadix;
    const u32 peers = __match_any_sync(0xffffffffu, d);
    const bool leader = lane_id() == 31 - __clz(peers);
    const u32 groups = __popc(__ballot_sync(0xffffffffu, leader));
    if (lane_id() == 0) atomicAdd(out, (unsigned long long)groups);
}

template <typename K, int I>
void launch_onesweep(const Ctx& c, u64 tiles, const K* src, K* dst, u64 pb, u64 pn, u32 shift, const u64* rd,
                     u64* wr, u32* w, bool ballot) {
    const bool four = c.cfg.sort_min_ctas == 4;  // 64 registers: 4 CTAs per SM
    if (ballot && four)
        onesweep_kernel<K, I, true, 4><<<(unsigned)tiles, kSortThreads, 0, c.stream>>>(src, dst, pb, pn, shift, rd,
                                                                                       wr, w, (u32)tiles);
    else if (ballot)
        onesweep_kernel<K, I, true><<<(unsigned)tiles, kSortThreads, 0, c.stream>>>(src, dst, pb, pn, shift, rd, wr,
                                                                                    w, (u32)tiles);
    else if (four)
        onesweep_kernel<K, I, false, 4><<<(unsigned)tiles, kSortThreads, 0, c.stream>>>(src, dst, pb, pn, shift, rd,
                                                                                        wr, w, (u32)tiles);
    else
        onesweep_kernel<K, I><<<(unsigned)tiles, kSortThreads, 0, c.stream>>>(src, dst, pb, pn, shift, rd, wr, w,
                                                                              (u32)tiles);
}

// All passes' digit histograms for the pipelined sort: `width`-bit digits,
// R bins per pass (warp-privatized copies as in radix_hist_kernel).
__global__ void __launch_bounds__(256) radix_hist_w_kernel(const u64* __restrict__ keys, u64 n, int npass,
                                                           u32 width, u32 nbits, int R, int copies,
                                                           u64* __restrict__ hist) {
    extern __shared__ u32 sh[];
    const int words = npass * R;
    for (int i = threadIdx.x; i < copies * words; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    u32* mine = sh + ((threadIdx.x >> 5) % copies) * words;
    const u32 dmask = (1u << width) - 1;
    constexpr int kU = 4;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i0 = (u64)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += kU * stride) {
        u64 k[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const u64 i = i0 + u * stride;
            k[u] = i < n ? __ldcs(keys + i) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (i0 + u * stride < n)
                for (int p = 0; p < npass; ++p) {
                    const u32 sh = p * width;
                    const u32 m = sh + width <= nbits ? dmask : (1u << (nbits - sh)) - 1;  // last pass: narrower
                    atomicAdd(&mine[p * R + ((u32)(k[u] >> sh) & m)], 1u);
                }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < words; i += blockDim.x) {
        u32 t = 0;
        for (int c = 0; c < copies; ++c) t += sh[c * words + i];
        if (t) atomicAdd(&hist[i], (u64)t);
    }
}

template <int R>
__global__ void __launch_bounds__(R) radix_bases_w_kernel(const u64* __restrict__ hist, u64* __restrict__ bases) {
    __shared__ u64 scan_tmp[R / 32 + 1];
    const int pass = blockIdx.x;
    u64 all;
    bases[pass * R + threadIdx.x] = block_exclusive_scan<u64, R>(hist[pass * R + threadIdx.x], all, scan_tmp);
}

template <int RB, bool IP, bool BALLOT>
void launch_pipe_ip(Ctx& c, const u64* src, u64* dst, u64 pb, u64 pn, u32 shift, u32 width, const u64* rd, u64* wr,
                    u32* w) {
    const size_t smem = sizeof(PipeSmem<RB, IP>);
    auto kern = onesweep_pipe_kernel<RB, IP, BALLOT>;
    static int per_sm = -1;  // co-resident CTAs per SM (one device per process)
    if (per_sm < 0) {
        GD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPT, smem));
        if (per_sm < 1) throw Error(GD_ERR_CUDA, "onesweep_pipe_kernel does not fit an SM");
    }
    const u64 tiles = (pn + kPTile - 1) / kPTile;
    const u64 grid = std::min<u64>(tiles, (u64)per_sm * c.num_sms);
    // cooperative launch: the static round-robin tile order needs every CTA
    // of the grid co-resident (the driver guarantees it or fails the launch)
    u32 nt = (u32)tiles;
    void* args[] = {(void*)&src, (void*)&dst, (void*)&pb, (void*)&pn, (void*)&shift, (void*)&width, (void*)&rd,
                    (void*)&wr, (void*)&w, (void*)&nt};
    GD_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)grid), dim3(kPT), args, smem, c.stream));
}

template <int RB>
void launch_pipe(Ctx& c, const u64* src, u64* dst, u64 pb, u64 pn, u32 shift, u32 width, const u64* rd, u64* wr,
                 u32* w) {
    switch (c.cfg.sort_pipeline) {
        case 2: launch_pipe_ip<RB, false, true>(c, src, dst, pb, pn, shift, width, rd, wr, w); break;
        case 3: launch_pipe_ip<RB, true, false>(c, src, dst, pb, pn, shift, width, rd, wr, w); break;
        default: launch_pipe_ip<RB, true, true>(c, src, dst, pb, pn, shift, width, rd, wr, w);
    }
}

// Pipelined LSD sort of u64 keys (gd_device_config.sort_digit_bits > 8 or
// sort_pipeline): npass = ceil(nbits / max_bits) passes of equal width.
u64* radix_sort_pipe(Ctx& c, u64* a, u64* b, u64 n, u32 nbits) {
    const u32 maxb = std::min<u32>(10, std::max<u32>(8, c.cfg.sort_digit_bits));
    const int npass = (int)((nbits + maxb - 1) / maxb);
    const u32 width = (nbits + npass - 1) / npass;
    const int RB = width <= 8 ? 8 : width == 9 ? 9 : 10;
    const int R = 1 << RB;
    const int nportions = (int)((n + kPortion - 1) / kPortion);
    const u64 hist_words = (u64)npass * R;
    DevBuf<u64> hist(c, hist_words);
    DevBuf<u64> bases(c, hist_words + 2 * R);
    c.memset(hist.p, 0, hist_words * sizeof(u64));
    {
        const int grid = (int)std::min<u64>((u64)c.num_sms * 4, (n + 255) / 256);
        cudaEvent_t t = c.prof_begin();
        const int copies = hist_words * 4 * 2 <= 48 * 1024 ? 2 : 1;
        radix_hist_w_kernel<<<grid, 256, (size_t)copies * hist_words * sizeof(u32), c.stream>>>(a, n, npass, width, nbits,
                                                                                                R, copies, hist.p);
        c.check_launch();
        c.prof_end(t, KC_SORT_HIST, n * sizeof(u64));
    }
    if (R == 256) radix_bases_w_kernel<256><<<npass, 256, 0, c.stream>>>(hist.p, bases.p);
    else if (R == 512) radix_bases_w_kernel<512><<<npass, 512, 0, c.stream>>>(hist.p, bases.p);
    else radix_bases_w_kernel<1024><<<npass, 1024, 0, c.stream>>>(hist.p, bases.p);
    c.check_launch();
    u64* pp[2] = {bases.p + hist_words, bases.p + hist_words + R};
    const u64 max_tiles = (std::min(n, kPortion) + kPTile - 1) / kPTile;
    const u64 ws_words = 4 + max_tiles * R;
    DevBuf<u32> ws(c, ws_words);
    u64* src = a;
    u64* dst = b;
    for (int pass = 0; pass < npass; ++pass) {
        const u32 shift = (u32)pass * width;
        const u32 wd = std::min<u32>(width, nbits - shift);
        for (int p = 0; p < nportions; ++p) {
            const u64 pb = (u64)p * kPortion;
            const u64 pn = std::min(kPortion, n - pb);
            const u64 tiles = (pn + kPTile - 1) / kPTile;
            c.memset(ws.p, 0, (4 + tiles * R) * sizeof(u32));
            const u64* rd = p == 0 ? bases.p + (u64)pass * R : pp[(p - 1) & 1];
            u64* wr = p + 1 < nportions ? pp[p & 1] : nullptr;
            cudaEvent_t t = c.prof_begin();
            if (RB == 8) launch_pipe<8>(c, src, dst, pb, pn, shift, wd, rd, wr, ws.p);
            else if (RB == 9) launch_pipe<9>(c, src, dst, pb, pn, shift, wd, rd, wr, ws.p);
            else launch_pipe<10>(c, src, dst, pb, pn, shift, wd, rd, wr, ws.p);
            c.check_launch();
            c.prof_end(t, KC_SORT_PASS, 2 * pn * sizeof(u64));
        }
        std::swap(src, dst);
    }
    return src;
}

template <typename K>
K* radix_sort_passes(Ctx& c, K* a, K* b, u64 n, u32 nbits, u32 pass_lo, u32 pass_hi, std::vector<char>* ballot_io,
                     std::vector<u64>* top_hist) {
    if (n <= 1 || nbits == 0) return a;
    const bool whole = pass_lo == 0 && pass_hi == ~0u && !ballot_io && !top_hist;
    if constexpr (sizeof(K) == 8) {
        if (whole && c.cfg.sort_pipeline && c.cfg.sort_pipeline != 4 && n >= c.cfg.sort_pipeline_min_keys)
            return reinterpret_cast<K*>(radix_sort_pipe(c, reinterpret_cast<u64*>(a), reinterpret_cast<u64*>(b), n,
                                                        nbits));
    }
    const int npass = (int)((nbits + kRadixBits - 1) / kRadixBits);
    const int p_lo = (int)std::min<u32>(pass_lo, (u32)npass), p_hi = (int)std::min<u32>(pass_hi, (u32)npass);
    const int nportions = (int)((n + kPortion - 1) / kPortion);
    const int items = sort_items<K>(c);
    const u64 TILE = (u64)kSortThreads * items;

    const u64 hist_words = (u64)npass * kRadix;
    DevBuf<u64> hist(c, hist_words);
    DevBuf<u64> bases(c, hist_words + 2 * kRadix);  // + two portion ping-pong rows
    c.memset(hist.p, 0, hist_words * sizeof(u64));
    {
        const int grid = (int)std::min<u64>((u64)c.num_sms * 4, (n + 255) / 256);
        cudaEvent_t t = c.prof_begin();
        const int copies = npass <= 8 ? 4 : 2;
        radix_hist_kernel<K><<<grid, 256, (size_t)copies * npass * kRadix * sizeof(u32), c.stream>>>(
            a, 0, n, npass, copies, hist.p);
        c.check_launch();
        c.prof_end(t, KC_SORT_HIST, n * sizeof(K));
    }
    radix_bases_kernel<<<npass, kRadix, 0, c.stream>>>(hist.p, bases.p);
    c.check_launch();
    u64* pp[2] = {bases.p + hist_words, bases.p + hist_words + kRadix};
    if (top_hist && p_hi > 0) {  // digit counts of the last requested pass
        top_hist->assign(kRadix, 0);
        c.d2h(top_hist->data(), hist.p + (u64)(p_hi - 1) * kRadix, kRadix * sizeof(u64));
        c.sync();
    }

    const u64 max_tiles = (std::min(n, kPortion) + TILE - 1) / TILE;
    const u64 ws_words = 1 + max_tiles * kRadix;
    // One look-back workspace per pass, cleared by a single memset, when
    // the keys fit one portion and all passes' workspaces stay small
    // (<= 16 MB); otherwise one workspace is reused and cleared before every
    // launch (bounded memory next to a large sort).
    const bool single = nportions == 1 && ws_words * (u64)npass * sizeof(u32) <= (16ull << 20);
    DevBuf<u32> ws(c, single ? ws_words * npass : ws_words);
    if (single) c.memset(ws.p, 0, ws_words * npass * sizeof(u32));
    K* src = a;
    K* dst = b;
    // Ranking per pass: ballot multi-split where the pass's digits are spread
    // (9 ballots, fixed cost) where a warp's 32 consecutive keys carry many
    // distinct digits, MATCH.ANY (cost grows with the distinct count) where
    // they carry few.  The count depends on the pass's input ORDER (C2: the
    // log keeps a Δ row's outputs together, so the low passes see few
    // distinct digits per warp; the src passes after them see many), so it
    // is sampled on the pass's actual input right before the pass: 2048
    // warps of consecutive keys, one readback per pass.  C2: ballot on
    // passes 3-4 only, final sort 34.2 -> ~30 ms (profiles/r2_sort_passes.md).
    // ballot_io: decisions given by the caller (sized npass), or empty: sample
    // every pass (from 1 M keys) and hand the decisions back — the segments
    // of a segmented sort sample once, on their first segment.
    std::vector<char> ballot(npass, 0);
    const bool given = ballot_io && (int)ballot_io->size() == npass;
    const u64 adapt_min = ballot_io ? (1ull << 20) : c.cfg.sort_pipeline_min_keys * 16;
    const bool adapt = !given && c.cfg.sort_ballot && n >= adapt_min && c.cfg.sort_pipeline == 0;
    DevBuf<unsigned long long> div;
    if (adapt) div = DevBuf<unsigned long long>(c, 1);
    for (int pass = p_lo; pass < p_hi; ++pass) {
        bool use_ballot = given ? (*ballot_io)[pass] != 0 : c.cfg.sort_pipeline == 4;
        if (adapt) {
            constexpr int kSampleWarps = 2048;
            c.memset(div.p, 0, sizeof(unsigned long long));
            digit_diversity_kernel<K><<<kSampleWarps / 8, 256, 0, c.stream>>>(src, n, (u32)(pass * kRadixBits), div.p);
            c.check_launch();
            unsigned long long tot = 0;
            c.read_words(&tot, div.p, 1);
            use_ballot = tot >= (unsigned long long)c.cfg.sort_ballot * kSampleWarps;  // mean distinct digits
            if (c.cfg.trace & 4)
                fprintf(stderr, "[sort] pass %d: %.1f distinct digits per warp -> %s\n", pass,
                        (double)tot / kSampleWarps, use_ballot ? "ballot" : "match");
        }
        ballot[pass] = use_ballot;
        for (int p = 0; p < nportions; ++p) {
            const u64 pb = (u64)p * kPortion;
            const u64 pn = std::min(kPortion, n - pb);
            const u64 tiles = (pn + TILE - 1) / TILE;
            u32* w = single ? ws.p + (u64)pass * ws_words : ws.p;
            if (!single) c.memset(w, 0, (1 + tiles * kRadix) * sizeof(u32));
            const u64* rd = p == 0 ? bases.p + (u64)pass * kRadix : pp[(p - 1) & 1];
            u64* wr = p + 1 < nportions ? pp[p & 1] : nullptr;
            cudaEvent_t t = c.prof_begin();
            const u32 shift = (u32)(pass * kRadixBits);
            if (items == 16) launch_onesweep<K, (sizeof(K) > 8 ? 8 : 16)>(c, tiles, src, dst, pb, pn, shift, rd, wr, w, ballot[pass]);
            else if (items == 8) launch_onesweep<K, 8>(c, tiles, src, dst, pb, pn, shift, rd, wr, w, ballot[pass]);
            else launch_onesweep<K, 4>(c, tiles, src, dst, pb, pn, shift, rd, wr, w, ballot[pass]);
            c.check_launch();
            c.prof_end(t, KC_SORT_PASS, 2 * pn * sizeof(K));
        }
        std::swap(src, dst);
    }
    if (ballot_io && !given) *ballot_io = ballot;
    return src;
}

template <typename K>
K* radix_sort(Ctx& c, K* a, K* b, u64 n, u32 nbits) {
    return radix_sort_passes<K>(c, a, b, n, nbits, 0, ~0u, nullptr, nullptr);
}

template u64* radix_sort<u64>(Ctx&, u64*, u64*, u64, u32);
template u64* radix_sort_passes<u64>(Ctx&, u64*, u64*, u64, u32, u32, u32, std::vector<char>*, std::vector<u64>*);
template u128* radix_sort<u128>(Ctx&, u128*, u128*, u64, u32);

}  // namespace gd
