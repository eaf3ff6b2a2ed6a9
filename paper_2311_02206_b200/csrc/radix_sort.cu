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

template <typename K, int I>
__global__ void __launch_bounds__(kSortThreads) onesweep_kernel(
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
    for (int i = 0; i < I; ++i) pm[i] = __match_any_sync(0xffffffffu, dig(i));
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
        constexpr int kLookWindow = 16;
        long long pred = (long long)tile - 1;
        while (true) {
            u32 s[kLookWindow];
#pragma unroll
            for (int w = 0; w < kLookWindow; ++w)
                s[w] = pred - w >= 0 ? ld_relaxed32(status + (u64)(pred - w) * kRadix + t) : kSFlagP;
            int first_inv = kLookWindow, first_p = kLookWindow;
#pragma unroll
            for (int w = kLookWindow - 1; w >= 0; --w) {
                const u32 f = s[w] >> 30;
                if (f == 0) first_inv = w;
                if (f == 2) first_p = w;
            }
            if (first_inv < first_p) {  // an unpublished tile before any prefix: wait on it
#pragma unroll
                for (int w = 0; w < kLookWindow; ++w)
                    if (w < first_inv) excl += s[w] & kSMask;
                pred -= first_inv;
                continue;
            }
#pragma unroll
            for (int w = 0; w < kLookWindow; ++w)
                if (w <= first_p) excl += s[w] & kSMask;
            if (first_p < kLookWindow) break;
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

template <typename K, int I>
void launch_onesweep(const Ctx& c, u64 tiles, const K* src, K* dst, u64 pb, u64 pn, u32 shift, const u64* rd,
                     u64* wr, u32* w) {
    onesweep_kernel<K, I><<<(unsigned)tiles, kSortThreads, 0, c.stream>>>(src, dst, pb, pn, shift, rd, wr, w,
                                                                          (u32)tiles);
}

template <typename K>
K* radix_sort(Ctx& c, K* a, K* b, u64 n, u32 nbits) {
    if (n <= 1 || nbits == 0) return a;
    const int npass = (int)((nbits + kRadixBits - 1) / kRadixBits);
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
    for (int pass = 0; pass < npass; ++pass) {
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
            if (items == 16) launch_onesweep<K, (sizeof(K) > 8 ? 8 : 16)>(c, tiles, src, dst, pb, pn, shift, rd, wr, w);
            else if (items == 8) launch_onesweep<K, 8>(c, tiles, src, dst, pb, pn, shift, rd, wr, w);
            else launch_onesweep<K, 4>(c, tiles, src, dst, pb, pn, shift, rd, wr, w);
            c.check_launch();
            c.prof_end(t, KC_SORT_PASS, 2 * pn * sizeof(K));
        }
        std::swap(src, dst);
    }
    return src;
}

template u64* radix_sort<u64>(Ctx&, u64*, u64*, u64, u32);
template u128* radix_sort<u128>(Ctx&, u128*, u128*, u64, u32);

}  // namespace gd
