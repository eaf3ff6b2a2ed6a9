// dedup.cu — hash pre-dedup of an iteration's join rows for the host-driven
// loop (engine.cu dedup_diff_merge), the dedup half of canonicalize
// (tuple_array.hpp:73-133) when the join output is mostly duplicates
// (CSPA's ValueAlias: 5.4e9 join rows for 3.3e8 distinct ones).  Every row
// CASes its key into an open-addressing set sized from the previous
// iteration's distinct count; first inserters append the key (one atomic per
// CTA tile), so only the distinct rows reach the radix sort.  When the set
// would pass load 1/2 the pass reports overflow and the caller sorts all rows.
#include <vector>

#include "dev_common.cuh"
#include "ops.h"

namespace gd {

namespace {

constexpr int kDT = 256, kDPer = 8;
constexpr u32 kMaxProbes = 256;  // longer runs only happen far above load 1/2

__global__ void __launch_bounds__(kDT) dedup_insert_kernel(const u64* __restrict__ keys, u64 m, u64* __restrict__ tab,
                                                           u64 mask, u64* __restrict__ out, u64 limit,
                                                           unsigned long long* counter) {
    __shared__ u32 s_warp[kDT / 32];
    __shared__ unsigned long long s_base;
    constexpr u64 kChunk = (u64)kDT * kDPer;
    for (u64 base = (u64)blockIdx.x * kChunk; base < m; base += (u64)gridDim.x * kChunk) {
        u64 key[kDPer], old[kDPer];
#pragma unroll
        for (int k = 0; k < kDPer; ++k) {
            const u64 j = base + (u64)k * kDT + threadIdx.x;
            key[k] = j < m ? __ldcs(keys + j) : kEmptySlot;
        }
        // load first, CAS only empty slots (duplicates — most rows here —
        // never issue an atomic; the CAS hits the loaded line in L2)
#pragma unroll
        for (int k = 0; k < kDPer; ++k)
            old[k] = key[k] != kEmptySlot ? __ldcg(&tab[fmix64(key[k]) & mask]) : key[k];
#pragma unroll
        for (int k = 0; k < kDPer; ++k)
            if (key[k] != kEmptySlot && old[k] == kEmptySlot)
                old[k] = atomicCAS(&tab[fmix64(key[k]) & mask], kEmptySlot, key[k]);
        u32 fresh = 0;
#pragma unroll
        for (int k = 0; k < kDPer; ++k) {
            if (key[k] == kEmptySlot) continue;
            u64 o = old[k], p = fmix64(key[k]) & mask;
            u32 probes = 0;
            while (o != kEmptySlot && o != key[k]) {  // linear probing
                if (++probes > kMaxProbes) {          // set (nearly) full: report overflow
                    atomicExch(counter, ~0ull >> 1);
                    break;
                }
                p = (p + 1) & mask;
                o = atomicCAS(&tab[p], kEmptySlot, key[k]);
            }
            fresh |= (u32)(o == kEmptySlot) << k;
        }
        // CTA append: warp ballots, one atomic per tile
        u32 mk[kDPer], tot = 0;
#pragma unroll
        for (int k = 0; k < kDPer; ++k) {
            mk[k] = __ballot_sync(0xffffffffu, fresh >> k & 1);
            tot += __popc(mk[k]);
        }
        const u32 warp = threadIdx.x >> 5;
        if (lane_id() == 0) s_warp[warp] = tot;
        __syncthreads();
        if (threadIdx.x == 0) {
            u32 all = 0;
            for (int w = 0; w < kDT / 32; ++w) {
                const u32 c = s_warp[w];
                s_warp[w] = all;
                all += c;
            }
            s_base = all ? atomicAdd(counter, (unsigned long long)all) : 0;
        }
        __syncthreads();
        u64 pos = s_base + s_warp[warp];
        const u32 lt = lanemask_lt();
#pragma unroll
        for (int k = 0; k < kDPer; ++k) {
            if ((fresh >> k & 1) && pos + __popc(mk[k] & lt) < limit) out[pos + __popc(mk[k] & lt)] = key[k];
            pos += __popc(mk[k]);
        }
        __syncthreads();
    }
}

// Partition pass: part(key) = top `bits` bits of fmix64(key) (the set's
// slot uses the low bits, so parts and slots are independent).  Count per
// part, then scatter with one reserved range per (CTA tile, part).
constexpr u32 kPartTile = 2048, kMaxParts = 1024;

__global__ void part_count_kernel(const u64* __restrict__ keys, u64 m, u32 bits, unsigned long long* counts) {
    __shared__ u32 sc[kMaxParts];
    const u32 P = 1u << bits;
    for (u32 i = threadIdx.x; i < P; i += blockDim.x) sc[i] = 0;
    __syncthreads();
    // four independent loads in flight per thread
    constexpr int kU = 4;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i0 = (u64)blockIdx.x * blockDim.x + threadIdx.x; i0 < m; i0 += kU * stride) {
        u64 k[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) k[u] = i0 + u * stride < m ? __ldcs(keys + i0 + u * stride) : 0;
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (i0 + u * stride < m) atomicAdd(&sc[fmix64(k[u]) >> (64 - bits)], 1u);
    }
    __syncthreads();
    for (u32 i = threadIdx.x; i < P; i += blockDim.x)
        if (sc[i]) atomicAdd(&counts[i], (unsigned long long)sc[i]);
}

__global__ void part_scatter_kernel(const u64* __restrict__ keys, u64 m, u32 bits,
                                    const unsigned long long* __restrict__ offsets, unsigned long long* cursors,
                                    u64* __restrict__ out) {
    __shared__ u32 sc[kMaxParts];
    __shared__ unsigned long long sb[kMaxParts];
    const u32 P = 1u << bits;
    constexpr u32 kPerT = kPartTile / 256;
    for (u64 t0 = (u64)blockIdx.x * kPartTile; t0 < m; t0 += (u64)gridDim.x * kPartTile) {
        for (u32 i = threadIdx.x; i < P; i += blockDim.x) sc[i] = 0;
        __syncthreads();
        u64 k[kPerT];
        u32 part[kPerT], rank[kPerT];
#pragma unroll
        for (u32 q = 0; q < kPerT; ++q) {
            const u64 i = t0 + q * 256 + threadIdx.x;
            part[q] = kMaxParts;
            if (i < m) {
                k[q] = __ldcs(keys + i);
                part[q] = (u32)(fmix64(k[q]) >> (64 - bits));
                rank[q] = atomicAdd(&sc[part[q]], 1u);
            }
        }
        __syncthreads();
        for (u32 i = threadIdx.x; i < P; i += blockDim.x)
            sb[i] = sc[i] ? offsets[i] + atomicAdd(&cursors[i], (unsigned long long)sc[i]) : 0;
        __syncthreads();
#pragma unroll
        for (u32 q = 0; q < kPerT; ++q)
            if (part[q] < kMaxParts) out[sb[part[q]] + rank[q]] = k[q];
        __syncthreads();
    }
}

}  // namespace

// Sets larger than kL2Slots are split: the rows are partitioned by hash
// (one streaming pass) and every part is deduplicated in the same
// L2-resident set of kL2Slots (64 MB), cleared between parts, so the probes
// hit L2 instead of random HBM lines.

u64 hash_dedup(Ctx& c, const u64* keys, u64 m, u64 expect_unique, u64* out, u64 out_cap) {
    // dedup_part_slots (power of two; tests shrink it)
    const u64 kL2Slots = c.cfg.dedup_part_slots;
    u64 cap = 1024;
    while (cap < 2 * expect_unique) cap <<= 1;
    DevBuf<unsigned long long> cnt(c, 1);
    c.memset(cnt.p, 0, sizeof(unsigned long long));
    const bool split = cap > kL2Slots && c.cfg.dedup_split;
    const u64 tcap = split ? kL2Slots : cap;
    DevBuf<u64> tab(c, tcap);
    auto run = [&](const u64* k, u64 n, u64 limit) {
        const int grid =
            (int)std::max<u64>(1, std::min<u64>((n + kDT * kDPer - 1) / (kDT * kDPer), (u64)c.num_sms * 8));
        c.memset(tab.p, 0xff, tcap * sizeof(u64));
        dedup_insert_kernel<<<grid, kDT, 0, c.stream>>>(k, n, tab.p, tcap - 1, out, limit, cnt.p);
        c.check_launch();
    };
    cudaEvent_t t = c.prof_begin();
    if (!split) {
        run(keys, m, std::min<u64>(cap / 2, out_cap));
    } else {
        u32 bits = 0;
        while ((cap >> bits) > kL2Slots) ++bits;
        const u32 P = 1u << bits;
        if (P > kMaxParts) return ~0ull;
        DevBuf<unsigned long long> counts(c, P), offs(c, P), cursors(c, P);
        c.memset(counts.p, 0, P * sizeof(unsigned long long));
        c.memset(cursors.p, 0, P * sizeof(unsigned long long));
        const int g = (int)std::max<u64>(1, std::min<u64>((m + 255) / 256, (u64)c.num_sms * 8));
        part_count_kernel<<<g, 256, 0, c.stream>>>(keys, m, bits, counts.p);
        c.check_launch();
        std::vector<unsigned long long> hc(P), ho(P);
        c.d2h(hc.data(), counts.p, P * sizeof(unsigned long long));
        c.sync();
        u64 acc = 0;
        for (u32 i = 0; i < P; ++i) {
            ho[i] = acc;
            acc += hc[i];
        }
        c.h2d(offs.p, ho.data(), P * sizeof(unsigned long long));
        DevBuf<u64> parted(c, std::max<u64>(m, 1));
        part_scatter_kernel<<<g, 256, 0, c.stream>>>(keys, m, bits, offs.p, cursors.p, parted.p);
        c.check_launch();
        // out stays a prefix: each part appends after the previous parts'
        // distinct keys (limit = out_cap overall, set load checked per part)
        for (u32 i = 0; i < P; ++i)
            if (hc[i]) run(parted.p + ho[i], hc[i], out_cap);
    }
    c.prof_end(t, KC_SELECT, m * 16);
    unsigned long long n;
    c.read_words(&n, cnt.p, 1);
    return n <= out_cap && (split || n <= cap / 2) ? n : ~0ull;
}

}  // namespace gd
