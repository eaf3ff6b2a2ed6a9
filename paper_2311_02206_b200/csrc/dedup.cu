// dedup.cu — hash pre-dedup of an iteration's join rows for the host-driven
// loop (engine.cu dedup_diff_merge), the dedup half of canonicalize
// (tuple_array.hpp:73-133) when the join output is mostly duplicates
// (CSPA's ValueAlias: 5.4e9 join rows for 3.3e8 distinct ones).  Every row
// CASes its key into an open-addressing set sized from the previous
// iteration's distinct count; first inserters append the key (one atomic per
// CTA tile), so only the distinct rows reach the radix sort.  When the set
// would pass load 1/2 the pass reports overflow and the caller sorts all rows.
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

}  // namespace

u64 hash_dedup(Ctx& c, const u64* keys, u64 m, u64 expect_unique, u64* out, u64 out_cap) {
    u64 cap = 1024;
    while (cap < 2 * expect_unique) cap <<= 1;
    const u64 limit = std::min<u64>(cap / 2, out_cap);
    DevBuf<u64> tab(c, cap);
    c.memset(tab.p, 0xff, cap * sizeof(u64));
    DevBuf<unsigned long long> cnt(c, 1);
    c.memset(cnt.p, 0, sizeof(unsigned long long));
    const int grid = (int)std::max<u64>(1, std::min<u64>((m + kDT * kDPer - 1) / (kDT * kDPer), (u64)c.num_sms * 8));
    cudaEvent_t t = c.prof_begin();
    dedup_insert_kernel<<<grid, kDT, 0, c.stream>>>(keys, m, tab.p, cap - 1, out, limit, cnt.p);
    c.check_launch();
    c.prof_end(t, KC_SELECT, m * 16);
    unsigned long long n;
    c.read_words(&n, cnt.p, 1);
    return n <= limit ? n : ~0ull;
}

}  // namespace gd
