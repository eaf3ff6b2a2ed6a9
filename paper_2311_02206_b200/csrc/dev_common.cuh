// dev_common.cuh — shared device types and primitives for the sm_100a
// GDlog hot path: key types, bit-packed tuple layout, warp/block scans and
// the decoupled look-back used by every single-pass kernel.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace gd {

using u32 = uint32_t;
using u64 = unsigned long long;
using u128 = unsigned __int128;

constexpr int kSms = 148;  // B200 (2 dies x 74 SMs)

// ---------------------------------------------------------------------
// Bit-packed tuple layout.  A tuple of arity k whose encoded
// column values are < 2^bits is stored as one integer key K (u64 or u128):
//   key = sum_c col_c << ((k - 1 - c) * bits)
// so unsigned integer order of keys == lexicographic row order
// (compare_rows, tuple_array.hpp:55-61).  Encoded values are never the
// all-ones pattern of `bits` bits, so no prefix of a key is all-ones.
struct Layout {
    u32 arity;
    u32 bits;
};

struct Perm8 {
    u32 p[8];
};

template <typename K>
__host__ __device__ __forceinline__ u64 col_of(K key, u32 arity, u32 bits, u32 c) {
    const u32 shift = (arity - 1 - c) * bits;
    const u64 mask = bits >= 64 ? ~0ull : ((1ull << bits) - 1);
    return (u64)(key >> shift) & mask;
}

template <typename K>
__host__ __device__ __forceinline__ K prefix_of(K key, u32 arity, u32 bits, u32 plen) {
    const u32 shift = (arity - plen) * bits;
    return shift >= sizeof(K) * 8 ? K(0) : (K)(key >> shift);
}

// Murmur3 finalizer (hash.hpp:13-20); also used for slot placement.
__host__ __device__ __forceinline__ u64 fmix64(u64 k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdULL;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ULL;
    k ^= k >> 33;
    return k;
}

template <typename K>
__host__ __device__ __forceinline__ u64 key_hash64(K k);
template <>
__host__ __device__ __forceinline__ u64 key_hash64<u64>(u64 k) { return fmix64(k); }
template <>
__host__ __device__ __forceinline__ u64 key_hash64<u128>(u128 k) {
    return fmix64((u64)k ^ fmix64((u64)(k >> 64) + 0x9e3779b97f4a7c15ull));
}

// ---------------------------------------------------------------------
// Warp / block primitives.

__device__ __forceinline__ u32 lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ u32 lanemask_lt() {
    u32 m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T n = __shfl_up_sync(0xffffffffu, v, o);
        if ((int)lane_id() >= o) v += n;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide exclusive scan; `smem` needs THREADS/32 + 1 entries.  Returns
// the exclusive prefix of the calling thread and the block total.
template <typename T, int THREADS>
__device__ __forceinline__ T block_exclusive_scan(T v, T& total, T* smem) {
    constexpr int W = THREADS / 32;
    const u32 warp = threadIdx.x >> 5;
    T inc = warp_inclusive_scan(v);
    if (lane_id() == 31) smem[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T w = lane_id() < W ? smem[lane_id()] : T(0);
        T wi = warp_inclusive_scan(w);
        if (lane_id() < W) smem[lane_id()] = wi - w;
        if (lane_id() == W - 1) smem[W] = wi;
    }
    __syncthreads();
    T excl = inc - v + smem[warp];
    total = smem[W];
    __syncthreads();
    return excl;
}

// ---------------------------------------------------------------------
// Relaxed GPU-scope loads/stores for look-back status words.

__device__ __forceinline__ u64 ld_relaxed(const u64* p) {
    u64 v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(u64* p, u64 v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u32 ld_relaxed32(const u32* p) {
    u32 v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed32(u32* p, u32 v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Decoupled look-back over 64-bit tile statuses: bits 63..62 hold the flag
// (1 = aggregate, 2 = inclusive prefix), bits 61..0 the value.  Called by
// the whole of warp 0; returns the exclusive prefix of `tile` (all lanes).
// Tiles must be claimed in launch order (claim_tile) so predecessors are
// resident or done: no deadlock.
constexpr u64 kFlagA = 1ull << 62;
constexpr u64 kFlagP = 2ull << 62;
constexpr u64 kValMask = (1ull << 62) - 1;

__device__ __forceinline__ u64 warp_lookback(u64* status, u64 tile, u64 aggregate) {
    const u32 lane = lane_id();
    if (tile == 0) {
        if (lane == 0) st_relaxed(status, kFlagP | aggregate);
        return 0;
    }
    if (lane == 0) st_relaxed(status + tile, kFlagA | aggregate);
    u64 excl = 0;
    long long pred = (long long)tile - 1;
    while (true) {
        const long long idx = pred - (long long)lane;
        u64 s = idx >= 0 ? ld_relaxed(status + idx) : kFlagP;
        const u32 flag = (u32)(s >> 62);
        if (__any_sync(0xffffffffu, flag == 0)) continue;  // spin on this window
        const u32 pmask = __ballot_sync(0xffffffffu, flag == 2);
        u64 v = s & kValMask;
        if (pmask) {
            const u32 first = __ffs(pmask) - 1;
            if (lane > first) v = 0;
            excl += warp_sum(v);
            break;
        }
        excl += warp_sum(v);
        pred -= 32;
    }
    if (lane == 0) st_relaxed(status + tile, kFlagP | (excl + aggregate));
    return excl;
}

// Workspace header of a look-back launch: [0] tile counter, [1..] statuses.
__device__ __forceinline__ u64 claim_tile(u64* ws, u64* smem_slot) {
    if (threadIdx.x == 0) *smem_slot = atomicAdd(ws, 1ull);
    __syncthreads();
    return *smem_slot;
}

}  // namespace gd
