// select.cuh — single-pass, order-preserving stream compaction (decoupled
// look-back).  Used for adjacent-unique (tuple_array.hpp:124-131), group
// starts (index_map.hpp:46-66), filter compaction (ra.hpp:244-262 with
// filters) and select_project (ra.hpp:267-293).
#pragma once

#include "dev_common.cuh"
#include "ctx.h"

namespace gd {

constexpr int kSelThreads = 256;
constexpr int kSelItems = 8;
constexpr u64 kSelTile = (u64)kSelThreads * kSelItems;

// ws: [0] tile counter, [1] total selected, [2..] tile statuses.
template <typename Pred, typename Emit>
__global__ void __launch_bounds__(kSelThreads) select_kernel(u64 n, Pred pred, Emit emit, u64* ws) {
    __shared__ u64 s_tile;
    __shared__ u64 s_scan[kSelThreads / 32 + 1];
    __shared__ u64 s_base;
    const u64 tile = claim_tile(ws, &s_tile);
    const u64 begin = tile * kSelTile + (u64)threadIdx.x * kSelItems;
    bool f[kSelItems];
    u64 cnt = 0;
#pragma unroll
    for (int j = 0; j < kSelItems; ++j) {
        const u64 idx = begin + j;
        f[j] = idx < n && pred(idx);
        cnt += f[j];
    }
    u64 total;
    const u64 excl = block_exclusive_scan<u64, kSelThreads>(cnt, total, s_scan);
    if (threadIdx.x < 32) {
        const u64 base = warp_lookback(ws + 2, tile, total);
        if (threadIdx.x == 0) {
            s_base = base;
            atomicAdd(ws + 1, total);
        }
    }
    __syncthreads();
    u64 pos = s_base + excl;
#pragma unroll
    for (int j = 0; j < kSelItems; ++j)
        if (f[j]) emit(begin + j, pos++);
}

// Launches the compaction without reading the count back; the selected
// total lands in ws.p[1] (n == 0: ws holds a zero).
template <typename Pred, typename Emit>
void run_select_async(Ctx& c, u64 n, Pred pred, Emit emit, DevBuf<u64>& ws) {
    const u64 tiles = (n + kSelTile - 1) / kSelTile;
    ws.reserve_discard(c, 2 + tiles);
    c.memset(ws.p, 0, (2 + tiles) * sizeof(u64));
    if (n == 0) return;
    cudaEvent_t t = c.prof_begin();
    select_kernel<<<(unsigned)tiles, kSelThreads, 0, c.stream>>>(n, pred, emit, ws.p);
    c.check_launch();
    c.prof_end(t, KC_SELECT, 0);
}

// Launches the compaction; returns the number of selected items (syncs).
template <typename Pred, typename Emit>
u64 run_select(Ctx& c, u64 n, Pred pred, Emit emit) {
    if (n == 0) return 0;
    DevBuf<u64> ws;
    run_select_async(c, n, pred, emit, ws);
    unsigned long long total;
    c.read_words(&total, ws.p + 1, 1);
    return total;
}

}  // namespace gd
