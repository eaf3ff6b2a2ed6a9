// merge.cu — the fused difference + merge of one iteration
// (difference, ra.hpp:386-422, then merge_sorted, ra.hpp:299-381, and the
// adjacent-dedup tail of canonicalize, tuple_array.hpp:124-131).
//
// Inputs: F canonical (sorted, unique) and N sorted with duplicates (the
// radix-sorted join output).  One merge-path pass emits
//     F' = F U N   and   D = unique(N) \ F
// in a single read of F and N and a single write of F' and D.
//
// Merge order breaks ties F-first, so an N element x is in F iff the F
// element immediately before it in merge order equals x, and is a
// duplicate iff the N element before it equals x.  Each tile of
// kMergeThreads * kMergeItems merged positions is delimited by a global
// merge-path search (partition kernel), staged in shared memory, merged by
// per-thread sequential merges, and its output offsets come from a block
// scan of kept-N counts plus a decoupled look-back across tiles.
#include "dev_common.cuh"
#include "ops.h"

namespace gd {

namespace {

constexpr int kMergeThreads = 256;
constexpr int kMergeItems = 8;
constexpr u64 kMergeTile = (u64)kMergeThreads * kMergeItems;

// splits[t] = number of F elements among the first min(t*tile, nf+nn)
// positions of the merged order (ties: F first).
template <typename K>
__global__ void merge_partition_kernel(const K* __restrict__ A, u64 na, const K* __restrict__ B,
                                       u64 nb, u64 tile, u64 nsplits, u64* __restrict__ splits) {
    const u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nsplits) return;
    const u64 diag = min(t * tile, na + nb);
    u64 lo = diag > nb ? diag - nb : 0;
    u64 hi = min(diag, na);
    while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (A[mid] <= B[diag - 1 - mid]) lo = mid + 1;
        else hi = mid;
    }
    splits[t] = lo;
}

// Shared-memory index padding: one spare element every 8, so the per-thread
// sequential merges (threads 8 elements apart) hit distinct banks.
__device__ __forceinline__ u32 pad8(u32 i) { return i + (i >> 3); }
constexpr u32 kPadTile = kMergeTile + (kMergeTile >> 3) + 8;

template <typename K>
struct MergeSmem {
    K in[kPadTile + 2];  // [halo F | F tile | halo N | N tile], padded indices
    K outF[kPadTile];
    K outD[kPadTile];
};

// ws: [0] tile counter, [1] kept total, [2] unique-N total, [3] overlap,
//     [4..] tile statuses.
template <typename K>
__global__ void __launch_bounds__(kMergeThreads) diff_merge_kernel(
    const K* __restrict__ F, u64 nf, const K* __restrict__ N, u64 nn,
    const u64* __restrict__ splits, K* __restrict__ Fout, K* __restrict__ Dout, u64* ws) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    MergeSmem<K>& sm = *reinterpret_cast<MergeSmem<K>*>(smem_raw);
    __shared__ u64 s_tile;
    __shared__ u64 s_scan[kMergeThreads / 32 + 1];
    __shared__ u64 s_base;

    const u64 tile = claim_tile(ws, &s_tile);
    const u64 total = nf + nn;
    const u64 diag0 = tile * kMergeTile;
    const u64 diag1 = min(diag0 + kMergeTile, total);
    const u64 a0 = splits[tile], a1 = splits[tile + 1];
    const u64 b0 = diag0 - a0, b1 = diag1 - a1;
    const u32 na = (u32)(a1 - a0), nb = (u32)(b1 - b0);

    // Stage (logical index -> padded slot): A(i) = F[a0 - 1 + i] for
    // i in [0, na] (A(0) is the halo), B(i) = N[b0 - 1 + i] at logical
    // offset na + 1.
    K* in = sm.in;
    const u32 boff = na + 1;
    for (u32 i = threadIdx.x; i < na; i += kMergeThreads) in[pad8(1 + i)] = F[a0 + i];
    for (u32 i = threadIdx.x; i < nb; i += kMergeThreads) in[pad8(boff + 1 + i)] = N[b0 + i];
    if (threadIdx.x == 0) {
        in[pad8(0)] = a0 > 0 ? F[a0 - 1] : K(0);
        in[pad8(boff)] = b0 > 0 ? N[b0 - 1] : K(0);
    }
    __syncthreads();
#define SA(i) in[pad8(i)]
#define SB(i) in[pad8(boff + (i))]

    // Per-thread sub-range of the tile's merge path.
    const u32 tn = na + nb;
    const u32 d = min((u32)threadIdx.x * kMergeItems, tn);
    const u32 de = min(d + kMergeItems, tn);
    u32 lo = d > nb ? d - nb : 0, hi = min(d, na);
    while (lo < hi) {
        const u32 mid = (lo + hi) >> 1;
        if (SA(1 + mid) <= SB(1 + (d - 1 - mid))) lo = mid + 1;
        else hi = mid;
    }
    const u32 ai0 = lo;

    // One sequential merge of <= kMergeItems steps into registers.
    // kind: 0 = F row, 1 = kept N row (new), 2 = dropped N row.
    K val[kMergeItems];
    u32 kinds = 0;  // 2 bits per step
    u32 ai = ai0, bi = d - ai0;
    u64 kept = 0, uniq = 0;
    bool overlap = false;
#pragma unroll
    for (int s = 0; s < kMergeItems; ++s) {
        if (d + s < de) {
            const K xa = SA(1 + ai);
            const K xb = SB(1 + bi);
            const bool takeA = bi >= nb || (ai < na && xa <= xb);
            if (takeA) {
                val[s] = xa;
                ++ai;
            } else {
                const bool dup = (b0 + bi > 0) && SB(bi) == xb;
                const bool inF = (a0 + ai > 0) && SA(ai) == xb;
                uniq += !dup;
                overlap |= (inF && !dup);
                const bool keep = !dup && !inF;
                kept += keep;
                val[s] = xb;
                kinds |= (keep ? 1u : 2u) << (2 * s);
                ++bi;
            }
        } else {
            kinds |= 3u << (2 * s);
        }
    }
    u64 tile_kept;
    const u64 excl = block_exclusive_scan<u64, kMergeThreads>(kept | (uniq << 32), tile_kept, s_scan);
    const u64 tile_uniq = tile_kept >> 32;
    tile_kept &= 0xffffffffull;
    const bool any_overlap = __syncthreads_or(overlap);
    if (threadIdx.x < 32) {
        const u64 base = warp_lookback(ws + 4, tile, tile_kept);
        if (threadIdx.x == 0) {
            s_base = base;
            atomicAdd(ws + 1, tile_kept);
            atomicAdd(ws + 2, tile_uniq);
            if (any_overlap) atomicOr(ws + 3, 1ull);
        }
    }
    // Registers -> staging at tile-local output positions.
    u32 a = ai0;
    u32 k = (u32)(excl & 0xffffffffull);  // kept N rows before this thread in the tile
#pragma unroll
    for (int s = 0; s < kMergeItems; ++s) {
        const u32 kind = (kinds >> (2 * s)) & 3u;
        if (kind == 0) {
            sm.outF[pad8(a + k)] = val[s];
            ++a;
        } else if (kind == 1) {
            sm.outF[pad8(a + k)] = val[s];
            sm.outD[pad8(k)] = val[s];
            ++k;
        }
    }
#undef SA
#undef SB
    __syncthreads();
    const u64 kbase = s_base;
    // Coalesced copy-out: F' rows [a0 + kbase, a1 + kbase + tile_kept),
    //                     D rows  [kbase, kbase + tile_kept).
    const u32 nout = na + (u32)tile_kept;
    if (Fout)
        for (u32 i = threadIdx.x; i < nout; i += kMergeThreads) Fout[a0 + kbase + i] = sm.outF[pad8(i)];
    if (Dout)
        for (u32 i = threadIdx.x; i < (u32)tile_kept; i += kMergeThreads) Dout[kbase + i] = sm.outD[pad8(i)];
}

}  // namespace

template <typename K>
MergeResult diff_merge(Ctx& c, const K* F, u64 nf, const K* N, u64 nn, K* Fout, K* Dout) {
    MergeResult r;
    if (nn == 0) {
        if (Fout && nf) c.d2d(Fout, F, nf * sizeof(K));
        return r;
    }
    const u64 total = nf + nn;
    const u64 tiles = (total + kMergeTile - 1) / kMergeTile;
    DevBuf<u64> splits(c, tiles + 1);
    cudaEvent_t tp = c.prof_begin();
    merge_partition_kernel<K><<<(unsigned)((tiles + 1 + 255) / 256), 256, 0, c.stream>>>(
        F, nf, N, nn, kMergeTile, tiles + 1, splits.p);
    c.check_launch();
    c.prof_end(tp, KC_OTHER, 0);
    DevBuf<u64> ws(c, 4 + tiles);
    c.memset(ws.p, 0, (4 + tiles) * sizeof(u64));
    const size_t smem = sizeof(MergeSmem<K>);
    static bool attr_set = false;
    if (!attr_set) {
        GD_CUDA(cudaFuncSetAttribute(diff_merge_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        attr_set = true;
    }
    cudaEvent_t t = c.prof_begin();
    diff_merge_kernel<K><<<(unsigned)tiles, kMergeThreads, smem, c.stream>>>(F, nf, N, nn, splits.p,
                                                                               Fout, Dout, ws.p);
    c.check_launch();
    const long rec = c.prof_end(t, KC_MERGE, 0);
    unsigned long long w[3];
    c.read_words(w, ws.p + 1, 3);
    r.delta_n = w[0];
    r.unique_new = w[1];
    r.overlap = w[2] != 0;
    // algorithmic bytes: read F and the sorted new rows, write
    // F' = F + D and D.
    c.prof_add_bytes(rec, sizeof(K) * ((nf + nn) + (Fout ? nf + r.delta_n : 0) + (Dout ? r.delta_n : 0)));
    return r;
}

template MergeResult diff_merge<u64>(Ctx&, const u64*, u64, const u64*, u64, u64*, u64*);
template MergeResult diff_merge<u128>(Ctx&, const u128*, u64, const u128*, u64, u128*, u128*);

}  // namespace gd
