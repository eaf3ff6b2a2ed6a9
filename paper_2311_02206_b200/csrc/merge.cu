// merge.cu — difference (ra.hpp:386-422) and merge_sorted (ra.hpp:299-381)
// of one iteration, with the adjacent-dedup tail of canonicalize
// (tuple_array.hpp:124-131) folded into the difference.
//
// Inputs: F canonical (sorted, unique) and N sorted with duplicates (the
// radix-sorted join output).
//
// difference_sorted:  D = unique(N) \ F.  One flag per N row: "first of its
//   run and absent from F", then an order-preserving compaction.  Membership
//   is a binary search of F when N is small next to F (the long tail: reads
//   O(|N| log |F|) sectors instead of streaming F), else a merge-path pass
//   that stages each tile's F and N segments in shared memory.
// merge_disjoint:  F' = F U D for disjoint canonical inputs.  A merge-path
//   partition fixes every tile's output range up front (output position =
//   merge-path diagonal), so there is no cross-tile dependency: tiles that
//   receive no D row are straight coalesced copies of F, the others merge in
//   bank-conflict-free padded shared memory.  HBM traffic: read F + D, write
//   F' — the roofline of the step.
#include "dev_common.cuh"
#include "ops.h"
#include "select.cuh"

namespace gd {

namespace {

constexpr int kMergeThreads = 256;
constexpr int kMergeItems = 8;
constexpr u64 kMergeTile = (u64)kMergeThreads * kMergeItems;

// splits[t] = number of A rows among the first min(t*tile, na+nb) positions
// of the merged order (ties: A first).
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

// Shared-memory index padding: one spare element every 8, so per-thread
// sequential merges (threads 8 elements apart) hit distinct banks.
__device__ __forceinline__ u32 pad8(u32 i) { return i + (i >> 3); }
constexpr u32 kPadTile = kMergeTile + (kMergeTile >> 3) + 8;

// ---- difference: flags ---------------------------------------------------

// Binary-search membership (|N| << |F|): keep[j] = first-of-run && not in F.
template <typename K>
__global__ void diff_flags_search_kernel(const K* __restrict__ F, u64 nf, const K* __restrict__ N, u64 nn,
                                         uint8_t* __restrict__ keep, u64* counters) {
    u64 uniq = 0;
    for (u64 j = (u64)blockIdx.x * blockDim.x + threadIdx.x; j < nn; j += (u64)gridDim.x * blockDim.x) {
        const K x = N[j];
        const bool first = j == 0 || N[j - 1] != x;
        bool in_f = false;
        if (first && nf) {
            u64 lo = 0, hi = nf;
            while (lo < hi) {
                const u64 mid = (lo + hi) >> 1;
                if (F[mid] < x) lo = mid + 1;
                else hi = mid;
            }
            in_f = lo < nf && F[lo] == x;
        }
        keep[j] = (first && !in_f) ? 1 : 0;
        uniq += first;
    }
    uniq = warp_sum(uniq);
    if (lane_id() == 0 && uniq) atomicAdd(counters, uniq);
}

// Binary-search membership against a tiered full relation (several sorted
// disjoint runs, engine.cu LSM mode).
constexpr int kMaxRuns = 24;
struct RunSet {
    const void* ptr[kMaxRuns];
    u64 n[kMaxRuns];
    u32 count;
};

template <typename K>
__global__ void diff_flags_search_runs_kernel(RunSet rs, const K* __restrict__ N, u64 nn,
                                              uint8_t* __restrict__ keep, u64* counters) {
    u64 uniq = 0;
    for (u64 j = (u64)blockIdx.x * blockDim.x + threadIdx.x; j < nn; j += (u64)gridDim.x * blockDim.x) {
        const K x = N[j];
        const bool first = j == 0 || N[j - 1] != x;
        bool in_f = false;
        if (first) {
            for (u32 r = 0; r < rs.count && !in_f; ++r) {
                const K* __restrict__ F = static_cast<const K*>(rs.ptr[r]);
                const u64 nf = rs.n[r];
                u64 lo = 0, hi = nf;
                while (lo < hi) {
                    const u64 mid = (lo + hi) >> 1;
                    if (F[mid] < x) lo = mid + 1;
                    else hi = mid;
                }
                in_f = lo < nf && F[lo] == x;
            }
        }
        keep[j] = (first && !in_f) ? 1 : 0;
        uniq += first;
    }
    uniq = warp_sum(uniq);
    if (lane_id() == 0 && uniq) atomicAdd(counters, uniq);
}

// Streaming membership (|N| comparable to |F|): merge-path tiles over
// (F, N); for each N row the largest F row <= it (merge order, F first)
// decides membership.
template <typename K>
__global__ void __launch_bounds__(kMergeThreads) diff_flags_stream_kernel(
    const K* __restrict__ F, u64 nf, const K* __restrict__ N, u64 nn, const u64* __restrict__ splits,
    uint8_t* __restrict__ keep, u64* counters) {
    __shared__ K sA[kMergeTile + 1];
    const u64 tile = blockIdx.x;
    const u64 diag0 = tile * kMergeTile;
    const u64 diag1 = min(diag0 + kMergeTile, nf + nn);
    const u64 a0 = splits[tile], a1 = splits[tile + 1];
    const u64 b0 = diag0 - a0, b1 = diag1 - a1;
    const u32 na = (u32)(a1 - a0);
    if (b1 == b0) return;
    for (u32 i = threadIdx.x; i < na; i += kMergeThreads) sA[1 + i] = F[a0 + i];
    if (threadIdx.x == 0) sA[0] = a0 > 0 ? F[a0 - 1] : K(0);
    __syncthreads();
    const bool has_halo = a0 > 0;
    u64 uniq = 0;
    for (u64 j = b0 + threadIdx.x; j < b1; j += kMergeThreads) {
        const K x = N[j];
        const bool first = j == 0 || N[j - 1] != x;
        // count of tile F rows <= x (upper bound over sA[1..na])
        u32 lo = 0, hi = na;
        while (lo < hi) {
            const u32 mid = (lo + hi) >> 1;
            if (sA[1 + mid] <= x) lo = mid + 1;
            else hi = mid;
        }
        const bool in_f = lo > 0 ? sA[lo] == x : (has_halo && sA[0] == x);
        keep[j] = (first && !in_f) ? 1 : 0;
        uniq += first;
    }
    uniq = warp_sum(uniq);
    if (lane_id() == 0 && uniq) atomicAdd(counters, uniq);
}

// ---- merge of disjoint canonical arrays -----------------------------------

template <typename K>
struct MergeSmem {
    K in[kPadTile + 2];
    K out[kPadTile];
};

template <typename K>
__global__ void __launch_bounds__(kMergeThreads) merge_disjoint_kernel(
    const K* __restrict__ A, u64 na_all, const K* __restrict__ B, u64 nb_all, const u64* __restrict__ splits,
    K* __restrict__ out, u64* overlap) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const u64 tile = blockIdx.x;
    const u64 diag0 = tile * kMergeTile;
    const u64 diag1 = min(diag0 + kMergeTile, na_all + nb_all);
    const u64 a0 = splits[tile], a1 = splits[tile + 1];
    const u64 b0 = diag0 - a0, b1 = diag1 - a1;
    const u32 na = (u32)(a1 - a0), nb = (u32)(b1 - b0);

    if (nb == 0) {
        // Pure copy of A[a0, a1) to out[diag0, ...): unrolled, coalesced.
        const K* __restrict__ src = A + a0;
        K* __restrict__ dst = out + diag0;
        K v[kMergeItems];
#pragma unroll
        for (int s = 0; s < kMergeItems; ++s) {
            const u32 i = threadIdx.x + s * kMergeThreads;
            if (i < na) v[s] = src[i];
        }
#pragma unroll
        for (int s = 0; s < kMergeItems; ++s) {
            const u32 i = threadIdx.x + s * kMergeThreads;
            if (i < na) dst[i] = v[s];
        }
        return;
    }

    MergeSmem<K>& sm = *reinterpret_cast<MergeSmem<K>*>(smem_raw);
    K* in = sm.in;
    const u32 boff = na;
    for (u32 i = threadIdx.x; i < na; i += kMergeThreads) in[pad8(i)] = A[a0 + i];
    for (u32 i = threadIdx.x; i < nb; i += kMergeThreads) in[pad8(boff + i)] = B[b0 + i];
    __syncthreads();
#define SA(i) in[pad8(i)]
#define SB(i) in[pad8(boff + (i))]
    const u32 tn = na + nb;
    const u32 d = min((u32)threadIdx.x * kMergeItems, tn);
    const u32 de = min(d + kMergeItems, tn);
    u32 lo = d > nb ? d - nb : 0, hi = min(d, na);
    while (lo < hi) {
        const u32 mid = (lo + hi) >> 1;
        if (SA(mid) <= SB(d - 1 - mid)) lo = mid + 1;
        else hi = mid;
    }
    u32 ai = lo, bi = d - lo;
    // an equal pair split by the tile boundary: A[a0-1] (end of the
    // previous tile, A first on ties) against this tile's first B row
    bool ov = threadIdx.x == 0 && a0 > 0 && A[a0 - 1] == SB(0);
#pragma unroll
    for (int s = 0; s < kMergeItems; ++s) {
        if (d + s < de) {
            const K xa = SA(ai);
            const K xb = SB(bi);
            const bool takeA = bi >= nb || (ai < na && xa <= xb);
            ov |= (ai < na && bi < nb && xa == xb);
            sm.out[pad8(d + s)] = takeA ? xa : xb;
            ai += takeA;
            bi += !takeA;
        }
    }
#undef SA
#undef SB
    if (__syncthreads_or(ov) && threadIdx.x == 0) atomicOr(overlap, 1ull);
    for (u32 i = threadIdx.x; i < tn; i += kMergeThreads) out[diag0 + i] = sm.out[pad8(i)];
}

struct FlagKeep {
    const uint8_t* f;
    __device__ bool operator()(u64 i) const { return f[i] != 0; }
};
template <typename K>
struct CopyRow {
    const K* in;
    K* out;
    __device__ void operator()(u64 i, u64 pos) const { out[pos] = in[i]; }
};

template <typename K>
u64* partition(Ctx& c, const K* A, u64 na, const K* B, u64 nb, DevBuf<u64>& splits, u64& tiles) {
    tiles = (na + nb + kMergeTile - 1) / kMergeTile;
    splits.reserve_discard(c, tiles + 1);
    cudaEvent_t tp = c.prof_begin();
    merge_partition_kernel<K><<<(unsigned)((tiles + 1 + 255) / 256), 256, 0, c.stream>>>(
        A, na, B, nb, kMergeTile, tiles + 1, splits.p);
    c.check_launch();
    c.prof_end(tp, KC_OTHER, 0);
    return splits.p;
}

}  // namespace

template <typename K>
MergeResult difference_sorted(Ctx& c, const K* F, u64 nf, const K* N, u64 nn, K* Dout) {
    MergeResult r;
    if (nn == 0) return r;
    DevBuf<uint8_t> keep(c, nn);
    DevBuf<u64> counters(c, 1);
    c.memset(counters.p, 0, sizeof(u64));
    // binary search when N is small next to F, else stream F once
    const bool search = nf == 0 || nn * 24 < nf;
    cudaEvent_t t;
    if (search) {
        const int grid = (int)std::max<u64>(1, std::min<u64>((nn + 255) / 256, (u64)c.num_sms * 16));
        t = c.prof_begin();
        diff_flags_search_kernel<K><<<grid, 256, 0, c.stream>>>(F, nf, N, nn, keep.p, counters.p);
        c.check_launch();
    } else {
        DevBuf<u64> splits;
        u64 tiles = 0;
        partition<K>(c, F, nf, N, nn, splits, tiles);
        t = c.prof_begin();
        diff_flags_stream_kernel<K><<<(unsigned)tiles, kMergeThreads, 0, c.stream>>>(F, nf, N, nn, splits.p,
                                                                                     keep.p, counters.p);
        c.check_launch();
    }
    // algorithmic bytes: N read + flags written (+ F streamed when streaming)
    c.prof_end(t, KC_DIFF, nn * (sizeof(K) + 1) + (search ? 0 : nf * sizeof(K)));
    DevBuf<u64> ws;
    run_select_async(c, nn, FlagKeep{keep.p}, CopyRow<K>{N, Dout}, ws);
    unsigned long long d, u;
    c.read2(&d, ws.p + 1, &u, counters.p);
    r.delta_n = d;
    r.unique_new = u;
    return r;
}

template <typename K>
MergeResult difference_runs(Ctx& c, const K* const* runs, const u64* ns, u32 nruns, const K* N, u64 nn,
                            K* Dout) {
    if (nruns <= 1) return difference_sorted<K>(c, nruns ? runs[0] : nullptr, nruns ? ns[0] : 0, N, nn, Dout);
    if (nruns > (u32)kMaxRuns) throw_logic("difference_runs: too many runs");
    MergeResult r;
    if (nn == 0) return r;
    RunSet rs{};
    u64 total = 0;
    for (u32 i = 0; i < nruns; ++i) {
        rs.ptr[i] = runs[i];
        rs.n[i] = ns[i];
        total += ns[i];
    }
    rs.count = nruns;
    DevBuf<uint8_t> keep(c, nn);
    DevBuf<u64> counters(c, 1);
    c.memset(counters.p, 0, sizeof(u64));
    const int grid = (int)std::max<u64>(1, std::min<u64>((nn + 255) / 256, (u64)c.num_sms * 16));
    cudaEvent_t t = c.prof_begin();
    diff_flags_search_runs_kernel<K><<<grid, 256, 0, c.stream>>>(rs, N, nn, keep.p, counters.p);
    c.check_launch();
    c.prof_end(t, KC_DIFF, nn * (sizeof(K) + 1));
    DevBuf<u64> ws;
    run_select_async(c, nn, FlagKeep{keep.p}, CopyRow<K>{N, Dout}, ws);
    unsigned long long d, u;
    c.read2(&d, ws.p + 1, &u, counters.p);
    r.delta_n = d;
    r.unique_new = u;
    (void)total;
    return r;
}

template <typename K>
bool merge_disjoint(Ctx& c, const K* A, u64 na, const K* B, u64 nb, K* out, bool check_overlap) {
    if (nb == 0) {
        if (na) c.d2d(out, A, na * sizeof(K));
        return false;
    }
    if (na == 0) {
        c.d2d(out, B, nb * sizeof(K));
        return false;
    }
    DevBuf<u64> splits;
    u64 tiles = 0;
    partition<K>(c, A, na, B, nb, splits, tiles);
    DevBuf<u64> ov(c, 1);
    c.memset(ov.p, 0, sizeof(u64));
    const size_t smem = sizeof(MergeSmem<K>);
    static int attr_device = -1;  // one process drives one device
    if (attr_device != c.device) {
        GD_CUDA(cudaFuncSetAttribute(merge_disjoint_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        attr_device = c.device;
    }
    cudaEvent_t t = c.prof_begin();
    merge_disjoint_kernel<K><<<(unsigned)tiles, kMergeThreads, smem, c.stream>>>(A, na, B, nb, splits.p, out, ov.p);
    c.check_launch();
    // algorithmic bytes: read A and B, write A + B
    c.prof_end(t, KC_MERGE, 2 * (na + nb) * sizeof(K));
    if (!check_overlap) return false;
    unsigned long long o;
    c.read_words(&o, ov.p, 1);
    return o != 0;
}

template <typename K>
MergeResult diff_merge(Ctx& c, const K* F, u64 nf, const K* N, u64 nn, K* Fout, K* Dout) {
    DevBuf<K> dtmp;
    if (!Dout) {
        dtmp = DevBuf<K>(c, std::max<u64>(nn, 1));
        Dout = dtmp.p;
    }
    MergeResult r = difference_sorted<K>(c, F, nf, N, nn, Dout);
    if (Fout) r.overlap = merge_disjoint<K>(c, F, nf, Dout, r.delta_n, Fout, true);
    return r;
}

#define GD_INST(K)                                                                         \
    template MergeResult difference_sorted<K>(Ctx&, const K*, u64, const K*, u64, K*);     \
    template bool merge_disjoint<K>(Ctx&, const K*, u64, const K*, u64, K*, bool);         \
    template MergeResult difference_runs<K>(Ctx&, const K* const*, const u64*, u32, const K*, u64, K*); \
    template MergeResult diff_merge<K>(Ctx&, const K*, u64, const K*, u64, K*, K*);
GD_INST(u64)
GD_INST(u128)
#undef GD_INST

}  // namespace gd
