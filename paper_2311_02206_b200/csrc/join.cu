// join.cu — the two-pass range-indexed join (join_count, ra.hpp:141-182;
// join_materialize, ra.hpp:189-263) and select_project (ra.hpp:267-293).
//
// Pass 1 (join_probe): one probe of the HISA index per outer row gives the
// inner range (start, count); the per-row counts are exclusive-scanned in
// the same kernel (block scan + decoupled look-back), so there is no
// separate count pass and no sequential prefix sum (ra.hpp:235-238).
// Pass 2 (join_materialize): load-balanced expansion — a merge-path split of
// (row ends, output indices) gives every CTA exactly kLbsTile items of
// rows+outputs regardless of skew (power-law hubs), and every output slot j
// is written by consecutive threads (coalesced).  Output order equals the
// reference's: outer-row order, then inner-range order.
#include "index.cuh"
#include "select.cuh"

namespace gd {

namespace {

constexpr int kProbeThreads = 256;
constexpr int kProbeItems = 8;
constexpr u64 kProbeTile = (u64)kProbeThreads * kProbeItems;
constexpr int kLbsThreads = 256;
constexpr u64 kLbsTile = 1024;

template <typename K>
__device__ __forceinline__ u64 outer_col(const DevJoin& jd, K o, u32 c) {
    return col_of(o, jd.outer_arity, jd.bits, jd.outer_perm[c]);
}

template <typename K>
__device__ __forceinline__ u64 op_val(const DevOperand& op, const DevJoin& jd, K o, K i) {
    if (op.kind == GD_OUTER_COL) return outer_col(jd, o, op.column);
    if (op.kind == GD_INNER_COL) return col_of(i, jd.inner_arity, jd.bits, op.column);
    return op.value;
}

template <typename K>
__device__ __forceinline__ K project(const DevJoin& jd, K o, K i) {
    K r = 0;
    for (u32 c = 0; c < jd.proj_arity; ++c)
        r |= (K)op_val(jd.proj[c], jd, o, i) << ((jd.proj_arity - 1 - c) * jd.bits);
    return r;
}

template <typename K>
__device__ __forceinline__ bool passes(const DevJoin& jd, K o, K i) {
    for (u32 f = 0; f < jd.nfilters; ++f) {
        const DevFilter& fl = jd.filters[f];
        const bool eq = !fl.never && op_val(fl.lhs, jd, o, i) == op_val(fl.rhs, jd, o, i);
        if (eq != (fl.require_equal != 0)) return false;
    }
    return true;
}

template <typename K>
__device__ __forceinline__ K outer_prefix(const DevJoin& jd, K o) {
    if (jd.outer_identity) return prefix_of(o, jd.outer_arity, jd.bits, jd.jcc);
    K p = 0;
    for (u32 c = 0; c < jd.jcc; ++c) p |= (K)outer_col(jd, o, c) << ((jd.jcc - 1 - c) * jd.bits);
    return p;
}

// ws: [0] tile counter, [1] candidate total, [2..] statuses.
template <typename K>
__global__ void __launch_bounds__(kProbeThreads) join_probe_kernel(
    const K* __restrict__ outer, u64 n, DevJoin jd, IndexView<K> ix, u64 inner_n,
    u64* __restrict__ row_start, u64* __restrict__ row_off, u64* ws) {
    __shared__ u64 s_tile;
    __shared__ u64 s_scan[kProbeThreads / 32 + 1];
    __shared__ u64 s_base;
    const u64 tile = claim_tile(ws, &s_tile);
    const u64 begin = tile * kProbeTile + (u64)threadIdx.x * kProbeItems;
    u64 st[kProbeItems], ln[kProbeItems];
    u64 sum = 0;
#pragma unroll
    for (int j = 0; j < kProbeItems; ++j) {
        st[j] = 0;
        ln[j] = 0;
        const u64 r = begin + j;
        if (r < n) {
            if (jd.jcc == 0) {
                ln[j] = inner_n;
            } else {
                index_probe(ix, outer_prefix(jd, outer[r]), st[j], ln[j]);
            }
        }
        sum += ln[j];
    }
    u64 tile_total;
    const u64 excl = block_exclusive_scan<u64, kProbeThreads>(sum, tile_total, s_scan);
    if (threadIdx.x < 32) {
        const u64 base = warp_lookback(ws + 2, tile, tile_total);
        if (threadIdx.x == 0) {
            s_base = base;
            atomicAdd(ws + 1, tile_total);
        }
    }
    __syncthreads();
    u64 off = s_base + excl;
#pragma unroll
    for (int j = 0; j < kProbeItems; ++j) {
        const u64 r = begin + j;
        if (r < n) {
            row_start[r] = st[j];
            row_off[r] = off;
            off += ln[j];
            if (r == n - 1) row_off[n] = off;
        }
    }
}

// Merge-path split of (row ends row_off[1..n], outputs 0..total-1).
__global__ void lbs_partition_kernel(const u64* __restrict__ row_off, u64 n, u64 total, u64 tile,
                                     u64 nsplits, u64* __restrict__ splits) {
    const u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nsplits) return;
    const u64 diag = min(t * tile, n + total);
    u64 lo = diag > total ? diag - total : 0;
    u64 hi = min(diag, n);
    while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (row_off[mid + 1] <= diag - 1 - mid) lo = mid + 1;
        else hi = mid;
    }
    splits[t] = lo;
}

template <typename K>
__global__ void __launch_bounds__(kLbsThreads) join_materialize_kernel(
    const K* __restrict__ outer, u64 n, const K* __restrict__ inner, DevJoin jd,
    const u64* __restrict__ row_start, const u64* __restrict__ row_off, u64 total,
    const u64* __restrict__ splits, K* __restrict__ out, uint8_t* __restrict__ flags) {
    __shared__ u64 s_off[kLbsTile + 1];
    __shared__ u64 s_start[kLbsTile + 1];
    __shared__ K s_outer[kLbsTile + 1];
    const u64 tile = blockIdx.x;
    const u64 diag0 = tile * kLbsTile;
    const u64 diag1 = min(diag0 + kLbsTile, n + total);
    const u64 a0 = splits[tile], a1 = splits[tile + 1];
    const u64 b0 = diag0 - a0, b1 = diag1 - a1;
    if (b1 <= b0) return;
    const u64 rlast = min(a1, n - 1);
    const u32 rcount = (u32)(rlast - a0 + 1);
    for (u32 i = threadIdx.x; i < rcount; i += kLbsThreads) {
        s_off[i] = row_off[a0 + i];
        s_start[i] = row_start[a0 + i];
        s_outer[i] = outer[a0 + i];
    }
    __syncthreads();
    for (u64 j = b0 + threadIdx.x; j < b1; j += kLbsThreads) {
        u32 lo = 0, hi = rcount;
        while (hi - lo > 1) {
            const u32 mid = (lo + hi) >> 1;
            if (s_off[mid] <= j) lo = mid;
            else hi = mid;
        }
        const K o = s_outer[lo];
        const K i = inner[s_start[lo] + (j - s_off[lo])];
        out[j] = project(jd, o, i);
        if (flags) flags[j] = passes(jd, o, i) ? 1 : 0;
    }
}

template <typename K>
struct SelPred {
    const K* rows;
    DevJoin jd;
    __device__ bool operator()(u64 r) const { return passes(jd, rows[r], K(0)); }
};
template <typename K>
struct SelEmit {
    const K* rows;
    DevJoin jd;
    K* out;
    __device__ void operator()(u64 r, u64 pos) const { out[pos] = project(jd, rows[r], K(0)); }
};

template <typename K>
__global__ void owner_kernel(const K* __restrict__ keys, u64 n, u32 nranks, u32* __restrict__ owner) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        owner[i] = (u32)(key_hash64<K>(keys[i]) % nranks);
}

__global__ void owner_flags_kernel(const u32* __restrict__ owner, u64 n, u32 k, uint8_t* __restrict__ flags) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        flags[i] = owner[i] == k ? 1 : 0;
}

}  // namespace

void owner_flags(Ctx& c, const u32* owner, u64 n, u32 k, uint8_t* flags) {
    if (n == 0) return;
    const int grid = (int)std::max<u64>(1, std::min<u64>((n + 255) / 256, (u64)c.num_sms * 8));
    owner_flags_kernel<<<grid, 256, 0, c.stream>>>(owner, n, k, flags);
    c.check_launch();
}

template <typename K>
u64 join_probe(Ctx& c, const K* outer, u64 n, const DevJoin& jd, const IndexView<K>* ix, u64 inner_n,
               u64* row_start, u64* row_off) {
    if (n == 0) {
        c.memset(row_off, 0, sizeof(u64));
        return 0;
    }
    const u64 tiles = (n + kProbeTile - 1) / kProbeTile;
    DevBuf<u64> ws(c, 2 + tiles);
    c.memset(ws.p, 0, (2 + tiles) * sizeof(u64));
    IndexView<K> view{};
    if (ix) view = *ix;
    cudaEvent_t t = c.prof_begin();
    join_probe_kernel<K><<<(unsigned)tiles, kProbeThreads, 0, c.stream>>>(outer, n, jd, view, inner_n,
                                                                           row_start, row_off, ws.p);
    c.check_launch();
    // algorithmic bytes: the outer rows + one 16-byte slot probe per row
    c.prof_end(t, KC_PROBE, n * (sizeof(K) + (jd.jcc ? sizeof(Slot) : 0)));
    unsigned long long total;
    c.read_words(&total, ws.p + 1, 1);
    return total;
}

template <typename K>
void join_materialize(Ctx& c, const K* outer, u64 n, const K* inner, const DevJoin& jd,
                      const u64* row_start, const u64* row_off, u64 total, K* out, uint8_t* flags) {
    if (total == 0 || n == 0) return;
    const u64 tiles = (n + total + kLbsTile - 1) / kLbsTile;
    DevBuf<u64> splits(c, tiles + 1);
    cudaEvent_t tp = c.prof_begin();
    lbs_partition_kernel<<<(unsigned)((tiles + 1 + 255) / 256), 256, 0, c.stream>>>(
        row_off, n, total, kLbsTile, tiles + 1, splits.p);
    c.check_launch();
    c.prof_end(tp, KC_OTHER, 0);
    cudaEvent_t t = c.prof_begin();
    join_materialize_kernel<K><<<(unsigned)tiles, kLbsThreads, 0, c.stream>>>(
        outer, n, inner, jd, row_start, row_off, total, splits.p, out, flags);
    c.check_launch();
    // algorithmic bytes: the matched inner rows read + the output rows written
    c.prof_end(t, KC_MATERIALIZE, 2 * total * sizeof(K));
}

template <typename K>
u64 select_project(Ctx& c, const K* rows, u64 n, const DevJoin& jd, K* out) {
    return run_select(c, n, SelPred<K>{rows, jd}, SelEmit<K>{rows, jd, out});
}

template <typename K>
void owner_of(Ctx& c, const K* keys, u64 n, u32 nranks, u32* owner) {
    if (n == 0) return;
    const int grid = (int)std::max<u64>(1, std::min<u64>((n + 255) / 256, (u64)c.num_sms * 8));
    owner_kernel<K><<<grid, 256, 0, c.stream>>>(keys, n, nranks, owner);
    c.check_launch();
}

#define GD_INST(K)                                                                                 \
    template u64 join_probe<K>(Ctx&, const K*, u64, const DevJoin&, const IndexView<K>*, u64, u64*, \
                               u64*);                                                              \
    template void join_materialize<K>(Ctx&, const K*, u64, const K*, const DevJoin&, const u64*,    \
                                      const u64*, u64, K*, uint8_t*);                              \
    template u64 select_project<K>(Ctx&, const K*, u64, const DevJoin&, K*);                       \
    template void owner_of<K>(Ctx&, const K*, u64, u32, u32*);
GD_INST(u64)
GD_INST(u128)
#undef GD_INST

}  // namespace gd
