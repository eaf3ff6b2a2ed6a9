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
#include "join.cuh"
#include "select.cuh"

namespace gd {

namespace {

constexpr int kProbeThreads = 256;
constexpr int kProbeItems = 4;
constexpr u64 kProbeTile = (u64)kProbeThreads * kProbeItems;
constexpr int kLbsThreads = 256;
constexpr u64 kLbsTile = 1024;

// Pass 1a: one probe per outer row, kProbeItems independent rows per thread
// (row = tile base + item * threads + tid: coalesced, and the items' slot
// loads are issued together for memory-level parallelism).  Writes the
// match start and count of every row and the tile's count sum; no
// cross-tile dependency.
template <typename K>
__global__ void __launch_bounds__(kProbeThreads) join_probe_kernel(
    const K* __restrict__ outer, u64 n, DevJoin jd, IndexView<K> ix, u64 inner_n,
    u64* __restrict__ row_start, u64* __restrict__ row_cnt, u64* __restrict__ tile_sum) {
    __shared__ u64 s_red[kProbeThreads / 32];
    const u64 base = (u64)blockIdx.x * kProbeTile + threadIdx.x;
    u64 sum = 0;
    if (jd.jcc == 0) {
#pragma unroll
        for (int j = 0; j < kProbeItems; ++j) {
            const u64 r = base + (u64)j * kProbeThreads;
            if (r < n) {
                row_start[r] = 0;
                row_cnt[r] = inner_n;
                sum += inner_n;
            }
        }
    } else {
        K pre[kProbeItems];
        u64 tag[kProbeItems], pos[kProbeItems];
        Slot s[kProbeItems];
#pragma unroll
        for (int j = 0; j < kProbeItems; ++j) {
            const u64 r = base + (u64)j * kProbeThreads;
            pre[j] = r < n ? outer_prefix(jd, outer[r]) : K(0);
        }
#pragma unroll
        for (int j = 0; j < kProbeItems; ++j) {
            tag[j] = index_tag<K>(pre[j]);
            pos[j] = slot_home(tag[j], ix.slot_count);
            s[j] = ix.slots[pos[j]];
        }
#pragma unroll
        for (int j = 0; j < kProbeItems; ++j) {
            const u64 r = base + (u64)j * kProbeThreads;
            if (r >= n) continue;
            u64 st = 0, ln = 0;
            if (s[j].tag == tag[j] && (sizeof(K) == 8 ||
                                       prefix_of(ix.rows[s[j].val & kStartMask], ix.arity, ix.bits, ix.plen) == pre[j])) {
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
    sum = warp_sum(sum);
    if (lane_id() == 0) s_red[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        u64 t = 0;
        for (int w = 0; w < kProbeThreads / 32; ++w) t += s_red[w];
        tile_sum[blockIdx.x] = t;
    }
}

// Pass 1b: exclusive scan of the per-tile sums (one block); total at [ntiles].
__global__ void __launch_bounds__(1024) scan_tiles_kernel(u64* __restrict__ tile_sum, u64 ntiles) {
    __shared__ u64 s_scan[1024 / 32 + 1];
    __shared__ u64 s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (u64 b = 0; b < ntiles; b += 1024) {
        const u64 i = b + threadIdx.x;
        const u64 v = i < ntiles ? tile_sum[i] : 0;
        u64 tot;
        const u64 ex = block_exclusive_scan<u64, 1024>(v, tot, s_scan);
        if (i < ntiles) tile_sum[i] = s_carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) s_carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) tile_sum[ntiles] = s_carry;
}

// Pass 1c: row offsets = tile prefix + in-tile exclusive scan of counts
// (in place over the counts); row_off[n] = total.
__global__ void __launch_bounds__(kProbeThreads) apply_offsets_kernel(u64* __restrict__ row_off, u64 n,
                                                                      const u64* __restrict__ tile_prefix) {
    __shared__ u64 s_scan[kProbeThreads / 32 + 1];
    const u64 begin = (u64)blockIdx.x * kProbeTile + (u64)threadIdx.x * kProbeItems;
    u64 c[kProbeItems];
    u64 sum = 0;
#pragma unroll
    for (int j = 0; j < kProbeItems; ++j) {
        c[j] = begin + j < n ? row_off[begin + j] : 0;
        sum += c[j];
    }
    u64 tot;
    u64 off = tile_prefix[blockIdx.x] + block_exclusive_scan<u64, kProbeThreads>(sum, tot, s_scan);
#pragma unroll
    for (int j = 0; j < kProbeItems; ++j) {
        const u64 r = begin + j;
        if (r < n) {
            row_off[r] = off;
            off += c[j];
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
    DevBuf<u64> tile_sum(c, tiles + 1);
    IndexView<K> view{};
    if (ix) view = *ix;
    cudaEvent_t t = c.prof_begin();
    join_probe_kernel<K><<<(unsigned)tiles, kProbeThreads, 0, c.stream>>>(outer, n, jd, view, inner_n,
                                                                           row_start, row_off, tile_sum.p);
    c.check_launch();
    // algorithmic bytes: the outer rows + one 16-byte slot probe per row
    c.prof_end(t, KC_PROBE, n * (sizeof(K) + (jd.jcc ? sizeof(Slot) : 0)));
    cudaEvent_t t2 = c.prof_begin();
    scan_tiles_kernel<<<1, 1024, 0, c.stream>>>(tile_sum.p, tiles);
    c.check_launch();
    apply_offsets_kernel<<<(unsigned)tiles, kProbeThreads, 0, c.stream>>>(row_off, n, tile_sum.p);
    c.check_launch();
    c.prof_end(t2, KC_SELECT, 0);
    unsigned long long total;
    c.read_words(&total, row_off + n, 1);
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
