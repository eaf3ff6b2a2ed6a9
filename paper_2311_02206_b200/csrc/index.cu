// index.cu — HISA index build (group_starts, index_map.hpp:46-66, and
// build_index, index_map.hpp:74-124) and batched range_lookup
// (container.hpp:52-89) on the device.
//
// Build = one order-preserving compaction of the group-start positions of
// the sorted keys (single pass, look-back), then one thread per group claims
// a slot with a 64-bit atomicCAS and publishes (start, len).  Slot count
// follows the reference rule ceil(distinct / load_factor) so occupancy and
// slot_count() match the CPU index; the slot layout itself is free (only
// lookups are compared, SURVEY §8c "Unpinned").
#include "index.cuh"
#include "select.cuh"

namespace gd {

namespace {

template <typename K>
struct GroupStartPred {
    const K* rows;
    u32 shift;
    __device__ bool operator()(u64 i) const {
        if (i == 0) return true;
        const K a = shift >= sizeof(K) * 8 ? K(0) : (K)(rows[i - 1] >> shift);
        const K b = shift >= sizeof(K) * 8 ? K(0) : (K)(rows[i] >> shift);
        return a != b;
    }
};
struct PosEmit {
    u64* gs;
    __device__ void operator()(u64 i, u64 pos) const { gs[pos] = i; }
};

__global__ void set_word_kernel(u64* p, u64 v) { *p = v; }

template <typename K>
__global__ void index_insert_kernel(const K* __restrict__ rows, u32 arity, u32 bits, u32 plen,
                                    const u64* __restrict__ gs, u64 groups, Slot* __restrict__ slots,
                                    u64 slot_count) {
    for (u64 g = (u64)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (u64)gridDim.x * blockDim.x) {
        const u64 st = gs[g];
        const u64 len = gs[g + 1] - st;
        const K prefix = prefix_of(rows[st], arity, bits, plen);
        const u64 tag = index_tag<K>(prefix);
        const u64 val = st | (min(len, kLenSat) << 40);
        u64 pos = slot_home(tag, slot_count);
        while (true) {
            const u64 prev = atomicCAS(&slots[pos].tag, kEmptySlot, tag);
            if (prev == kEmptySlot) {
                slots[pos].val = val;
                break;
            }
            pos = pos + 1 == slot_count ? 0 : pos + 1;
        }
    }
}

template <typename K>
__global__ void index_lookup_kernel(IndexView<K> ix, const K* __restrict__ prefixes,
                                    const uint8_t* __restrict__ valid, u64 nkeys, u64* out_start,
                                    u64* out_count) {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < nkeys; i += (u64)gridDim.x * blockDim.x) {
        u64 st = 0, len = 0;
        if (!valid || valid[i]) index_probe(ix, prefixes[i], st, len);
        out_start[i] = st;
        out_count[i] = len;
    }
}

inline int grid_for(const Ctx& c, u64 n, int threads = 256) {
    const u64 want = (n + threads - 1) / threads;
    return (int)std::max<u64>(1, std::min<u64>(want, (u64)c.num_sms * 8));
}

}  // namespace

template <typename K>
u64 group_starts(Ctx& c, const K* rows, u64 n, u32 arity, u32 bits, u32 plen, DevBuf<u64>& gs) {
    gs.reserve_discard(c, n + 1);
    const u32 shift = (arity - plen) * bits;
    const u64 g = run_select(c, n, GroupStartPred<K>{rows, shift}, PosEmit{gs.p});
    set_word_kernel<<<1, 1, 0, c.stream>>>(gs.p + g, n);
    c.check_launch();
    return g;
}

template <typename K>
void build_index(Ctx& c, const K* rows, u64 n, u32 arity, u32 bits, u32 plen, double lf,
                 DevIndex<K>& out) {
    DevBuf<u64> gs;
    const u64 groups = group_starts<K>(c, rows, n, arity, bits, plen, gs);
    out.groups = groups;
    out.plen = plen;
    // The reference's sizing (and accounted bytes) use the configured load
    // factor; the device table is allocated at <= 0.5 so linear-probe chains
    // stay short (expected ~1.5 probes per hit, ~2.5 per miss).
    out.logical_slots = slot_count_for(groups, lf);
    out.slot_count = slot_count_for(groups, std::min(lf, 0.5));
    out.slots.reserve_discard(c, out.slot_count);
    c.memset(out.slots.p, 0xff, out.slot_count * sizeof(Slot));
    if (groups) {
        cudaEvent_t t = c.prof_begin();
        index_insert_kernel<K><<<grid_for(c, groups), 256, 0, c.stream>>>(
            rows, arity, bits, plen, gs.p, groups, out.slots.p, out.slot_count);
        c.check_launch();
        c.prof_end(t, KC_INDEX, groups * (16 + 2 * 8 + sizeof(K)));
    }
}

template <typename K>
void index_lookup(Ctx& c, const IndexView<K>& ix, const K* prefixes, const uint8_t* valid, u64 nkeys,
                  u64* out_start, u64* out_count) {
    if (nkeys == 0) return;
    index_lookup_kernel<K><<<grid_for(c, nkeys), 256, 0, c.stream>>>(ix, prefixes, valid, nkeys,
                                                                      out_start, out_count);
    c.check_launch();
}

#define GD_INST(K)                                                                             \
    template u64 group_starts<K>(Ctx&, const K*, u64, u32, u32, u32, DevBuf<u64>&);            \
    template void build_index<K>(Ctx&, const K*, u64, u32, u32, u32, double, DevIndex<K>&);    \
    template void index_lookup<K>(Ctx&, const IndexView<K>&, const K*, const uint8_t*, u64,    \
                                  u64*, u64*);
GD_INST(u64)
GD_INST(u128)
#undef GD_INST

}  // namespace gd
