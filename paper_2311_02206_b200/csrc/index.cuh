// index.cuh — device side of the HISA index (index_map.hpp:18-124,
// container.hpp:52-89): open addressing from a join-prefix to the sorted
// range (start, len) of its rows.  16-byte slots hold the exact prefix as
// the tag (u64 keys) — or a 64-bit hash of it, verified against the stored
// row (u128 keys) — and the range packed as start(40) | len(24).  A probe is
// one random 16-byte read in the common case; only ranges longer than
// 2^24-1 rows fall back to a binary search for their end.
#pragma once

#include "dev_common.cuh"
#include "ops.h"

namespace gd {

template <typename K>
__device__ __forceinline__ u64 index_tag(K prefix);
template <>
__device__ __forceinline__ u64 index_tag<u64>(u64 prefix) { return prefix; }
template <>
__device__ __forceinline__ u64 index_tag<u128>(u128 prefix) {
    const u64 h = key_hash64<u128>(prefix);
    return h == kEmptySlot ? kEmptySlot - 1 : h;
}

__device__ __forceinline__ u64 slot_home(u64 tag, u64 slot_count) {
    return __umul64hi(fmix64(tag ^ 0x2545f4914f6cdd1dull), slot_count);
}

// End of the run of rows sharing `prefix`, starting at `start` (binary
// search; only used for saturated length fields).
template <typename K>
__device__ u64 run_end(const IndexView<K>& ix, K prefix, u64 start) {
    u64 lo = start + 1, hi = ix.n;
    while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (prefix_of(ix.rows[mid], ix.arity, ix.bits, ix.plen) == prefix) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <typename K>
__device__ __forceinline__ bool index_probe(const IndexView<K>& ix, K prefix, u64& start, u64& len) {
    const u64 tag = index_tag<K>(prefix);
    u64 pos = slot_home(tag, ix.slot_count);
    for (u64 probes = 0; probes < ix.slot_count; ++probes) {
        const Slot s = ix.slots[pos];
        if (s.tag == kEmptySlot) break;
        if (s.tag == tag) {
            const u64 st = s.val & kStartMask;
            bool match = true;
            if (sizeof(K) > 8) match = prefix_of(ix.rows[st], ix.arity, ix.bits, ix.plen) == prefix;
            if (match) {
                const u64 l = s.val >> 40;
                start = st;
                len = l == kLenSat ? run_end(ix, prefix, st) - st : l;
                return true;
            }
        }
        pos = pos + 1 == ix.slot_count ? 0 : pos + 1;
    }
    start = 0;
    len = 0;
    return false;
}

}  // namespace gd
