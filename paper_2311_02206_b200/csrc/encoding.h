// encoding.h — choice of the device tuple encoding.
//
// Datalog without arithmetic only compares values for equality and the
// output order is lexicographic, so any ORDER-PRESERVING injective map of
// the value domain gives bit-identical canonical outputs after decoding.
// Identity packing (bits = bitwidth(max value + 1)) is used when the widest
// tuple fits the key; otherwise values are replaced by their rank in the
// sorted distinct value set (a device-built dictionary).  Keys are u64 when
// arity * bits <= 64, else u128.
#pragma once

#include <utility>
#include <vector>

#include "ops.h"

namespace gd {

struct EncodingOwner {
    Encoding e;
    DevBuf<u64> dict;
};

inline void choose_encoding(Ctx& c, const std::vector<std::pair<const u64*, u64>>& arrays,
                            const std::vector<u64>& constants, u32 max_arity, EncodingOwner& out) {
    if (max_arity == 0) max_arity = 1;
    if (max_arity > kMaxArity) throw_unsupported("arity above " + std::to_string(kMaxArity));
    u64 maxval = 0;
    u64 total = 0;
    for (auto& a : arrays) {
        if (a.second) maxval = std::max(maxval, max_value(c, a.first, a.second));
        total += a.second;
    }
    for (u64 v : constants) maxval = std::max(maxval, v);
    if (maxval == kEmptySlot) throw_load("value equals the reserved sentinel (kEmptySlot)");
    const u32 b_id = std::max(1u, bitwidth(maxval + 1));
    out.e = Encoding{};
    out.dict.release();
    if (max_arity * b_id <= 64) {
        out.e.bits = b_id;
        out.e.key_words = 1;
        return;
    }
    // Dictionary of every stored value and every rule constant.
    const u64 all_n = total + constants.size();
    DevBuf<u64> all(c, all_n);
    u64 off = 0;
    for (auto& a : arrays) {
        c.d2d(all.p + off, a.first, a.second * sizeof(u64));
        off += a.second;
    }
    if (!constants.empty()) {
        c.h2d(all.p + off, constants.data(), constants.size() * sizeof(u64));
        c.sync();  // constants vector is host memory owned by the caller
    }
    const u64 d = build_dictionary(c, all.p, all_n, maxval, out.dict);
    const u32 b_d = std::max(1u, bitwidth(d));
    if (max_arity * b_d <= 64) {
        out.e = Encoding{b_d, 1, true, out.dict.p, d};
    } else if (max_arity * b_id <= 128) {
        out.dict.release();
        out.e = Encoding{b_id, 2, false, nullptr, 0};
    } else if (max_arity * b_d <= 128) {
        out.e = Encoding{b_d, 2, true, out.dict.p, d};
    } else {
        throw_unsupported("tuples of arity " + std::to_string(max_arity) + " with " + std::to_string(d) +
                          " distinct values exceed the 128-bit device key");
    }
}

}  // namespace gd
