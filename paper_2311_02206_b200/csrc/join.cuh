// join.cuh — device helpers of the range-indexed join shared by join.cu
// (kernel-level join_count / join_materialize, ra.hpp:141-263) and loop.cu
// (the resident fixpoint loop): outer-view column access with the folded
// source permutation, projection (column_map, ra.hpp:25-40) and post-match
// filters (row_filter, ra.hpp:42-52).
#pragma once

#include "dev_common.cuh"
#include "ops.h"

namespace gd {

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

}  // namespace gd
