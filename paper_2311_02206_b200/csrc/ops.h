// ops.h — host launchers of the sm_100a kernels (internal API of
// libgdlog_b200.so).  Every launcher is stream-ordered on ctx.stream; the
// ones returning a count synchronize once to read it back.
#pragma once

#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "ctx.h"
#include "gdlog_b200.h"

namespace gd {

using u32 = uint32_t;
using u64 = unsigned long long;
using u128 = unsigned __int128;

constexpr u64 kEmptySlot = ~0ull;       // types.hpp:16
constexpr u32 kMaxArity = GD_MAX_ARITY;

inline u32 bitwidth(u64 v) {  // bits needed to represent v (0 -> 0)
    u32 b = 0;
    while (v) { ++b; v >>= 1; }
    return b;
}

// ---- radix_sort.cu --------------------------------------------------
// Sorts n keys by their low `nbits` bits (all higher bits must be zero).
// Uses b as scratch; returns the buffer holding the sorted keys (a or b).
template <typename K>
K* radix_sort(Ctx& c, K* a, K* b, u64 n, u32 nbits);
// Only the LSD passes [pass_lo, pass_hi) of the same sort (8-bit digits;
// higher key bits are ignored by a pass, so a segment whose top digits are
// equal sorts on its low passes alone).  ballot_io: per-pass ranking choice
// to use, or empty to sample each pass and return the choices; top_hist:
// receives the digit counts of pass pass_hi - 1 (one host sync).
template <typename K>
K* radix_sort_passes(Ctx& c, K* a, K* b, u64 n, u32 nbits, u32 pass_lo, u32 pass_hi, std::vector<char>* ballot_io,
                     std::vector<u64>* top_hist);

// ---- delta.cu (download compression) ----------------------------------
constexpr u32 kDeltaBlock = 64;  // keys per delta block
struct DeltaPacked {
    u64 n = 0, nb = 0, words = 0;
    DevBuf<u64> heads;        // first key of each block
    DevBuf<uint8_t> widths;   // bits per gap of each block
    DevBuf<u64> offs;         // first payload word of each block (nb + 1)
    DevBuf<u64> payload;      // gaps, bit-packed per block
};
// Delta bit-packs n strictly increasing keys; returns the payload words.
u64 delta_pack(Ctx& c, const u64* keys, u64 n, DeltaPacked& out);
// dev_out[k] = d.offs[min(k * blocks_per_chunk, nb)] for k = 0..nchunks.
void delta_chunk_offsets(Ctx& c, const DeltaPacked& d, u64 blocks_per_chunk, u64 nchunks, u64* dev_out);

// Byte-offset blocks (download_delta = 2): each block of kByteBlock keys
// is its first key plus every key's offset from it at the block's byte
// width (1 / 2 / 4 / 8: cls code 0..3), so the host rebuilds rows with
// plain vector loads and adds (host_decode.cpp) instead of a bit-serial
// prefix sum.
constexpr u32 kByteBlock = 32;
struct BytePacked {
    u64 n = 0, nb = 0, bytes = 0;
    DevBuf<u64> heads;       // first key of each block
    DevBuf<uint8_t> cls;     // offset width code of each block
    DevBuf<u64> offs;        // first payload byte of each block (nb + 1)
    DevBuf<uint8_t> payload;
};
u64 byte_pack(Ctx& c, const u64* keys, u64 n, BytePacked& out);
// The same into caller buffers, stream-ordered with no host sync (segmented
// final sort, engine.cu): heads / cls get ceil(n / 32) entries, offs one
// more, payload up to 8 n bytes, unit_offs[k] = offs[min(k * blocks_per_unit,
// nb)] for k = 0..ceil(nb / blocks_per_unit).
void byte_pack_into(Ctx& c, const u64* keys, u64 n, u64* heads, uint8_t* cls, u64* offs, uint8_t* payload,
                    u64 blocks_per_unit, u64* unit_offs);
// dst[k] = src[min(k * stride, n)] for k = 0..m.
void gather_strided(Ctx& c, const u64* src, u64 stride, u64 n, u64 m, u64* dst);
// out[i] = off[lo + i] - off[lo] for i < n1 (a row range's join offsets from 0).
void offsets_rebase(Ctx& c, const u64* off, u64 lo, u64 n1, u64* out);
// dev_out[k] = d.offs[min(k * blocks_per_unit, nb)] for k = 0..nunits.
void byte_unit_offsets(Ctx& c, const BytePacked& d, u64 blocks_per_unit, u64 nunits, u64* dev_out);

// ---- primitives.cu --------------------------------------------------
u64 max_value(Ctx& c, const u64* vals, u64 n);  // 0 for n == 0

// Sorted-unique over a sorted array: out may not alias in. Returns count.
template <typename K>
u64 unique_sorted(Ctx& c, const K* in, u64 n, K* out);

// Encoding: identity or order-preserving dictionary.
struct Encoding {
    u32 bits = 0;      // bits per column
    u32 key_words = 1; // 1 -> u64 keys, 2 -> u128 keys
    bool dict = false;
    const u64* d_dict = nullptr;  // sorted distinct values (dict mode)
    u64 dict_n = 0;
};

template <typename K>
void pack_rows(Ctx& c, const u64* rows, u64 n, u32 arity, const Encoding& e, K* out);
template <typename K>
void unpack_rows(Ctx& c, const K* keys, u64 n, u32 arity, const Encoding& e, u64* out);
// Encodes host-side constants (returns false if a value is absent from the
// dictionary: such a constant can never match).
bool encode_value(Ctx& c, const Encoding& e, u64 v, u64* enc);

// Builds the sorted distinct value set of `vals` (device) into `dict`;
// returns its size.
u64 build_dictionary(Ctx& c, const u64* vals, u64 n, u64 maxval, DevBuf<u64>& dict);

// Reference prefix_hash / slot_key of every row (hash.hpp:28-60).
void prefix_hash_rows(Ctx& c, const u64* rows, u64 n, u32 arity, u32 ncols, u64* out);

// Order-independent digest of packed rows: sum of fmix64(prefix_hash(row)).
template <typename K>
u64 digest_rows(Ctx& c, const K* keys, u64 n, u32 arity, const Encoding& e);

// Stable compaction of keys by a byte flag array; returns kept count.
template <typename K>
u64 compact_flagged(Ctx& c, const K* in, const uint8_t* flags, u64 n, K* out);

// Row-major u64 column permutation: out[r][j] = in[r][perm[j]].
void permute_raw_rows(Ctx& c, const u64* in, u64 n, u32 arity, const u32* perm, u64* out);
// Packs `plen`-column key rows (row-major u64) into prefixes; valid[i] = 0
// when some value cannot occur under the encoding (absent from the
// dictionary / beyond the identity range).
template <typename K>
void pack_keys_checked(Ctx& c, const u64* keys, u64 n, u32 plen, const Encoding& e, K* out, uint8_t* valid);

// Column permutation of packed keys (out[j] = in[perm[j]]), unsorted.
template <typename K>
void permute_keys(Ctx& c, const K* in, u64 n, u32 arity, u32 bits, const u32* perm, K* out);

// ---- dedup.cu -------------------------------------------------------
// Distinct keys of keys[0, m) (unordered) into out via a hash set sized for
// expect_unique; returns their count, or ~0 when more than min(set load
// 1/2, out_cap) distinct keys exist (the caller then sorts all m rows).
u64 hash_dedup(Ctx& c, const u64* keys, u64 m, u64 expect_unique, u64* out, u64 out_cap);

// ---- merge.cu -------------------------------------------------------
struct MergeResult {
    u64 delta_n = 0;     // rows of N kept (not in F, first of their run)
    u64 unique_new = 0;  // distinct rows of N
    bool overlap = false;  // some row of N is in F
};
// One merge-path pass over canonical F and sorted N (duplicates allowed):
//   Fout (nullable) <- F U N,   Dout (nullable) <- unique(N) \ F.
// Fout must hold nf + nn rows, Dout nn rows.
template <typename K>
MergeResult diff_merge(Ctx& c, const K* F, u64 nf, const K* N, u64 nn, K* Fout, K* Dout);
// D = unique(N) \ F (difference + adjacent dedup); Dout holds nn rows.
template <typename K>
MergeResult difference_sorted(Ctx& c, const K* F, u64 nf, const K* N, u64 nn, K* Dout);
// D = unique(N) \ (R_0 U ... U R_k) for sorted disjoint runs R_i.
template <typename K>
MergeResult difference_runs(Ctx& c, const K* const* runs, const u64* ns, u32 nruns, const K* N, u64 nn,
                            K* Dout);
// out = A U B for canonical inputs; returns true if they overlap (only
// checked — one extra synchronization — when check_overlap is set).
template <typename K>
bool merge_disjoint(Ctx& c, const K* A, u64 na, const K* B, u64 nb, K* out, bool check_overlap = false);

// ---- index.cu -------------------------------------------------------
struct Slot {
    u64 tag;  // exact prefix (u64 keys) or 64-bit prefix hash (u128 keys)
    u64 val;  // start (40 bits) | min(len, 2^24-1) << 40
};
constexpr u64 kStartMask = (1ull << 40) - 1;
constexpr u64 kLenSat = (1ull << 24) - 1;

template <typename K>
struct DevIndex {
    DevBuf<Slot> slots;
    u64 slot_count = 0;     // physical slots (probe table)
    u64 logical_slots = 0;  // index_map::slot_count() of the reference sizing rule
    u64 groups = 0;
    u32 plen = 0;
};

template <typename K>
struct IndexView {
    const Slot* slots;
    u64 slot_count;
    const K* rows;
    u64 n;
    u32 arity;
    u32 bits;
    u32 plen;
};

// slot_count rule of build_index (index_map.hpp:87-94).
inline u64 slot_count_for(u64 distinct, double lf) {
    if (distinct == 0) return 1;
    u64 sc = (u64)std::ceil((double)distinct / lf);
    while ((double)distinct > lf * (double)sc) ++sc;
    return sc;
}

// Group starts of the sorted keys by `plen`-column prefix; gs gets
// groups + 1 entries (gs[groups] = n).  Returns groups.
template <typename K>
u64 group_starts(Ctx& c, const K* rows, u64 n, u32 arity, u32 bits, u32 plen, DevBuf<u64>& gs);

template <typename K>
void build_index(Ctx& c, const K* rows, u64 n, u32 arity, u32 bits, u32 plen, double lf,
                 DevIndex<K>& out);

// Lookups of packed prefixes (prefix_of semantics); valid[i] == 0 marks a
// key that cannot exist (e.g. a value absent from the dictionary).
template <typename K>
void index_lookup(Ctx& c, const IndexView<K>& ix, const K* prefixes, const uint8_t* valid,
                  u64 nkeys, u64* out_start, u64* out_count);

// ---- join.cu --------------------------------------------------------
struct DevOperand {
    u32 kind;    // gd_operand_kind
    u32 column;
    u64 value;   // encoded constant
};
struct DevFilter {
    DevOperand lhs, rhs;
    u32 require_equal;
    u32 never;   // constant absent from the dictionary: lhs==rhs impossible
};
struct DevJoin {
    u32 jcc;
    u32 proj_arity;
    u32 nfilters;
    u32 bits;
    u32 outer_arity;
    u32 outer_identity;
    u32 inner_arity;
    u32 reserved;
    u32 outer_perm[kMaxArity];
    DevOperand proj[kMaxArity];
    DevFilter filters[GD_MAX_FILTERS];
};

// Pass 1: per outer row, the inner match range (start, count) via the
// index (or the whole inner when jcc == 0), fused with the exclusive scan
// of counts.  row_off gets n+1 entries.  Returns the candidate total.
template <typename K>
u64 join_probe(Ctx& c, const K* outer, u64 n, const DevJoin& jd, const IndexView<K>* ix,
               u64 inner_n, u64* row_start, u64* row_off);

// Pass 2: load-balanced materialize of `total` candidates into out (plus a
// per-candidate filter flag when jd.nfilters > 0).
template <typename K>
void join_materialize(Ctx& c, const K* outer, u64 n, const K* inner, const DevJoin& jd,
                      const u64* row_start, const u64* row_off, u64 total, K* out,
                      uint8_t* flags);

// select_project (ra.hpp:267-293) over packed rows: filter + project +
// stable compaction.  Returns rows written.
template <typename K>
u64 select_project(Ctx& c, const K* rows, u64 n, const DevJoin& jd, K* out);

// Owner rank of each packed key (multi-GPU partitioning).
template <typename K>
void owner_of(Ctx& c, const K* keys, u64 n, u32 nranks, u32* owner);
// flags[i] = (owner[i] == k)
void owner_flags(Ctx& c, const u32* owner, u64 n, u32 k, uint8_t* flags);

}  // namespace gd
