// primitives.cu — encoding (identity / order-preserving dictionary bit
// packing), reductions, adjacent-unique, compaction, the reference's
// prefix hash, relation digests and column permutation of packed keys.
#include "dev_common.cuh"
#include "ops.h"
#include "select.cuh"

namespace gd {

namespace {

__global__ void max_kernel(const u64* __restrict__ v, u64 n, u64* out) {
    u64 m = 0;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        m = max(m, v[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane_id() == 0) atomicMax(out, m);
}

__device__ __forceinline__ u64 dict_rank(const u64* __restrict__ dict, u64 dn, u64 v) {
    u64 lo = 0, hi = dn;
    while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (dict[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <typename K>
__global__ void pack_kernel(const u64* __restrict__ rows, u64 n, u32 arity, u32 bits,
                            const u64* __restrict__ dict, u64 dn, K* __restrict__ out) {
    for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (u64)gridDim.x * blockDim.x) {
        K key = 0;
        for (u32 c = 0; c < arity; ++c) {
            u64 v = rows[r * arity + c];
            if (dict) v = dict_rank(dict, dn, v);
            key |= (K)v << ((arity - 1 - c) * bits);
        }
        out[r] = key;
    }
}

template <typename K>
__global__ void unpack_kernel(const K* __restrict__ keys, u64 n, u32 arity, u32 bits,
                              const u64* __restrict__ dict, u64* __restrict__ out) {
    for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (u64)gridDim.x * blockDim.x) {
        const K key = keys[r];
        for (u32 c = 0; c < arity; ++c) {
            u64 v = col_of(key, arity, bits, c);
            if (dict) v = dict[v];
            out[r * arity + c] = v;
        }
    }
}

__global__ void dict_lookup_kernel(const u64* __restrict__ dict, u64 dn, u64 v, u64* out) {
    const u64 r = dict_rank(dict, dn, v);
    out[0] = r;
    out[1] = (r < dn && dict[r] == v) ? 1 : 0;
}

// hash.hpp:28-53, bit-exact.
__device__ __forceinline__ u64 rotl64(u64 x, int r) { return (x << r) | (x >> (64 - r)); }

__device__ u64 ref_prefix_hash(const u64* cols, u32 n) {
    const u64 c1 = 0x87c37b91114253d5ULL, c2 = 0x4cf5ad432745937fULL;
    u64 h1 = 0, h2 = 0;
    for (u32 i = 0; i + 1 < n; i += 2) {
        u64 k1 = cols[i], k2 = cols[i + 1];
        k1 *= c1; k1 = rotl64(k1, 31); k1 *= c2; h1 ^= k1;
        h1 = rotl64(h1, 27); h1 += h2; h1 = h1 * 5 + 0x52dce729;
        k2 *= c2; k2 = rotl64(k2, 33); k2 *= c1; h2 ^= k2;
        h2 = rotl64(h2, 31); h2 += h1; h2 = h2 * 5 + 0x38495ab5;
    }
    if (n % 2) {
        u64 k1 = cols[n - 1];
        k1 *= c1; k1 = rotl64(k1, 31); k1 *= c2; h1 ^= k1;
    }
    const u64 len = (u64)n * 8u;
    h1 ^= len; h2 ^= len;
    h1 += h2; h2 += h1;
    h1 = fmix64(h1);
    h2 = fmix64(h2);
    return h1 + h2;
}

__global__ void prefix_hash_kernel(const u64* __restrict__ rows, u64 n, u32 arity, u32 ncols,
                                   u64* __restrict__ out) {
    for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (u64)gridDim.x * blockDim.x) {
        u64 cols[kMaxArity];
        for (u32 c = 0; c < ncols; ++c) cols[c] = rows[r * arity + c];
        const u64 h = ref_prefix_hash(cols, ncols);
        out[r] = h == kEmptySlot ? kEmptySlot - 1 : h;  // slot_key, hash.hpp:57-60
    }
}

template <typename K>
__global__ void digest_kernel(const K* __restrict__ keys, u64 n, u32 arity, u32 bits,
                              const u64* __restrict__ dict, u64* out) {
    u64 acc = 0;
    for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (u64)gridDim.x * blockDim.x) {
        u64 cols[kMaxArity];
        const K key = keys[r];
        for (u32 c = 0; c < arity; ++c) {
            u64 v = col_of(key, arity, bits, c);
            cols[c] = dict ? dict[v] : v;
        }
        acc += fmix64(ref_prefix_hash(cols, arity));
    }
    acc = warp_sum(acc);
    if (lane_id() == 0) atomicAdd(out, acc);
}

template <typename K>
__global__ void permute_kernel(const K* __restrict__ in, u64 n, u32 arity, u32 bits, Perm8 perm,
                               K* __restrict__ out) {
    for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (u64)gridDim.x * blockDim.x) {
        const K key = in[r];
        K o = 0;
        for (u32 j = 0; j < arity; ++j)
            o |= (K)col_of(key, arity, bits, perm.p[j]) << ((arity - 1 - j) * bits);
        out[r] = o;
    }
}

__global__ void permute_raw_kernel(const u64* __restrict__ in, u64 n, u32 arity, Perm8 perm,
                                   u64* __restrict__ out) {
    for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (u64)gridDim.x * blockDim.x)
        for (u32 j = 0; j < arity; ++j) out[r * arity + j] = in[r * arity + perm.p[j]];
}

template <typename K>
__global__ void pack_keys_kernel(const u64* __restrict__ keys, u64 n, u32 plen, u32 bits,
                                 const u64* __restrict__ dict, u64 dn, K* __restrict__ out,
                                 uint8_t* __restrict__ valid) {
    const u64 lim = bits >= 64 ? ~0ull : (1ull << bits) - 1;  // all-ones is never a value
    for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (u64)gridDim.x * blockDim.x) {
        K key = 0;
        bool ok = true;
        for (u32 c = 0; c < plen; ++c) {
            u64 v = keys[r * plen + c];
            if (dict) {
                const u64 rk = dict_rank(dict, dn, v);
                ok &= rk < dn && dict[rk] == v;
                v = rk;
            } else {
                ok &= v < lim;
            }
            key |= (K)(v & lim) << ((plen - 1 - c) * bits);
        }
        out[r] = key;
        valid[r] = ok ? 1 : 0;
    }
}

template <typename K>
struct UniquePred {
    const K* in;
    __device__ bool operator()(u64 i) const { return i == 0 || in[i] != in[i - 1]; }
};
template <typename K>
struct CopyEmit {
    const K* in;
    K* out;
    __device__ void operator()(u64 i, u64 pos) const { out[pos] = in[i]; }
};
struct FlagPred {
    const uint8_t* f;
    __device__ bool operator()(u64 i) const { return f[i] != 0; }
};

inline int grid_for(const Ctx& c, u64 n, int threads = 256) {
    const u64 want = (n + threads - 1) / threads;
    return (int)std::max<u64>(1, std::min<u64>(want, (u64)c.num_sms * 8));
}

}  // namespace

u64 max_value(Ctx& c, const u64* vals, u64 n) {
    if (n == 0) return 0;
    DevBuf<u64> out(c, 1);
    c.memset(out.p, 0, sizeof(u64));
    max_kernel<<<grid_for(c, n), 256, 0, c.stream>>>(vals, n, out.p);
    c.check_launch();
    unsigned long long m;
    c.read_words(&m, out.p, 1);
    return m;
}

template <typename K>
u64 unique_sorted(Ctx& c, const K* in, u64 n, K* out) {
    return run_select(c, n, UniquePred<K>{in}, CopyEmit<K>{in, out});
}

template <typename K>
u64 compact_flagged(Ctx& c, const K* in, const uint8_t* flags, u64 n, K* out) {
    return run_select(c, n, FlagPred{flags}, CopyEmit<K>{in, out});
}

template <typename K>
void pack_rows(Ctx& c, const u64* rows, u64 n, u32 arity, const Encoding& e, K* out) {
    if (n == 0) return;
    pack_kernel<K><<<grid_for(c, n), 256, 0, c.stream>>>(rows, n, arity, e.bits,
                                                          e.dict ? e.d_dict : nullptr, e.dict_n, out);
    c.check_launch();
}

template <typename K>
void unpack_rows(Ctx& c, const K* keys, u64 n, u32 arity, const Encoding& e, u64* out) {
    if (n == 0) return;
    unpack_kernel<K><<<grid_for(c, n), 256, 0, c.stream>>>(keys, n, arity, e.bits,
                                                            e.dict ? e.d_dict : nullptr, out);
    c.check_launch();
}

bool encode_value(Ctx& c, const Encoding& e, u64 v, u64* enc) {
    if (!e.dict) {
        *enc = v;
        return e.bits >= 64 || (v + 1) < (1ull << e.bits);
    }
    DevBuf<u64> out(c, 2);
    dict_lookup_kernel<<<1, 1, 0, c.stream>>>(e.d_dict, e.dict_n, v, out.p);
    c.check_launch();
    unsigned long long r[2];
    c.read_words(r, out.p, 2);
    *enc = r[0];
    return r[1] != 0;
}

u64 build_dictionary(Ctx& c, const u64* vals, u64 n, u64 maxval, DevBuf<u64>& dict) {
    DevBuf<u64> a(c, n), b(c, n);
    c.d2d(a.p, vals, n * sizeof(u64));
    u64* sorted = radix_sort<u64>(c, a.p, b.p, n, bitwidth(maxval));
    dict.reserve_discard(c, n);
    return unique_sorted<u64>(c, sorted, n, dict.p);
}

void prefix_hash_rows(Ctx& c, const u64* rows, u64 n, u32 arity, u32 ncols, u64* out) {
    if (n == 0) return;
    prefix_hash_kernel<<<grid_for(c, n), 256, 0, c.stream>>>(rows, n, arity, ncols, out);
    c.check_launch();
}

template <typename K>
u64 digest_rows(Ctx& c, const K* keys, u64 n, u32 arity, const Encoding& e) {
    if (n == 0) return 0;
    DevBuf<u64> out(c, 1);
    c.memset(out.p, 0, sizeof(u64));
    digest_kernel<K><<<grid_for(c, n), 256, 0, c.stream>>>(keys, n, arity, e.bits,
                                                            e.dict ? e.d_dict : nullptr, out.p);
    c.check_launch();
    unsigned long long d;
    c.read_words(&d, out.p, 1);
    return d;
}

void permute_raw_rows(Ctx& c, const u64* in, u64 n, u32 arity, const u32* perm, u64* out) {
    if (n == 0) return;
    Perm8 p{};
    for (u32 i = 0; i < arity; ++i) p.p[i] = perm[i];
    permute_raw_kernel<<<grid_for(c, n), 256, 0, c.stream>>>(in, n, arity, p, out);
    c.check_launch();
}

template <typename K>
void pack_keys_checked(Ctx& c, const u64* keys, u64 n, u32 plen, const Encoding& e, K* out, uint8_t* valid) {
    if (n == 0) return;
    pack_keys_kernel<K><<<grid_for(c, n), 256, 0, c.stream>>>(keys, n, plen, e.bits, e.dict ? e.d_dict : nullptr,
                                                               e.dict_n, out, valid);
    c.check_launch();
}

template <typename K>
void permute_keys(Ctx& c, const K* in, u64 n, u32 arity, u32 bits, const u32* perm, K* out) {
    if (n == 0) return;
    Perm8 p{};
    for (u32 i = 0; i < arity; ++i) p.p[i] = perm[i];
    permute_kernel<K><<<grid_for(c, n), 256, 0, c.stream>>>(in, n, arity, bits, p, out);
    c.check_launch();
}

#define GD_INST(K)                                                                          \
    template u64 unique_sorted<K>(Ctx&, const K*, u64, K*);                                 \
    template u64 compact_flagged<K>(Ctx&, const K*, const uint8_t*, u64, K*);               \
    template void pack_rows<K>(Ctx&, const u64*, u64, u32, const Encoding&, K*);            \
    template void unpack_rows<K>(Ctx&, const K*, u64, u32, const Encoding&, u64*);          \
    template u64 digest_rows<K>(Ctx&, const K*, u64, u32, const Encoding&);                 \
    template void permute_keys<K>(Ctx&, const K*, u64, u32, u32, const u32*, K*);               \
    template void pack_keys_checked<K>(Ctx&, const u64*, u64, u32, const Encoding&, K*, uint8_t*);
GD_INST(u64)
GD_INST(u128)
#undef GD_INST

}  // namespace gd
