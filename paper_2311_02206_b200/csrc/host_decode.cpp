// host_decode.cpp — row rebuild of byte-offset blocks (host_decode.h).
//
// A full block of 32 keys at width w is 32 w payload bytes; on an AVX-512
// host every 8 keys are one widening load (vpmovzx), one add of the block's
// first key, a shift and two masks for the two columns, two permutes into
// row order and two 64-byte non-temporal stores — about two instructions
// per row, so the host side runs at its memory write bandwidth (16 B per
// row) instead of being bound by a bit-serial decode.
#include "host_decode.h"

#include <string.h>

#if defined(__x86_64__)
#include <immintrin.h>
#endif

namespace gd {

namespace {

constexpr uint32_t kBlock = 32;

inline uint64_t off_at(const uint8_t* p, uint32_t code, uint32_t i) {
    switch (code) {
        case 0: return p[i];
        case 1: {
            uint16_t v;
            memcpy(&v, p + 2 * i, 2);
            return v;
        }
        case 2: {
            uint32_t v;
            memcpy(&v, p + 4 * i, 4);
            return v;
        }
        default: {
            uint64_t v;
            memcpy(&v, p + 8 * i, 8);
            return v;
        }
    }
}

// Any arity, any alignment, partial blocks.
void decode_block_scalar(uint64_t head, uint32_t code, const uint8_t* p, uint32_t cnt, uint32_t ar, uint32_t bits,
                         uint64_t mask, uint64_t* dst) {
    for (uint32_t i = 0; i < cnt; ++i, dst += ar) {
        const uint64_t key = head + off_at(p, code, i);
        for (uint32_t col = 0; col < ar; ++col) dst[col] = (key >> ((ar - 1 - col) * bits)) & mask;
    }
}

#if defined(__x86_64__)
// Arity 2, 16-byte aligned rows, full blocks (64-byte stores where a block's
// rows start a line).
__attribute__((target("avx512f,avx512dq"))) void decode_avx512(const uint64_t* heads, const uint8_t* cls,
                                                      const uint8_t* payload, uint64_t first_row, uint64_t nblocks,
                                                      uint64_t n_total, uint32_t bits, uint64_t mask, uint64_t* out) {
    const __m512i vmask = _mm512_set1_epi64((long long)mask);
    const __m128i sh = _mm_cvtsi32_si128((int)bits);
    const __m512i i0 = _mm512_set_epi64(11, 3, 10, 2, 9, 1, 8, 0);  // rows 0-3: (hi0, lo0, hi1, lo1, ...)
    const __m512i i1 = _mm512_set_epi64(15, 7, 14, 6, 13, 5, 12, 4);
    const uint8_t* p = payload;
    for (uint64_t b = 0; b < nblocks; ++b) {
        const uint64_t row = first_row + b * kBlock;
        const uint32_t cnt = (uint32_t)(n_total - row < kBlock ? n_total - row : kBlock);
        const uint32_t code = cls[b];
        uint64_t* dst = out + 2 * row;
        if (cnt < kBlock) {
            decode_block_scalar(heads[b], code, p, cnt, 2, bits, mask, dst);
            p += (uint64_t)cnt << code;
            continue;
        }
        const __m512i head = _mm512_set1_epi64((long long)heads[b]);
        const bool line = !(reinterpret_cast<uintptr_t>(dst) & 63);  // else 16-byte aligned rows
#pragma GCC unroll 4
        for (int q = 0; q < 4; ++q) {
            __m512i off;
            switch (code) {
                case 0: off = _mm512_cvtepu8_epi64(_mm_loadl_epi64(reinterpret_cast<const __m128i*>(p + 8 * q))); break;
                case 1: off = _mm512_cvtepu16_epi64(_mm_loadu_si128(reinterpret_cast<const __m128i*>(p + 16 * q))); break;
                case 2: off = _mm512_cvtepu32_epi64(_mm256_loadu_si256(reinterpret_cast<const __m256i*>(p + 32 * q))); break;
                default: off = _mm512_loadu_si512(p + 64 * q); break;
            }
            const __m512i key = _mm512_add_epi64(head, off);
            const __m512i hi = _mm512_and_si512(_mm512_srl_epi64(key, sh), vmask);
            const __m512i lo = _mm512_and_si512(key, vmask);
            const __m512i r0 = _mm512_permutex2var_epi64(hi, i0, lo), r1 = _mm512_permutex2var_epi64(hi, i1, lo);
            if (line) {
                _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + 16 * q), r0);
                _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + 16 * q + 8), r1);
            } else {  // rows of a segment that starts off a 64-byte line: one 16-byte store per row
                __m128i* d = reinterpret_cast<__m128i*>(dst + 16 * q);
                _mm_stream_si128(d + 0, _mm512_extracti64x2_epi64(r0, 0));
                _mm_stream_si128(d + 1, _mm512_extracti64x2_epi64(r0, 1));
                _mm_stream_si128(d + 2, _mm512_extracti64x2_epi64(r0, 2));
                _mm_stream_si128(d + 3, _mm512_extracti64x2_epi64(r0, 3));
                _mm_stream_si128(d + 4, _mm512_extracti64x2_epi64(r1, 0));
                _mm_stream_si128(d + 5, _mm512_extracti64x2_epi64(r1, 1));
                _mm_stream_si128(d + 6, _mm512_extracti64x2_epi64(r1, 2));
                _mm_stream_si128(d + 7, _mm512_extracti64x2_epi64(r1, 3));
            }
        }
        p += (uint64_t)kBlock << code;
    }
    _mm_sfence();
}

bool has_avx512() {
    static const bool v = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512dq");
    return v;
}
#endif

}  // namespace

bool byte_decode_vectorized() {
#if defined(__x86_64__)
    return has_avx512();
#else
    return false;
#endif
}

void byte_decode_rows(const unsigned long long* heads_, const uint8_t* cls, const uint8_t* payload,
                      uint64_t first_row, uint64_t nblocks, uint64_t n_total, uint32_t ar, uint32_t bits,
                      unsigned long long* out_) {
    static_assert(sizeof(unsigned long long) == sizeof(uint64_t), "u64 layout");
    const uint64_t* heads = reinterpret_cast<const uint64_t*>(heads_);
    uint64_t* out = reinterpret_cast<uint64_t*>(out_);
    const uint64_t mask = bits >= 64 ? ~0ull : (1ull << bits) - 1;
#if defined(__x86_64__)
    if (ar == 2 && !(reinterpret_cast<uintptr_t>(out) & 15) && has_avx512()) {
        decode_avx512(heads, cls, payload, first_row, nblocks, n_total, bits, mask, out);
        return;
    }
#endif
    const uint8_t* p = payload;
    for (uint64_t b = 0; b < nblocks; ++b) {
        const uint64_t row = first_row + b * kBlock;
        const uint32_t cnt = (uint32_t)(n_total - row < kBlock ? n_total - row : kBlock);
        decode_block_scalar(heads[b], cls[b], p, cnt, ar, bits, mask, out + ar * row);
        p += (uint64_t)cnt << cls[b];
    }
}

}  // namespace gd
