// host_decode.h — host side of the byte-offset download (download_delta = 2,
// engine.cu download_bytes_rows): rebuilds rows from byte-offset blocks
// (delta.cu byte_pack) with vector loads, adds and non-temporal stores.
// Plain C++ (compiled by the host compiler, AVX-512 chosen at run time).
#pragma once

#include <stdint.h>

namespace gd {

// Blocks [0, nblocks) of one staged unit: heads[i] / cls[i] of block i,
// payload = its first offset byte; block i holds rows first_row + 32 i ...
// (min(32, n_total - that) of them).  Row r is written to out + r * ar,
// column j = (key >> (ar - 1 - j) * bits) & mask(bits).
void byte_decode_rows(const unsigned long long* heads, const uint8_t* cls, const uint8_t* payload, uint64_t first_row,
                      uint64_t nblocks, uint64_t n_total, uint32_t ar, uint32_t bits, unsigned long long* out);

// True when the AVX-512 decoder is used (x86-64 host with AVX-512F/DQ).
bool byte_decode_vectorized();

}  // namespace gd
