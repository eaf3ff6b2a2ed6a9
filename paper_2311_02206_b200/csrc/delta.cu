// delta.cu — delta bit-packing of a canonical (strictly increasing) key array
// for the host download (engine.cu download_packed).
//
// The output relation crosses PCIe as packed keys; sorted keys differ by
// small gaps (C2: mostly the distance to the next reachable node), so each
// block of kDeltaBlock keys is sent as its first key plus the remaining
// gaps at the block's own bit width — ~3 bytes per row instead of 8 for
// C2 — and host threads rebuild the keys (a prefix sum) while unpacking
// them into rows.  PCIe was the bound of the e2e download.
//
//   heads[b]   first key of block b
//   widths[b]  bits per gap in block b (0..64)
//   offs[b]    first payload word of block b (exclusive scan of
//              ceil((cnt_b - 1) * w_b / 64)), offs[nb] = total words
//   payload    gap i of block b (i = 0..cnt_b-2) at bits [i*w, i*w + w) of
//              the block's words, little-endian within and across words
#include "dev_common.cuh"
#include "ops.h"

namespace gd {

namespace {

constexpr u32 kDB = kDeltaBlock;  // keys per block (64: two per lane)

__device__ __forceinline__ u32 bits_of(u64 v) { return v ? 64 - __clzll(v) : 0; }

// One warp per block: widths and payload word counts.
__global__ void delta_width_kernel(const u64* __restrict__ keys, u64 n, u64 nb, uint8_t* __restrict__ widths,
                                   u64* __restrict__ words) {
    const u64 warp = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const u32 lane = lane_id();
    for (u64 b = warp; b < nb; b += ((u64)gridDim.x * blockDim.x) >> 5) {
        const u64 base = b * kDB;
        const u64 cnt = min((u64)kDB, n - base);
        const u64 i0 = base + 2 * lane, i1 = i0 + 1;
        const u64 k0 = 2 * lane < cnt ? keys[i0] : 0, k1 = 2 * lane + 1 < cnt ? keys[i1] : 0;
        const u64 prev = __shfl_up_sync(0xffffffffu, k1, 1);  // key 2*lane - 1
        u32 w = 0;
        if (lane > 0 && 2 * lane < cnt) w = bits_of(k0 - prev);
        if (2 * lane + 1 < cnt) w = max(w, bits_of(k1 - k0));
#pragma unroll
        for (int o = 16; o; o >>= 1) w = max(w, __shfl_xor_sync(0xffffffffu, w, o));
        if (lane == 0) {
            widths[b] = (uint8_t)w;
            words[b] = ((cnt - 1) * w + 63) / 64;
        }
    }
}

// Exclusive scan of u64 counts in place, three launches: tile sums, one CTA
// over the tile sums, tile-local scans with the tile base.
constexpr int kScanT = 256, kScanI = 16;
constexpr u64 kScanTile = (u64)kScanT * kScanI;

__global__ void __launch_bounds__(kScanT) scan_tile_sums_kernel(const u64* __restrict__ v, u64 n,
                                                                u64* __restrict__ sums) {
    __shared__ u64 red[kScanT / 32];
    const u64 t0 = (u64)blockIdx.x * kScanTile;
    u64 s = 0;
    for (int i = 0; i < kScanI; ++i) {
        const u64 j = t0 + (u64)i * kScanT + threadIdx.x;
        if (j < n) s += v[j];
    }
    s = warp_sum(s);
    if (lane_id() == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        u64 t = 0;
        for (int w = 0; w < kScanT / 32; ++w) t += red[w];
        sums[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(1024) scan_sums_kernel(u64* __restrict__ sums, u64 m, u64* __restrict__ total) {
    __shared__ u64 tmp[1024 / 32 + 1];
    u64 carry = 0;
    for (u64 b = 0; b < m; b += 1024) {
        const u64 j = b + threadIdx.x;
        const u64 v = j < m ? sums[j] : 0;
        u64 all;
        const u64 ex = block_exclusive_scan<u64, 1024>(v, all, tmp);
        if (j < m) sums[j] = carry + ex;
        carry += all;
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(kScanT) scan_tiles_kernel(const u64* __restrict__ v, u64 n,
                                                            const u64* __restrict__ sums, u64* __restrict__ out) {
    __shared__ u64 tmp[kScanT / 32 + 1];
    const u64 first = (u64)blockIdx.x * kScanTile + (u64)threadIdx.x * kScanI;
    u64 c[kScanI];
    u64 s = 0;
#pragma unroll
    for (int i = 0; i < kScanI; ++i) {
        c[i] = first + i < n ? v[first + i] : 0;
        s += c[i];
    }
    u64 all;
    u64 off = sums[blockIdx.x] + block_exclusive_scan<u64, kScanT>(s, all, tmp);
#pragma unroll
    for (int i = 0; i < kScanI; ++i) {
        if (first + i < n) out[first + i] = off;
        off += c[i];
    }
}

// One warp per block: the gaps OR-ed into the block's words in shared
// memory (a gap straddles at most two words), then written out whole.
__global__ void __launch_bounds__(256) delta_pack_kernel(const u64* __restrict__ keys, u64 n, u64 nb,
                                                         const uint8_t* __restrict__ widths, const u64* __restrict__ offs,
                                                         u64* __restrict__ heads, u64* __restrict__ payload) {
    __shared__ unsigned long long sw[256 / 32][kDB];
    const u32 lane = lane_id(), wl = threadIdx.x >> 5;
    unsigned long long* w = sw[wl];
    const u64 warp = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (u64 b = warp; b < nb; b += ((u64)gridDim.x * blockDim.x) >> 5) {
        const u64 base = b * kDB;
        const u64 cnt = min((u64)kDB, n - base);
        const u32 width = widths[b];
        const u64 nw = ((cnt - 1) * width + 63) / 64;
        w[lane] = 0;
        w[lane + 32] = 0;
        __syncwarp();
        const u64 k0 = 2 * lane < cnt ? keys[base + 2 * lane] : 0;
        const u64 k1 = 2 * lane + 1 < cnt ? keys[base + 2 * lane + 1] : 0;
        const u64 prev = __shfl_up_sync(0xffffffffu, k1, 1);
        if (lane == 0) heads[b] = k0;
        auto put = [&](u64 gi, u64 d) {  // gap index gi = key index - 1
            const u64 pos = gi * width;
            const u32 q = (u32)(pos >> 6), sh = (u32)(pos & 63);
            atomicOr(&w[q], d << sh);
            if (sh && sh + width > 64) atomicOr(&w[q + 1], d >> (64 - sh));
        };
        if (width) {
            if (lane > 0 && 2 * lane < cnt) put(2 * lane - 1, k0 - prev);
            if (2 * lane + 1 < cnt) put(2 * lane, k1 - k0);
        }
        __syncwarp();
        u64* out = payload + offs[b];
        for (u32 j = lane; j < nw; j += 32) out[j] = w[j];
        __syncwarp();
    }
}

// ---- byte-offset blocks (download_delta = 2) ----
// A warp takes kBW consecutive blocks of kByteBlock keys per step, their
// loads issued together (one key per lane per block).
constexpr int kBW = 4;

// The block's offset class (bytes per offset from its first key: 1 / 2 / 4
// / 8, code 0..3) and its payload bytes.
__global__ void byte_class_kernel(const u64* __restrict__ keys, u64 n, u64 nb, uint8_t* __restrict__ cls,
                                  u64* __restrict__ bytes) {
    const u64 warp = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const u64 nw = ((u64)gridDim.x * blockDim.x) >> 5;
    const u32 lane = lane_id();
    for (u64 b0 = warp * kBW; b0 < nb; b0 += nw * kBW) {
        u64 k[kBW];
        u32 cnt[kBW];
#pragma unroll
        for (int q = 0; q < kBW; ++q) {
            const u64 b = b0 + q;
            cnt[q] = b < nb ? (u32)min((u64)kByteBlock, n - b * kByteBlock) : 0u;
            k[q] = lane < cnt[q] ? keys[b * kByteBlock + lane] : 0;
        }
#pragma unroll
        for (int q = 0; q < kBW; ++q) {
            if (!cnt[q]) break;  // warp-uniform
            const u64 head = __shfl_sync(0xffffffffu, k[q], 0);
            const u64 last = __shfl_sync(0xffffffffu, k[q], cnt[q] - 1);
            if (lane == q) {
                const u64 r = last - head;
                const u32 code = r < (1ull << 8) ? 0 : r < (1ull << 16) ? 1 : r < (1ull << 32) ? 2 : 3;
                cls[b0 + q] = (uint8_t)code;
                bytes[b0 + q] = (u64)cnt[q] << code;
            }
        }
    }
}

// The first key to heads, offset i (key_i - head) to payload[offs[b] + i *
// width], little-endian.
__global__ void byte_pack_kernel(const u64* __restrict__ keys, u64 n, u64 nb, const uint8_t* __restrict__ cls,
                                 const u64* __restrict__ offs, u64* __restrict__ heads, uint8_t* __restrict__ payload) {
    const u64 warp = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const u64 nw = ((u64)gridDim.x * blockDim.x) >> 5;
    const u32 lane = lane_id();
    for (u64 b0 = warp * kBW; b0 < nb; b0 += nw * kBW) {
        u64 k[kBW], base[kBW];
        u32 cnt[kBW], code[kBW];
#pragma unroll
        for (int q = 0; q < kBW; ++q) {
            const u64 b = b0 + q;
            cnt[q] = b < nb ? (u32)min((u64)kByteBlock, n - b * kByteBlock) : 0u;
            k[q] = lane < cnt[q] ? keys[b * kByteBlock + lane] : 0;
            code[q] = cnt[q] ? cls[b] : 0u;
            base[q] = cnt[q] ? offs[b] : 0ull;
        }
#pragma unroll
        for (int q = 0; q < kBW; ++q) {
            if (!cnt[q]) break;  // warp-uniform
            const u64 head = __shfl_sync(0xffffffffu, k[q], 0);
            if (lane == 0) heads[b0 + q] = head;
            if (lane < cnt[q]) {
                const u64 o = k[q] - head;
                uint8_t* p = payload + base[q] + ((u64)lane << code[q]);
                switch (code[q]) {
                    case 0: *p = (uint8_t)o; break;
                    case 1: for (int i = 0; i < 2; ++i) p[i] = (uint8_t)(o >> (8 * i)); break;
                    case 2: for (int i = 0; i < 4; ++i) p[i] = (uint8_t)(o >> (8 * i)); break;
                    default: for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(o >> (8 * i)); break;
                }
            }
        }
    }
}

__global__ void gather_kernel(const u64* __restrict__ src, u64 stride, u64 n, u64 m, u64* __restrict__ dst) {
    const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i <= m) dst[i] = src[min(i * stride, n)];
}

}  // namespace

u64 delta_pack(Ctx& c, const u64* keys, u64 n, DeltaPacked& out) {
    const u64 nb = (n + kDB - 1) / kDB;
    out.nb = nb;
    out.n = n;
    out.heads = DevBuf<u64>(c, std::max<u64>(nb, 1));
    out.widths = DevBuf<uint8_t>(c, std::max<u64>(nb, 1));
    out.offs = DevBuf<u64>(c, nb + 1);
    if (!nb) {
        c.memset(out.offs.p, 0, sizeof(u64));
        return 0;
    }
    DevBuf<u64> words(c, nb);
    const int grid = c.num_sms * 8;
    delta_width_kernel<<<grid, 256, 0, c.stream>>>(keys, n, nb, out.widths.p, words.p);
    c.check_launch();
    const u64 tiles = (nb + kScanTile - 1) / kScanTile;
    DevBuf<u64> sums(c, tiles);
    scan_tile_sums_kernel<<<(unsigned)tiles, kScanT, 0, c.stream>>>(words.p, nb, sums.p);
    c.check_launch();
    scan_sums_kernel<<<1, 1024, 0, c.stream>>>(sums.p, tiles, out.offs.p + nb);
    c.check_launch();
    scan_tiles_kernel<<<(unsigned)tiles, kScanT, 0, c.stream>>>(words.p, nb, sums.p, out.offs.p);
    c.check_launch();
    unsigned long long total = 0;
    c.read_words(&total, out.offs.p + nb, 1);
    out.payload = DevBuf<u64>(c, std::max<u64>(total, 1));
    out.words = total;
    delta_pack_kernel<<<grid, 256, 0, c.stream>>>(keys, n, nb, out.widths.p, out.offs.p, out.heads.p,
                                                   out.payload.p);
    c.check_launch();
    return total;
}

u64 byte_pack(Ctx& c, const u64* keys, u64 n, BytePacked& out) {
    const u64 nb = (n + kByteBlock - 1) / kByteBlock;
    out.nb = nb;
    out.n = n;
    out.heads = DevBuf<u64>(c, std::max<u64>(nb, 1));
    out.cls = DevBuf<uint8_t>(c, std::max<u64>(nb, 1));
    out.offs = DevBuf<u64>(c, nb + 1);
    if (!nb) {
        c.memset(out.offs.p, 0, sizeof(u64));
        out.bytes = 0;
        return 0;
    }
    DevBuf<u64> bytes(c, nb);
    const int grid = c.num_sms * 8;
    byte_class_kernel<<<grid, 256, 0, c.stream>>>(keys, n, nb, out.cls.p, bytes.p);
    c.check_launch();
    const u64 tiles = (nb + kScanTile - 1) / kScanTile;
    DevBuf<u64> sums(c, tiles);
    scan_tile_sums_kernel<<<(unsigned)tiles, kScanT, 0, c.stream>>>(bytes.p, nb, sums.p);
    c.check_launch();
    scan_sums_kernel<<<1, 1024, 0, c.stream>>>(sums.p, tiles, out.offs.p + nb);
    c.check_launch();
    scan_tiles_kernel<<<(unsigned)tiles, kScanT, 0, c.stream>>>(bytes.p, nb, sums.p, out.offs.p);
    c.check_launch();
    unsigned long long total = 0;
    c.read_words(&total, out.offs.p + nb, 1);
    out.payload = DevBuf<uint8_t>(c, std::max<u64>(total, 1));
    out.bytes = total;
    byte_pack_kernel<<<grid, 256, 0, c.stream>>>(keys, n, nb, out.cls.p, out.offs.p, out.heads.p, out.payload.p);
    c.check_launch();
    return total;
}

void byte_pack_into(Ctx& c, const u64* keys, u64 n, u64* heads, uint8_t* cls, u64* offs, uint8_t* payload,
                    u64 blocks_per_unit, u64* unit_offs) {
    const u64 nb = (n + kByteBlock - 1) / kByteBlock;
    if (!nb) return;
    DevBuf<u64> bytes(c, nb);
    const int grid = (int)std::min<u64>((u64)c.num_sms * 8, (nb + 8 * kBW - 1) / (8 * kBW));
    byte_class_kernel<<<grid, 256, 0, c.stream>>>(keys, n, nb, cls, bytes.p);
    c.check_launch();
    const u64 tiles = (nb + kScanTile - 1) / kScanTile;
    DevBuf<u64> sums(c, tiles);
    scan_tile_sums_kernel<<<(unsigned)tiles, kScanT, 0, c.stream>>>(bytes.p, nb, sums.p);
    c.check_launch();
    scan_sums_kernel<<<1, 1024, 0, c.stream>>>(sums.p, tiles, offs + nb);
    c.check_launch();
    scan_tiles_kernel<<<(unsigned)tiles, kScanT, 0, c.stream>>>(bytes.p, nb, sums.p, offs);
    c.check_launch();
    byte_pack_kernel<<<grid, 256, 0, c.stream>>>(keys, n, nb, cls, offs, heads, payload);
    c.check_launch();
    const u64 nunits = (nb + blocks_per_unit - 1) / blocks_per_unit;
    gather_kernel<<<(unsigned)((nunits + 1 + 255) / 256), 256, 0, c.stream>>>(offs, blocks_per_unit, nb, nunits,
                                                                             unit_offs);
    c.check_launch();
}

__global__ void rebase_kernel(const u64* __restrict__ off, u64 lo, u64 n1, u64* __restrict__ out) {
    const u64 base = off[lo];
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n1; i += (u64)gridDim.x * blockDim.x)
        out[i] = off[lo + i] - base;
}

void gather_strided(Ctx& c, const u64* src, u64 stride, u64 n, u64 m, u64* dst) {
    gather_kernel<<<(unsigned)((m + 1 + 255) / 256), 256, 0, c.stream>>>(src, stride, n, m, dst);
    c.check_launch();
}

void offsets_rebase(Ctx& c, const u64* off, u64 lo, u64 n1, u64* out) {
    if (!n1) return;
    const int grid = (int)std::max<u64>(1, std::min<u64>((n1 + 255) / 256, (u64)c.num_sms * 8));
    rebase_kernel<<<grid, 256, 0, c.stream>>>(off, lo, n1, out);
    c.check_launch();
}

void byte_unit_offsets(Ctx& c, const BytePacked& d, u64 blocks_per_unit, u64 nunits, u64* dev_out) {
    gather_kernel<<<(unsigned)((nunits + 1 + 255) / 256), 256, 0, c.stream>>>(d.offs.p, blocks_per_unit, d.nb,
                                                                             nunits, dev_out);
    c.check_launch();
}

void delta_chunk_offsets(Ctx& c, const DeltaPacked& d, u64 blocks_per_chunk, u64 nchunks, u64* dev_out) {
    gather_kernel<<<(unsigned)((nchunks + 1 + 255) / 256), 256, 0, c.stream>>>(d.offs.p, blocks_per_chunk, d.nb,
                                                                              nchunks, dev_out);
    c.check_launch();
}

}  // namespace gd
