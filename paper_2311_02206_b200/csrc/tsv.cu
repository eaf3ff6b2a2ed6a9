// tsv.cu — fact ingestion and canonical TSV output on the device (SURVEY
// §8f rank 3): read_facts for numeric fact files (io.hpp:64-114),
// file_is_all_integers (io.hpp:145-170) and to_tsv / write_relation
// (io.hpp:118-143).  At 10^8 facts the reference's single-threaded getline /
// from_chars parse and ostringstream formatting dominate wall time outside
// the fixpoint; here the text crosses PCIe once and every line (or row) is a
// thread.
//
// Parse: newline positions by order-preserving compaction, then one thread
// per line applies the reference's rules — one trailing '\r' stripped, blank
// and '#' lines skipped, columns split on runs of ' ' / '\t', each token an
// unsigned decimal (digits only, no overflow), UINT64_MAX reserved, exactly
// `arity` columns.  The first offending line (smallest line number, as the
// reference stops there) is reported; the host re-reads that one line to
// build the reference's message.  Surviving rows are compacted in file
// order and canonicalized (sort + unique), like read_facts.
//
// Format: per row its text length (decimal digits + tabs + '\n'), an
// exclusive scan (decoupled look-back), then every row writes its bytes at
// its offset — the bytes of `out << row[c]` joined by '\t', one row per line.
#include <string>

#include "dev_common.cuh"
#include "ops.h"
#include "select.cuh"
#include "tsv.h"

namespace gd {

namespace {

struct NlPred {
    const char* t;
    __device__ bool operator()(u64 i) const { return t[i] == '\n'; }
};
struct NlEmit {
    u64* pos;
    __device__ void operator()(u64 i, u64 p) const { pos[p] = i; }
};

__device__ __forceinline__ bool is_blank(char ch) { return ch == ' ' || ch == '\t'; }

// mode 0: parse into rows[line * arity + c] (keep[line] = 1 for data lines)
// mode 1: file_is_all_integers (any bad token -> first_err)
__global__ void parse_lines_kernel(const char* __restrict__ text, u64 len, const u64* __restrict__ nl, u64 n_nl,
                                   u64 nlines, u32 arity, int mode, u64* __restrict__ rows,
                                   uint8_t* __restrict__ keep, unsigned long long* first_err) {
    for (u64 L = (u64)blockIdx.x * blockDim.x + threadIdx.x; L < nlines; L += (u64)gridDim.x * blockDim.x) {
        const u64 s = L == 0 ? 0 : nl[L - 1] + 1;
        u64 e = L < n_nl ? nl[L] : len;
        if (e > s && text[e - 1] == '\r') --e;
        if (mode == 0) keep[L] = 0;
        u64 i = s;
        while (i < e && is_blank(text[i])) ++i;
        if (i == e || text[i] == '#') continue;
        u32 cols = 0;
        bool bad = false;
        while (i < e) {
            while (i < e && is_blank(text[i])) ++i;
            if (i == e) break;
            u64 v = 0;
            bool ok = true;
            u64 j = i;
            for (; j < e && !is_blank(text[j]); ++j) {
                const char ch = text[j];
                if (ch < '0' || ch > '9') {
                    ok = false;
                    continue;
                }
                const u64 d = (u64)(ch - '0');
                if (v > (~0ull - d) / 10) ok = false;  // from_chars: result_out_of_range
                else v = v * 10 + d;
            }
            if (ok && v == kEmptySlot) ok = false;  // reserved sentinel (types.hpp:16)
            if (mode == 0 && cols < arity) rows[L * arity + cols] = v;
            ++cols;
            bad |= !ok;
            i = j;
        }
        if ((mode == 0 && cols != arity) || bad) {
            atomicMin(first_err, (unsigned long long)L);
            continue;
        }
        if (mode == 0) keep[L] = 1;
    }
}

struct KeepPred {
    const uint8_t* keep;
    __device__ bool operator()(u64 i) const { return keep[i] != 0; }
};
struct RowEmit {
    const u64* in;
    u64* out;
    u32 arity;
    __device__ void operator()(u64 i, u64 p) const {
        for (u32 c = 0; c < arity; ++c) out[p * arity + c] = in[i * arity + c];
    }
};

__device__ __forceinline__ u32 decimal_digits(u64 v) {
    u32 d = 1;
    u64 p = 10;
    while (d < 20 && v >= p) {
        ++d;
        p *= 10;
    }
    return d;
}

__global__ void tsv_lengths_kernel(const u64* __restrict__ rows, u64 n, u32 arity, u64* __restrict__ len) {
    for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (u64)gridDim.x * blockDim.x) {
        u64 l = arity;  // (arity - 1) tabs + '\n'
        for (u32 c = 0; c < arity; ++c) l += decimal_digits(rows[r * arity + c]);
        len[r] = l;
    }
}

// Exclusive scan of u64 values, single pass (decoupled look-back); ws =
// [tile counter, total, statuses...] zeroed.
constexpr int kScanT = 256, kScanI = 8;
constexpr u64 kScanTile = (u64)kScanT * kScanI;
__global__ void __launch_bounds__(kScanT) scan_u64_kernel(const u64* __restrict__ in, u64* __restrict__ out, u64 n,
                                                          u64* ws) {
    __shared__ u64 s_tile, s_base;
    __shared__ u64 s_scan[kScanT / 32 + 1];
    const u64 tile = claim_tile(ws, &s_tile);
    const u64 first = tile * kScanTile + (u64)threadIdx.x * kScanI;
    u64 v[kScanI];
    u64 sum = 0;
#pragma unroll
    for (int j = 0; j < kScanI; ++j) {
        v[j] = first + j < n ? in[first + j] : 0;
        sum += v[j];
    }
    u64 total;
    const u64 ex = block_exclusive_scan<u64, kScanT>(sum, total, s_scan);
    if (threadIdx.x < 32) {
        const u64 b = warp_lookback(ws + 2, tile, total);
        if (threadIdx.x == 0) {
            s_base = b;
            if (tile == gridDim.x - 1) ws[1] = b + total;
        }
    }
    __syncthreads();
    u64 off = s_base + ex;
#pragma unroll
    for (int j = 0; j < kScanI; ++j) {
        if (first + j < n) out[first + j] = off;
        off += v[j];
    }
}

__global__ void tsv_format_kernel(const u64* __restrict__ rows, u64 n, u32 arity, const u64* __restrict__ off,
                                  char* __restrict__ out) {
    for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (u64)gridDim.x * blockDim.x) {
        char* p = out + off[r];
        for (u32 c = 0; c < arity; ++c) {
            if (c) *p++ = '\t';
            u64 v = rows[r * arity + c];
            const u32 d = decimal_digits(v);
            for (u32 k = d; k-- > 0;) {
                p[k] = (char)('0' + v % 10);
                v /= 10;
            }
            p += d;
        }
        *p = '\n';
    }
}

int grid_of(const Ctx& c, u64 n) {
    return (int)std::max<u64>(1, std::min<u64>((n + 255) / 256, (u64)c.num_sms * 16));
}

// Line index: newline positions and the line count (std::getline: a final
// segment without '\n' is a line too).
u64 index_lines(Ctx& c, const char* d_text, u64 len, DevBuf<u64>& nl, u64* n_nl_out) {
    nl.reserve_discard(c, std::max<u64>(len, 1));
    DevBuf<u64> ws;
    u64 n_nl = 0;
    if (len) {
        run_select_async(c, len, NlPred{d_text}, NlEmit{nl.p}, ws);
        unsigned long long t;
        c.read_words(&t, ws.p + 1, 1);
        n_nl = t;
    }
    *n_nl_out = n_nl;
    // the last byte tells whether a final unterminated line exists
    u64 nlines = n_nl;
    if (len) {
        char last = 0;
        c.d2h(&last, d_text + len - 1, 1);
        c.sync();
        if (last != '\n') ++nlines;
    }
    return nlines;
}

}  // namespace

// Host restatement of the reference's per-line checks for the one line the
// device flagged, producing read_facts' exact message (io.hpp:87-108).
std::string tsv_line_error(const char* text, u64 len, u64 line_idx, u32 arity, const std::string& name) {
    u64 s = 0, L = 0;
    while (L < line_idx && s < len) {
        const void* q = memchr(text + s, '\n', len - s);
        if (!q) break;
        s = (u64)(static_cast<const char*>(q) - text) + 1;
        ++L;
    }
    u64 e = s;
    while (e < len && text[e] != '\n') ++e;
    if (e > s && text[e - 1] == '\r') --e;
    std::vector<std::string> cols;
    u64 i = s;
    while (i < e) {
        while (i < e && (text[i] == ' ' || text[i] == '\t')) ++i;
        const u64 st = i;
        while (i < e && text[i] != ' ' && text[i] != '\t') ++i;
        if (i > st) cols.emplace_back(text + st, i - st);
    }
    const std::string where = name + ":" + std::to_string(line_idx + 1) + ": ";
    if (cols.size() != arity)
        return where + "expected " + std::to_string(arity) + " columns, got " + std::to_string(cols.size());
    for (const std::string& tok : cols) {
        bool ok = !tok.empty();
        u64 v = 0;
        for (char ch : tok) {
            if (ch < '0' || ch > '9') {
                ok = false;
                break;
            }
            const u64 d = (u64)(ch - '0');
            if (v > (~0ull - d) / 10) {
                ok = false;
                break;
            }
            v = v * 10 + d;
        }
        if (!ok) return where + "'" + tok + "' is not an unsigned integer";
        if (v == kEmptySlot) return where + "value is reserved";
    }
    return where + "malformed line";
}

u64 parse_facts_device(Ctx& c, const char* h_text, u64 len, u32 arity, const std::string& name, DevBuf<u64>& rows) {
    if (arity == 0) throw_load("read_facts: arity must be positive");
    DevBuf<char> text(c, std::max<u64>(len, 1));
    c.h2d(text.p, h_text, len);
    DevBuf<u64> nl;
    u64 n_nl = 0;
    const u64 nlines = index_lines(c, text.p, len, nl, &n_nl);
    rows.reserve_discard(c, 1);
    if (nlines == 0) return 0;
    DevBuf<u64> raw(c, nlines * arity);
    DevBuf<uint8_t> keep(c, nlines);
    DevBuf<unsigned long long> err(c, 1);
    c.memset(err.p, 0xff, sizeof(unsigned long long));
    parse_lines_kernel<<<grid_of(c, nlines), 256, 0, c.stream>>>(text.p, len, nl.p, n_nl, nlines, arity, 0, raw.p,
                                                                 keep.p, err.p);
    c.check_launch();
    unsigned long long bad;
    c.read_words(&bad, err.p, 1);
    if (bad != ~0ull) throw_load(tsv_line_error(h_text, len, bad, arity, name));
    DevBuf<u64> packed(c, nlines * arity);
    DevBuf<u64> ws;
    run_select_async(c, nlines, KeepPred{keep.p}, RowEmit{raw.p, packed.p, arity}, ws);
    unsigned long long m;
    c.read_words(&m, ws.p + 1, 1);
    return canonicalize_rows(c, packed.p, m, arity, rows);
}

bool facts_all_integers_device(Ctx& c, const char* h_text, u64 len) {
    DevBuf<char> text(c, std::max<u64>(len, 1));
    c.h2d(text.p, h_text, len);
    DevBuf<u64> nl;
    u64 n_nl = 0;
    const u64 nlines = index_lines(c, text.p, len, nl, &n_nl);
    if (nlines == 0) return true;
    DevBuf<unsigned long long> err(c, 1);
    c.memset(err.p, 0xff, sizeof(unsigned long long));
    parse_lines_kernel<<<grid_of(c, nlines), 256, 0, c.stream>>>(text.p, len, nl.p, n_nl, nlines, 1, 1, nullptr,
                                                                 nullptr, err.p);
    c.check_launch();
    unsigned long long bad;
    c.read_words(&bad, err.p, 1);
    return bad == ~0ull;
}

u64 rows_to_tsv_device(Ctx& c, const u64* d_rows, u64 n, u32 arity, char* h_out, u64 capacity) {
    if (n == 0) return 0;
    DevBuf<u64> len(c, n), off(c, n);
    tsv_lengths_kernel<<<grid_of(c, n), 256, 0, c.stream>>>(d_rows, n, arity, len.p);
    c.check_launch();
    const u64 tiles = (n + kScanTile - 1) / kScanTile;
    DevBuf<u64> ws(c, 2 + tiles);
    c.memset(ws.p, 0, (2 + tiles) * sizeof(u64));
    scan_u64_kernel<<<(unsigned)tiles, kScanT, 0, c.stream>>>(len.p, off.p, n, ws.p);
    c.check_launch();
    unsigned long long total;
    c.read_words(&total, ws.p + 1, 1);
    if (!h_out) return total;
    if (capacity < total) throw Error(GD_ERR_INVALID_ARG, "to_tsv: output buffer too small");
    DevBuf<char> text(c, total);
    tsv_format_kernel<<<grid_of(c, n), 256, 0, c.stream>>>(d_rows, n, arity, off.p, text.p);
    c.check_launch();
    c.d2h(h_out, text.p, total);
    c.sync();
    return total;
}

}  // namespace gd
