// Host rebuild of byte-offset download blocks (csrc/host_decode.cpp) on the
// CPU: every offset width, partial last blocks, arities 1-3, destinations at
// every 16-byte shift of a 64-byte line, blocks split across two calls (unit
// boundaries) — rows must equal the keys' columns.  Exits non-zero on the
// first mismatch.  Built and run by tests/test_host_decode.py.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "host_decode.h"

int main() {
    std::mt19937_64 rng(7);
    int failures = 0, cases = 0;
    for (int trial = 0; trial < 12; ++trial) {
        const int ar = 1 + trial % 3;
        const unsigned bits = ar == 1 ? 40 : ar == 2 ? 20 + trial : 18;
        const uint64_t kmask = bits * ar >= 64 ? ~0ull : (1ull << (bits * ar)) - 1;
        // sorted distinct keys with gaps of every width class
        std::vector<unsigned long long> keys;
        uint64_t k = rng() % 1000;
        const uint64_t n0 = 5000 + 37 * trial;
        for (uint64_t i = 0; i < n0; ++i) {
            const int r = (int)(rng() % 10);
            const uint64_t g = r < 5 ? 1 + rng() % 3 : r < 8 ? 1 + rng() % 3000 : r < 9 ? 1 + rng() % (1u << 20)
                                                                                        : 1 + rng() % (1ull << 33);
            k += g;
            keys.push_back(k & kmask);
        }
        std::sort(keys.begin(), keys.end());
        keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
        const uint64_t n = keys.size(), nb = (n + 31) / 32;
        std::vector<unsigned long long> heads(nb);
        std::vector<uint8_t> cls(nb), pay;
        std::vector<uint64_t> boff(nb + 1, 0);
        for (uint64_t b = 0; b < nb; ++b) {
            const uint64_t c = std::min<uint64_t>(32, n - b * 32), h = keys[b * 32], r = keys[b * 32 + c - 1] - h;
            const int code = r < 256 ? 0 : r < 65536 ? 1 : r < (1ull << 32) ? 2 : 3;
            heads[b] = h;
            cls[b] = (uint8_t)code;
            boff[b] = pay.size();
            for (uint64_t i = 0; i < c; ++i) {
                const uint64_t o = keys[b * 32 + i] - h;
                for (int q = 0; q < (1 << code); ++q) pay.push_back((uint8_t)(o >> (8 * q)));
            }
        }
        boff[nb] = pay.size();
        pay.resize(pay.size() + 64);
        for (int shift = 0; shift < 4; ++shift) {
            std::vector<unsigned long long> back(n * ar + 64, 0xABABABABABABABABull);
            const uintptr_t a = reinterpret_cast<uintptr_t>(back.data());
            const size_t base = ((64 - a % 64) % 64) / 8;  // first 64-byte aligned word
            unsigned long long* out = back.data() + base + 2 * shift;
            const uint64_t split = nb / 3;  // two units
            gd::byte_decode_rows(heads.data(), cls.data(), pay.data(), 0, split, n, ar, bits, out);
            gd::byte_decode_rows(heads.data() + split, cls.data() + split, pay.data() + boff[split], split * 32,
                                 nb - split, n, ar, bits, out);
            const uint64_t cm = bits >= 64 ? ~0ull : (1ull << bits) - 1;
            uint64_t bad = 0;
            for (uint64_t i = 0; i < n; ++i)
                for (int col = 0; col < ar; ++col)
                    bad += out[i * ar + col] != ((keys[i] >> ((ar - 1 - col) * bits)) & cm);
            for (uint64_t i = n * ar; i < n * ar + 8; ++i) bad += out[i] != 0xABABABABABABABABull;  // nothing past
            ++cases;
            if (bad) {
                ++failures;
                fprintf(stderr, "trial %d arity %d shift %d: %llu bad words\n", trial, ar, shift,
                        (unsigned long long)bad);
            }
        }
    }
    printf("host_decode: %d cases, %d failed, vectorized %d\n", cases, failures, (int)gd::byte_decode_vectorized());
    return failures ? 1 : 0;
}
