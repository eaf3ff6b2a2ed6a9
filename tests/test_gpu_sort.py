"""The LSD radix sort under canonicalize (tuple_array.hpp:73-133) on device
keys (< 2^nbits, the contract of gd_sort_keys_device): the classic onesweep
and the pipelined kernels (bulk-copy prefetch, 8/9/10-bit digits, ballot or
MATCH.ANY ranking, in-place or separate staging) against numpy's sort —
odd tails, single tiles, nbits 1..64, skewed C2-shaped keys."""
import ctypes as C

import numpy as np
import pytest

from paper_2311_02206_b200 import arraylog as al

pytestmark = pytest.mark.gpu

MODES = {
    "classic": {"sort_pipeline": 0},
    "pipe8": {"sort_pipeline": 1, "sort_digit_bits": 8, "sort_pipeline_min_keys": 0},
    "pipe9": {"sort_pipeline": 1, "sort_digit_bits": 9, "sort_pipeline_min_keys": 0},
    "pipe10": {"sort_pipeline": 1, "sort_digit_bits": 10, "sort_pipeline_min_keys": 0},
    "pipe8s": {"sort_pipeline": 2, "sort_digit_bits": 8, "sort_pipeline_min_keys": 0},
    "pipe10s": {"sort_pipeline": 2, "sort_digit_bits": 10, "sort_pipeline_min_keys": 0},
    "pipe10m": {"sort_pipeline": 3, "sort_digit_bits": 10, "sort_pipeline_min_keys": 0},
    "classicb": {"sort_pipeline": 4},
}


def sort_device(ctx, keys: np.ndarray, nbits: int) -> np.ndarray:
    import torch
    a = torch.from_numpy(keys.view(np.int64).copy()).cuda()
    b = torch.empty_like(a)
    it = C.c_int(0)
    ctx.check(ctx.lib.gd_sort_keys_device(ctx.h, a.data_ptr(), b.data_ptr(), len(keys), nbits, C.byref(it)))
    torch.cuda.synchronize()
    return (b if it.value else a).cpu().numpy().view(np.uint64)


def expected(keys: np.ndarray, nbits: int) -> np.ndarray:
    low = keys & np.uint64((1 << nbits) - 1 if nbits < 64 else (1 << 64) - 1)
    return keys[np.argsort(low, kind="stable")]


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("n,nbits", [(1, 8), (2, 1), (3, 46), (4095, 10), (4096, 9), (4097, 23), (12_345, 64),
                                      (100_003, 46), (1_048_579, 47), (3_000_001, 54)])
def test_sort_matches_stable_argsort(mode, n, nbits):
    ctx = al.default_context()
    rng = np.random.default_rng(n * 131 + nbits)
    hi = (1 << nbits) if nbits < 64 else None
    keys = (rng.integers(0, hi, size=n, dtype=np.uint64) if hi else
            rng.integers(0, 1 << 63, size=n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, size=n, dtype=np.uint64))
    with ctx.configured(**MODES[mode]):
        got = sort_device(ctx, keys, nbits)
    assert np.array_equal(got, expected(keys, nbits))


@pytest.mark.parametrize("mode", ["classic", "pipe10"])
def test_sort_skewed_power_law_keys(mode):
    """C2-shaped keys: (src << 23 | dst) with heavy-tailed sources."""
    ctx = al.default_context()
    rng = np.random.default_rng(11)
    n = 2_000_003
    src = np.floor((5_000_000 - 1) * rng.random(n) ** 1.05 * rng.random(n) ** 6).astype(np.uint64)
    dst = rng.integers(0, 5_000_000, size=n, dtype=np.uint64)
    keys = src << np.uint64(23) | dst
    with ctx.configured(**MODES[mode]):
        got = sort_device(ctx, keys, 46)
    assert np.array_equal(got, np.sort(keys))
