"""Stage-level parity of the CUDA primitives against the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m", [1, 2, 3, 10, 257, 4096, 100_003, 2_000_000])
@pytest.mark.parametrize("seed", [0, 7, 0xDEADBEEFCAFEF00D])
def test_shuffle_matches_fisher_yates(ctx, oracle, m, seed):
    got = ctx.shuffle_positions(seed, m)
    want = oracle.shuffle_positions(seed, m)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n", [1, 5, 2047, 2048, 2049, 1_000_000, 10_000_019])
def test_scan_u32(ctx, n):
    rng = np.random.default_rng(n)
    a = rng.integers(0, 1 << 20, size=n, dtype=np.uint32)
    got = ctx.scan_u32(a)
    want = np.concatenate([[0], np.cumsum(a.astype(np.uint64))[:-1]]).astype(np.uint64)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n,bits", [(1, 8), (100, 8), (4097, 17), (1_000_000, 17), (3_000_001, 32)])
@pytest.mark.parametrize("desc", [False, True])
def test_radix_sort_stable(ctx, n, bits, desc):
    rng = np.random.default_rng(n + bits)
    keys = rng.integers(0, 1 << min(bits, 31), size=n, dtype=np.uint32) & np.uint32((1 << bits) - 1 if bits < 32 else 0xFFFFFFFF)
    vals = np.arange(n, dtype=np.uint32)
    k, v = ctx.radix_sort(keys, vals, bits, desc)
    order = np.argsort(-keys.astype(np.int64) if desc else keys, kind="stable")
    assert np.array_equal(v, vals[order])
    assert np.array_equal(k, keys[order])
