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


def _fy_model(seed, m, forced):
    # Rng::shuffle (rng.hpp:61-68) over the counter-based draws, with the
    # first draw of step `forced` rejected: that step and every later one
    # (smaller i) use one more draw (rng.hpp:32-41)
    M64 = (1 << 64) - 1

    def draw(k):
        z = (seed + k * 0x9E3779B97F4A7C15) & M64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    v = list(range(m))
    for i in range(m, 1, -1):
        k = m - i + 1 + (1 if forced and i <= forced else 0)
        j = draw(k) % i
        v[i - 1], v[j] = v[j], v[i - 1]
    return np.array(v, dtype=np.uint32)


@pytest.mark.parametrize("forced", [0, 2, 1234, 5000])
def test_shuffle_rejection_repair(ctx, monkeypatch, forced):
    # the repair path of a rejected draw (probability < m / 2^64 in real
    # runs), forced through hbp_test_set_force_reject and checked against the model
    import ctypes as C
    ctx.lib.hbp_test_set_force_reject.argtypes = [C.c_void_p, C.c_uint64]
    ctx.check(ctx.lib.hbp_test_set_force_reject(ctx.h, forced))
    try:
        got = ctx.shuffle_positions(77, 5000)
    finally:
        ctx.check(ctx.lib.hbp_test_set_force_reject(ctx.h, 0))
    assert np.array_equal(got, _fy_model(77, 5000, forced))


@pytest.mark.parametrize("n", [8191, 8192, 8193])
@pytest.mark.parametrize("bits", [1, 15, 28, 32])
@pytest.mark.parametrize("desc", [False, True])
def test_radix_sort_small_and_onesweep_boundary(ctx, n, bits, desc):
    # n <= 8192 takes the one-CTA sort (every digit pass in one launch), above
    # it the onesweep passes; both stable and equal to a stable argsort
    rng = np.random.default_rng(n * 64 + bits)
    hi = (1 << bits) if bits < 32 else (1 << 32)
    keys = rng.integers(0, hi, size=n, dtype=np.uint64).astype(np.uint32)
    keys[: n // 8] = keys[0]  # ties: stability matters
    vals = np.arange(n, dtype=np.uint32)
    k, v = ctx.radix_sort(keys, vals, bits, desc)
    order = np.argsort(-keys.astype(np.int64) if desc else keys, kind="stable")
    assert np.array_equal(v, vals[order])
    assert np.array_equal(k, keys[order])


@pytest.mark.parametrize("m", [8191, 8192, 8193])
def test_shuffle_around_the_in_kernel_scan(ctx, oracle, m):
    # up to 8192 elements the target counts are scanned by the targets
    # kernel's last block, above by the look-back scan
    got = ctx.shuffle_positions(99, m)
    assert np.array_equal(got, oracle.shuffle_positions(99, m))
