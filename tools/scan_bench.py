#!/usr/bin/env python3
"""Device time of the engine's look-back scan (hbp_test_scan_u32: u32 in,
u64 exclusive prefix out, 12 B per element) with CUDA events on the
engine's stream:  python tools/scan_bench.py [--n 9700000]"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_07680_b200 import abi  # noqa: E402
from radix_bench import stage_stats  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=9_700_000)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    ctx = abi.Context(0)
    x = np.random.default_rng(1).integers(0, 1 << 20, a.n, dtype=np.uint32)
    want = np.concatenate([[0], np.cumsum(x.astype(np.uint64))[:-1]])
    assert np.array_equal(ctx.scan_u32(x), want)
    peak = 6546.6
    for _ in range(a.reps):
        ctx.lib.hbp_ctx_set_profiling(ctx.h, 1)
        ctx.scan_u32(x)
        ctx.synchronize()
        ctx.lib.hbp_ctx_set_profiling(ctx.h, 0)
        st = stage_stats(ctx)
        print({k: f"{v[0] * 1e3 / max(v[1], 1):.1f} us x{v[1]} = {v[2] / (v[0] / 1e3) / 1e9:.0f} GB/s "
                  f"({v[2] / (v[0] / 1e3) / 1e9 / peak:.0%})" for k, v in st.items()})


if __name__ == "__main__":
    main()
