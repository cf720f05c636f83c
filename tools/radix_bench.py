#!/usr/bin/env python3
"""Device time of the engine's radix sort (hbp_test_radix_sort) per kernel
family, CUDA events on the engine's stream (hbp_ctx_set_profiling):
    python tools/radix_bench.py [--n 9800000] [--bits 15] [--desc]"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_07680_b200 import abi  # noqa: E402


def stage_stats(ctx):
    out = {}
    name = C.create_string_buffer(128)
    ms, launches, nbytes = C.c_double(), C.c_int64(), C.c_double()
    i = 0
    while ctx.lib.hbp_ctx_stage_stats(ctx.h, i, name, 128, C.byref(ms), C.byref(launches), C.byref(nbytes)) == 0:
        out[name.value.decode()] = (ms.value, launches.value, nbytes.value)
        i += 1
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=9_800_000)
    ap.add_argument("--bits", type=int, default=15)
    ap.add_argument("--desc", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    ctx = abi.Context(0)
    rng = np.random.default_rng(1)
    keys = np.minimum(np.exp(rng.normal(7.2, 0.7, a.n)), (1 << a.bits) - 1).astype(np.uint32)
    vals = np.arange(a.n, dtype=np.uint32)
    for _ in range(2):
        ctx.radix_sort(keys, vals, a.bits, a.desc)
    peak = 6546.6
    for _ in range(a.reps):
        ctx.lib.hbp_ctx_set_profiling(ctx.h, 1)
        ctx.radix_sort(keys, vals, a.bits, a.desc)
        ctx.synchronize()
        ctx.lib.hbp_ctx_set_profiling(ctx.h, 0)
        st = stage_stats(ctx)
        print({k: f"{v[0] * 1e3 / max(v[1], 1):.1f} us x{v[1]} = {v[2] / (v[0] / 1e3) / 1e9:.0f} GB/s "
                  f"({v[2] / (v[0] / 1e3) / 1e9 / peak:.0%})" for k, v in st.items() if k.startswith("radix")})


if __name__ == "__main__":
    main()
