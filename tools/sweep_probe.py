#!/usr/bin/env python3
"""Where a sweep's plan builds spend their time (GPU box):
    python tools/sweep_probe.py [--c5]
C3 shapes: one build_plan of the C1 corpus (100K) per chosen length set,
warm, with wall time, launches, host round trips and the per-family device
time. --c5: the same for the first length sets of C5 over the C4 corpus
(100M, DeepSeek-V2 cost model)."""
import argparse
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2503_07680_b200 import abi  # noqa: E402


def stages(ctx, lib):
    out = {}
    name = C.create_string_buffer(128)
    ms, n, b = C.c_double(), C.c_int64(), C.c_double()
    i = 0
    while lib.hbp_ctx_stage_stats(ctx.h, i, name, 128, C.byref(ms), C.byref(n), C.byref(b)) == 0:
        out[name.value.decode()] = (ms.value, n.value)
        i += 1
    return out


def probe(ctx, lib, s, groups, reps=3):
    for _ in range(2):
        p = ctx.build_plan_samples(s, groups, groups[0][0], device_count=8, seed=7)
        p = None
    ctx.synchronize()
    t = []
    l0 = ctx.launches
    for _ in range(reps):
        t0 = time.perf_counter()
        p = ctx.build_plan_samples(s, groups, groups[0][0], device_count=8, seed=7)
        ctx.synchronize()
        t.append((time.perf_counter() - t0) * 1e3)
        p = None
    launches = (ctx.launches - l0) // reps
    lib.hbp_ctx_set_profiling(ctx.h, 1)
    p = ctx.build_plan_samples(s, groups, groups[0][0], device_count=8, seed=7)
    ctx.synchronize()
    lib.hbp_ctx_set_profiling(ctx.h, 0)
    st = stages(ctx, lib)
    dev = sum(v[0] for v in st.values())
    top = sorted(st.items(), key=lambda kv: -kv[1][0])[:8]
    print(f"groups {[g[0] for g in groups]}: wall {min(t):.2f} ms, device {dev:.2f} ms, {launches} launches, "
          f"{p.n_iterations if hasattr(p, 'n_iterations') else ''}", flush=True)
    print("   " + ", ".join(f"{k} {v[0]:.2f}/{v[1]}" for k, v in top), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c5", action="store_true")
    a = ap.parse_args()
    lib = abi.load_library()
    ctx = abi.Context(0)
    if not a.c5:
        L = np.maximum(bench.synth(lib, bench.C1), 128)
        s, keep = abi.make_samples(None, L, "c1")
        for ls in ([131072], [8192, 131072], [2048, 16384, 131072], [1024, 4096, 16384, 65536, 131072],
                   [512, 1024, 2048, 4096, 8192, 16384, 32768, 65536, 131072]):
            probe(ctx, lib, s, [(l, 1, 0) for l in ls])
    else:
        import torch
        L = bench.synth(lib, bench.C4)
        d = torch.from_numpy(L).cuda()
        s, keep = abi.device_samples(0, d.data_ptr(), len(L), "c5")
        for ls in ([131072], [256, 131072], [16384, 131072], [256, 1024, 4096, 16384, 65536, 131072]):
            probe(ctx, lib, s, [(l, 1, 0) for l in ls], reps=2)


if __name__ == "__main__":
    main()
