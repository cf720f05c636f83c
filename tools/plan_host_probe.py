#!/usr/bin/env python3
"""Host vs device time of one small plan (C1 corpus, one C3 length set) on
one stream: wall time per build_plan, CPU time of the calling thread, device
kernel time (event-bracketed stages), launches and host round trips.
    python tools/plan_host_probe.py"""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import bench  # noqa: E402
from paper_2503_07680_b200 import abi  # noqa: E402

lib = abi.load_library()
ctx = abi.Context(0)
L = np.maximum(bench.synth(lib, bench.C1), 128)
for gl in ([131072], [8192, 32768, 131072], [512, 2048, 8192, 32768, 131072], [512, 1024, 2048, 4096, 8192, 16384, 32768, 65536, 131072]):
    groups = [(g, 1, 0) for g in gl]
    for _ in range(3):
        ctx.build_plan(None, L, groups, gl[0], device_count=8, seed=7)
    ctx.synchronize()
    n0, l0 = ctx.syncs if hasattr(ctx, "syncs") else 0, ctx.launches
    K = 20
    c0 = time.thread_time()
    t0 = time.perf_counter()
    for _ in range(K):
        ctx.build_plan(None, L, groups, gl[0], device_count=8, seed=7)
    ctx.synchronize()
    wall = (time.perf_counter() - t0) / K * 1e3
    cpu = (time.thread_time() - c0) / K * 1e3
    lib.hbp_ctx_set_profiling(ctx.h, 1)
    ctx.build_plan(None, L, groups, gl[0], device_count=8, seed=7)
    ctx.synchronize()
    lib.hbp_ctx_set_profiling(ctx.h, 0)
    name = C.create_string_buffer(128)
    ms, n, b = C.c_double(), C.c_int64(), C.c_double()
    i = 0
    dev = 0.0
    rows = []
    while lib.hbp_ctx_stage_stats(ctx.h, i, name, 128, C.byref(ms), C.byref(n), C.byref(b)) == 0:
        dev += ms.value
        rows.append((ms.value, n.value, name.value.decode()))
        i += 1
    print(f"groups {len(gl)}: wall {wall:.2f} ms/plan, host cpu {cpu:.2f} ms/plan, device kernels {dev:.2f} ms, "
          f"launches/plan {(ctx.launches - l0) / (K + 1):.0f}")
    if "-v" in sys.argv:
        for r in sorted(rows, reverse=True)[:8]:
            print(f"    {r[2]:24s} {r[0]:.3f} ms {r[1]} launches")
    if "-n" in sys.argv:
        for r in sorted(rows, key=lambda r: -r[1])[:14]:
            print(f"    {r[2]:24s} {r[1]} launches {r[0]:.3f} ms")
