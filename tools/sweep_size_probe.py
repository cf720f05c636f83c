import os, sys, time
sys.path.insert(0, '.')
import numpy as np
import bench
from paper_2503_07680_b200 import abi, sweep
lib = abi.load_library(); ctx = abi.Context(0)
for cnt in (100_000, 50_000, 25_000):
    L = np.maximum(bench.synth(lib, dict(bench.C1, count=cnt)), 128)
    cands = sweep.make_candidates(ctx, 131072, bench.SWEEP_SMALLER, bench.SWEEP_SP)
    s, keep = abi.make_samples(None, L, "c1")
    ctx.sweep_samples(s, cands, None, device_count=8, seed=7); ctx.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); ctx.sweep_samples(s, cands, None, device_count=8, seed=7); ctx.synchronize(); ts.append(time.perf_counter() - t0)
    print(cnt, [round(len(cands)/t) for t in ts], "launches", ctx.launches, flush=True)
