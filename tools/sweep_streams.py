#!/usr/bin/env python3
"""C3 sweep throughput against the number of worker streams (HBP_SWEEP_STREAMS):
    python tools/sweep_streams.py [W ...]"""
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, ROOT)
    import numpy as np
    import bench
    from paper_2503_07680_b200 import abi, sweep
    lib = abi.load_library()
    ctx = abi.Context(0)
    L = np.maximum(bench.synth(lib, bench.C1), 128)
    cands = sweep.make_candidates(ctx, 131072, bench.SWEEP_SMALLER, bench.SWEEP_SP)
    s, keep = abi.make_samples(None, L, "c1")
    ctx.sweep_samples(s, cands, None, device_count=8, seed=7)  # warm-up: every worker, pools grown
    ctx.synchronize()
    t0 = time.perf_counter()
    secs, best = ctx.sweep_samples(s, cands, None, device_count=8, seed=7)
    el = time.perf_counter() - t0
    print(f"W={os.environ.get('HBP_SWEEP_STREAMS')}: {len(cands) / el:.0f} candidates/s ({el:.3f} s), best {best}, "
          f"cores {os.cpu_count()}", flush=True)
else:
    for w in sys.argv[1:] or ["4", "8", "16", "32"]:
        subprocess.run([sys.executable, __file__, "--one"], env=dict(os.environ, HBP_SWEEP_STREAMS=w))
