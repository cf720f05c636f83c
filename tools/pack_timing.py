"""pack() per strategy on C1's corpus at each C1 capacity: GPU (CUDA events
around the C-ABI call, device-resident plan) vs the reference compiled in
place (oracle/_ref, one core). python tools/pack_timing.py [strategies]"""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch, bench
from paper_2503_07680_b200 import abi
sys.path.insert(0, 'oracle')
import pyoracle

lib = abi.load_library(); ctx = abi.Context(0)
L = np.maximum(bench.synth(lib, bench.C1), 128)
ref = pyoracle.Oracle("reference") if pyoracle.available("reference") else None
kinds = sys.argv[1].split(",") if len(sys.argv) > 1 else ["isf", "ffd", "ffs", "bfs", "spfhp", "random"]
for cap in (8192, 32768, 131072):
    Lc = L[L <= cap]
    for k in kinds:
        for _ in range(2):
            ctx.pack(None, Lc, cap, k, seed=7)
        ctx.synchronize()
        t0 = time.perf_counter()
        got = ctx.pack(None, Lc, cap, k, seed=7)
        ctx.synchronize()
        g = time.perf_counter() - t0
        r = None
        if ref is not None:
            t0 = time.perf_counter()
            want = ref.pack(None, Lc, cap, k, seed=7)
            r = time.perf_counter() - t0
            f = got.flat()
            assert np.array_equal(f.pack_member_offsets, want.pack_member_offsets), (cap, k)
        print(f"cap {cap:6d} n {len(Lc):6d} {k:6s} gpu {g*1e3:8.2f} ms  reference {r*1e3 if r else float('nan'):9.1f} ms")
