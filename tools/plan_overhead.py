import sys, time, ctypes as C
sys.path.insert(0, '.')
import numpy as np, bench
from paper_2503_07680_b200 import abi
lib = abi.load_library(); ctx = abi.Context(0)
L = np.maximum(bench.synth(lib, bench.C1), 128)
s, keep = abi.make_samples(None, L, "c1")
for groups in ([(8192,1,0),(32768,4,0),(131072,8,0)], [(512,1,0),(1024,1,0),(2048,1,0),(4096,1,0),(8192,1,0),(16384,1,0),(32768,1,0),(65536,1,0),(131072,8,0)]):
    for _ in range(3): ctx.build_plan_samples(s, groups, groups[0][0], device_count=8, seed=7)
    ctx.synchronize()
    l0 = ctx.launches; t0 = time.perf_counter(); K = 10
    for _ in range(K): ctx.build_plan_samples(s, groups, groups[0][0], device_count=8, seed=7)
    ctx.synchronize(); wall = (time.perf_counter() - t0) / K * 1e3
    lib.hbp_ctx_set_profiling(ctx.h, 1)
    ctx.build_plan_samples(s, groups, groups[0][0], device_count=8, seed=7); ctx.synchronize()
    lib.hbp_ctx_set_profiling(ctx.h, 0)
    name = C.create_string_buffer(128); ms, n, b = C.c_double(), C.c_int64(), C.c_double(); i = 0; tot = 0.0
    while lib.hbp_ctx_stage_stats(ctx.h, i, name, 128, C.byref(ms), C.byref(n), C.byref(b)) == 0:
        tot += ms.value; i += 1
    print(f"{len(groups)} groups: wall {wall:.2f} ms/plan, launches {(ctx.launches - l0)/K:.0f}/plan, kernel time (event-bracketed) {tot:.2f} ms")
