#!/usr/bin/env python3
"""Per-launch device time of the first-fit chain on one C2 step under
different chain settings (env HBP_CHAIN_M / HBP_CHAIN_NOFENCE), one process
per setting: python tools/chain_sweep.py [m ...]"""
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one():
    sys.path.insert(0, ROOT)
    import bench
    from paper_2503_07680_b200 import abi
    lib = abi.load_library()
    ctx = abi.Context(0)
    L = bench.synth(lib, dict(bench.C2))
    for _ in range(2):
        ctx.build_plan(None, L, bench.C2_GROUPS, 16384, device_count=bench.DEVICES, seed=bench.PLAN_SEED)
    lib.hbp_ctx_set_profiling(ctx.h, 1)
    ctx.build_plan(None, L, bench.C2_GROUPS, 16384, device_count=bench.DEVICES, seed=bench.PLAN_SEED)
    ctx.synchronize()
    lib.hbp_ctx_set_profiling(ctx.h, 0)
    name = C.create_string_buffer(128)
    ms, n, b = C.c_double(), C.c_int64(), C.c_double()
    i, tot = 0, 0.0
    out = {}
    while lib.hbp_ctx_stage_stats(ctx.h, i, name, 128, C.byref(ms), C.byref(n), C.byref(b)) == 0:
        out[name.value.decode()] = (round(ms.value, 3), n.value)
        tot += ms.value
        i += 1
    print(f"  fit.chain {out.get('fit.chain')}  all kernels {tot:.2f} ms", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        one()
        sys.exit(0)
    ms = [int(x) for x in sys.argv[1:]] or [4, 8, 16, 32]
    for m in ms:
        for fence in (1, 0):
            env = dict(os.environ, HBP_CHAIN_M=str(m))
            if not fence:
                env["HBP_CHAIN_NOFENCE"] = "1"
            print(f"m={m} fence={fence}", flush=True)
            subprocess.run([sys.executable, __file__, "one"], env=env, timeout=300)
