"""All per-family stage times of one C2 step (event-bracketed launches)."""
import ctypes as C
import sys
sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_2503_07680_b200 import abi  # noqa: E402
lib = abi.load_library(); ctx = abi.Context(0)
L = bench.synth(lib, dict(bench.C2))
for _ in range(3):
    p = ctx.build_plan(None, L, bench.C2_GROUPS, 16384, device_count=8, seed=1); p.report(); p.simulate(); p = None
ctx.synchronize()
lib.hbp_ctx_set_profiling(ctx.h, 1)
p = ctx.build_plan(None, L, bench.C2_GROUPS, 16384, device_count=8, seed=1); p.report(); p.simulate()
ctx.synchronize()
lib.hbp_ctx_set_profiling(ctx.h, 0)
name = C.create_string_buffer(128); ms, n, b = C.c_double(), C.c_int64(), C.c_double(); i = 0; rows = []
while lib.hbp_ctx_stage_stats(ctx.h, i, name, 128, C.byref(ms), C.byref(n), C.byref(b)) == 0:
    rows.append((ms.value, n.value, name.value.decode())); i += 1
tot = sum(r[0] for r in rows)
print(f"total {tot:.2f} ms over {sum(r[1] for r in rows)} launches")
for r in sorted(rows, reverse=True):
    print(f"{r[2]:28s} {r[0]:7.3f} ms {r[1]:4d} launches {r[0] / max(r[1], 1) * 1e3:7.1f} us/launch")
