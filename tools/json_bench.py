"""Plan manifest throughput at C2 (10M samples): hbp_plan_to_json into a
pre-touched host buffer (GPU text build + pinned download + copy-out)."""
import ctypes as C
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2503_07680_b200 import abi  # noqa: E402

lib = abi.load_library()
ctx = abi.Context(0)
L = bench.synth(lib, dict(bench.C2))
plan = ctx.build_plan(None, L, bench.C2_GROUPS, 16384, device_count=8, seed=1)
s, keep = abi.make_samples(None, L, "json")
lib.hbp_plan_to_json.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(abi.Samples), C.c_char_p, C.c_int64,
                                 C.POINTER(C.c_int64)]
n = C.c_int64()
ctx.check(lib.hbp_plan_to_json(ctx.h, plan.h, C.byref(s), None, 0, C.byref(n)))
buf = np.ones(n.value, dtype=np.uint8)  # touched
for _ in range(3):
    t = time.perf_counter()
    ctx.check(lib.hbp_plan_to_json(ctx.h, plan.h, C.byref(s), buf.ctypes.data_as(C.c_char_p), n.value, C.byref(n)))
    el = time.perf_counter() - t
print(f"hbp_plan_to_json C2: {n.value / 1e6:.1f} MB in {el * 1e3:.1f} ms ({n.value / el / 1e9:.2f} GB/s into host memory)")
lib.hbp_ctx_set_profiling(ctx.h, 1)
ctx.check(lib.hbp_plan_to_json(ctx.h, plan.h, C.byref(s), buf.ctypes.data_as(C.c_char_p), n.value, C.byref(n)))
lib.hbp_ctx_set_profiling(ctx.h, 0)
name = C.create_string_buffer(128)
ms, cnt, b = C.c_double(), C.c_int64(), C.c_double()
i = 0
while lib.hbp_ctx_stage_stats(ctx.h, i, name, 128, C.byref(ms), C.byref(cnt), C.byref(b)) == 0:
    print(f"  {name.value.decode()}: {ms.value:.2f} ms")
    i += 1
