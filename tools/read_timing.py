"""plan_from_json of a C2 plan manifest (10M samples, ~0.9 GB): GPU reader
(wall clock, host text in -> device plan + host member arrays) with its
per-stage device times, and the reference (oracle/_ref, one core) on the
manifest of a bounded 1M-sample plan; each in the canonical layout
write_plan produces (plan_read.cu) and minified (json.dumps separators
",", ":" -- the general reader, plan_json.cu). python tools/read_timing.py"""
import ctypes as C
import json
import sys
import time
sys.path.insert(0, '.')
sys.path.insert(0, 'oracle')
import bench  # noqa: E402
from paper_2503_07680_b200 import abi  # noqa: E402
import pyoracle  # noqa: E402

lib = abi.load_library()
ctx = abi.Context(0)
ref = pyoracle.Oracle("reference") if pyoracle.available("reference") else None


def run(n, layout, text):
    for _ in range(2):
        p, i, l = ctx.plan_from_json(text)
    p = None
    t0 = time.perf_counter()
    p, i, l = ctx.plan_from_json(text)
    g = time.perf_counter() - t0
    p = None
    lib.hbp_ctx_set_profiling(ctx.h, 1)
    q = ctx.plan_from_json(text)
    ctx.synchronize()
    lib.hbp_ctx_set_profiling(ctx.h, 0)
    q = None
    st = {}
    name = C.create_string_buffer(128)
    ms, k, b = C.c_double(), C.c_int64(), C.c_double()
    j = 0
    while lib.hbp_ctx_stage_stats(ctx.h, j, name, 128, C.byref(ms), C.byref(k), C.byref(b)) == 0:
        st[name.value.decode()] = ms.value
        j += 1
    dev = sum(st.values())
    r = float("nan")
    if ref is not None and n <= 1_000_000:
        t0 = time.perf_counter()
        ref.plan_from_json(text)
        r = time.perf_counter() - t0
    print(f"{n:9d} samples {layout:9s} {len(text)/1e6:8.1f} MB  gpu e2e {g*1e3:8.1f} ms  device {dev:7.2f} ms  "
          f"reference {r*1e3:9.1f} ms | " + " ".join(f"{k} {v:.2f}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:8]),
          flush=True)


for n in (1_000_000, 10_000_000):
    L = bench.synth(lib, dict(bench.C2), n)
    plan = ctx.build_plan(None, L, bench.C2_GROUPS, 16384, device_count=8, seed=1)
    canon = plan.to_json(None, L)
    plan = None
    run(n, "canonical", canon)
    run(n, "minified", json.dumps(json.loads(canon), separators=(",", ":")).encode())
