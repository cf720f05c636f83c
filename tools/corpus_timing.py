"""load_lengths of a C2-sized raw-lengths / CSV corpus (10M samples):
GPU (text H2D + parse + lengths D2H, wall clock; device-only per-stage
times from the context profiler) vs the reference's istream parser
(oracle/_ref, one core). python tools/corpus_timing.py [count]"""
import ctypes as C
import sys, time
sys.path.insert(0, '.')
sys.path.insert(0, 'oracle')
import numpy as np, bench
from paper_2503_07680_b200 import abi
import pyoracle

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
lib = abi.load_library(); ctx = abi.Context(0)
L = bench.synth(lib, dict(bench.C2, count=n))
raw = ("\n".join(map(str, L.tolist())) + "\n").encode()
csv = ("id,length\n" + "".join(f"{i},{v}\n" for i, v in enumerate(L.tolist()))).encode()
ref = pyoracle.Oracle("reference") if pyoracle.available("reference") else None
jsonl = "".join(f'{{"id":{i},"length":{v}}}\n' for i, v in enumerate(L.tolist())).encode()
for fmt, text in (("raw-lengths", raw), ("csv", csv), ("jsonl", jsonl)):
    for _ in range(2):
        got = ctx.load_lengths(text, fmt)
    t0 = time.perf_counter()
    got = ctx.load_lengths(text, fmt)
    g = time.perf_counter() - t0
    lib.hbp_ctx_set_profiling(ctx.h, 1)
    ctx.load_lengths(text, fmt)
    lib.hbp_ctx_set_profiling(ctx.h, 0)
    st = {}
    name = C.create_string_buffer(128); ms, k, b = C.c_double(), C.c_int64(), C.c_double(); i = 0
    while lib.hbp_ctx_stage_stats(ctx.h, i, name, 128, C.byref(ms), C.byref(k), C.byref(b)) == 0:
        st[name.value.decode()] = (ms.value, k.value); i += 1
    assert np.array_equal(got, L)
    r = float("nan")
    if ref is not None:
        t0 = time.perf_counter()
        _, want = ref.load_lengths(text, fmt, "corpus")
        r = time.perf_counter() - t0
        assert np.array_equal(want, L)
    dev = sum(v[0] for v in st.values())  # ms
    print(f"{fmt:12s} {len(text)/1e6:8.1f} MB  gpu e2e {g*1e3:8.2f} ms  device {dev:6.3f} ms "
          f"({len(text)/dev/1e6:7.1f} GB/s of text)  reference {r*1e3:9.1f} ms  | " +
          " ".join(f"{k} {v[0]:.3f}" for k, v in st.items()))
