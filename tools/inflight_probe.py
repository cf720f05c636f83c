#!/usr/bin/env python3
"""C2 step throughput with 1 to 4 plans in flight (one context and host
thread each; ctypes releases the GIL inside the C-ABI calls), inputs on the
device or in pinned host memory (e2e: copies in, plan view out).
    python tools/inflight_probe.py [--steps 8]"""
import argparse
import ctypes as C
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2503_07680_b200 import abi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--only", default="", help="e.g. device3: only that mode, --reps times")
    a = ap.parse_args()
    lib = abi.load_library()
    ctxs = [abi.Context(0) for _ in range(4)]
    L = bench.synth(lib, dict(bench.C2))
    n = len(L)
    d_len = torch.from_numpy(L).cuda()
    h_len = torch.from_numpy(L).pin_memory()
    prof = abi.default_profile()

    def step(ctx, e2e):
        if e2e:
            s, keep = abi.make_samples(None, h_len.numpy(), "bench")
        else:
            s, keep = abi.device_samples(0, d_len.data_ptr(), n, "bench")
        plan = ctx.build_plan_samples(s, bench.C2_GROUPS, 16384, device_count=bench.DEVICES, seed=bench.PLAN_SEED)
        plan.report()
        plan.simulate(prof)
        if e2e:
            v = abi.PlanView()
            ctx.check(lib.hbp_plan_view_get(ctx.h, plan.h, C.byref(v)))
        return plan

    modes = [(e2e, k) for e2e in (False, True) for k in (1, 2, 3, 4)]
    if a.only:
        modes = [(a.only.startswith("e2e"), int(a.only[-1]))] * a.reps
    for e2e, inflight in modes:
        if True:
            for c in ctxs[:inflight]:
                step(c, e2e)
            torch.cuda.synchronize()
            warm = [threading.Thread(target=lambda c=c: (step(c, e2e), c.synchronize())) for c in ctxs[:inflight]]
            for t in warm:
                t.start()
            for t in warm:
                t.join()  # the pool grows to hold the in-flight working sets before the timed steps
            per = [a.steps // inflight + (1 if i < a.steps % inflight else 0) for i in range(inflight)]

            def work(i):
                for _ in range(per[i]):
                    step(ctxs[i], e2e)
                ctxs[i].synchronize()

            t0 = time.perf_counter()
            th = [threading.Thread(target=work, args=(i,)) for i in range(inflight)]
            for t in th:
                t.start()
            for t in th:
                t.join()
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
            print(f"{'e2e' if e2e else 'device'} in flight {inflight}: {el / a.steps * 1e3:.2f} ms/step "
                  f"= {a.steps * n / el / 1e6:.0f}M samples/s", flush=True)


if __name__ == "__main__":
    main()
