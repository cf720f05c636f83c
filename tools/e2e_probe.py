#!/usr/bin/env python3
"""Host-side phase timing of the bench's e2e step (diagnostics):
    python tools/e2e_probe.py"""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_07680_b200 import abi  # noqa: E402


def main():
    lib = abi.load_library()
    ctx = abi.Context(0)
    L = bench.synth(lib, dict(bench.C2))
    n = len(L)
    d_len = torch.from_numpy(L).cuda()
    h_len = torch.from_numpy(L).pin_memory()
    prof = abi.default_profile()

    def step_device():
        s, keep = abi.device_samples(0, d_len.data_ptr(), n, "bench")
        plan = ctx.build_plan_samples(s, bench.C2_GROUPS, 16384, device_count=8, seed=1)
        plan.report()
        plan.simulate(prof)
        return plan

    def step_e2e():
        t = [time.perf_counter()]
        s, keep = abi.make_samples(None, h_len.numpy(), "bench")
        t.append(time.perf_counter())
        plan = ctx.build_plan_samples(s, bench.C2_GROUPS, 16384, device_count=8, seed=1)
        ctx.synchronize()
        t.append(time.perf_counter())
        plan.report()
        plan.simulate(prof)
        ctx.synchronize()
        t.append(time.perf_counter())
        v = abi.PlanView()
        ctx.check(lib.hbp_plan_view_get(ctx.h, plan.h, C.byref(v)))
        t.append(time.perf_counter())
        del plan
        t.append(time.perf_counter())
        return [round(1000 * (b - a), 2) for a, b in zip(t[:-1], t[1:])]

    for i in range(3):
        step_device()
        print("warm e2e", step_e2e(), flush=True)
    keep = None
    for i in range(4):
        keep = step_device()
    for i in range(6):
        print("e2e [samples, build, report+sim, view, free]", step_e2e(), flush=True)


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def bench_like():
    """The bench's exact sequence (warm-up, device loop, e2e loop with L2
    flush and events), printing host phase times of every e2e step."""
    lib = abi.load_library()
    ctx = abi.Context(0)
    stream = torch.cuda.ExternalStream(lib.hbp_ctx_stream(ctx.h))
    L = bench.synth(lib, dict(bench.C2))
    n = len(L)
    d_len = torch.from_numpy(L).cuda()
    h_len = torch.from_numpy(L).pin_memory()
    prof = abi.default_profile()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step_device():
        s, keep = abi.device_samples(0, d_len.data_ptr(), n, "bench")
        plan = ctx.build_plan_samples(s, bench.C2_GROUPS, 16384, device_count=8, seed=1)
        plan.report()
        plan.simulate(prof)
        return plan

    def step_e2e():
        t = [time.perf_counter()]
        s, keep = abi.make_samples(None, h_len.numpy(), "bench")
        plan = ctx.build_plan_samples(s, bench.C2_GROUPS, 16384, device_count=8, seed=1)
        t.append(time.perf_counter())
        plan.report()
        plan.simulate(prof)
        t.append(time.perf_counter())
        v = abi.PlanView()
        ctx.check(lib.hbp_plan_view_get(ctx.h, plan.h, C.byref(v)))
        t.append(time.perf_counter())
        return plan, [round(1000 * (b - a), 2) for a, b in zip(t[:-1], t[1:])]

    def timed(fn, k, show):
        out = None
        for _ in range(k):
            out = None
            t0 = time.perf_counter()
            flush.zero_()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            out = fn()
            b.record(stream)
            torch.cuda.synchronize()
            if show:
                print(f"pre {1e3 * (t1 - t0):.1f} ms, event {a.elapsed_time(b):.1f} ms, phases {out[1]}", flush=True)
        return out

    for _ in range(3):
        step_device()
        step_e2e()
    plan = timed(step_device, 10, False)
    timed(step_e2e, 10, True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "bench":
    bench_like()
