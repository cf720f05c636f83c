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


if __name__ == "__main__":
    main()
