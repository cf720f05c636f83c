#!/usr/bin/env python3
"""One C2 step (build_plan + report + simulate, 10M samples) for ncu captures:
    ncu ... python tools/profile_step.py [--n N] [--steps K]
Prints the engine's per-family stage times of the last step."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2503_07680_b200 import abi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--steps", type=int, default=1)
    a = ap.parse_args()
    lib = abi.load_library()
    ctx = abi.Context(0)
    spec = dict(bench.C2, count=a.n)
    L = bench.synth(lib, spec)
    for _ in range(a.steps):
        plan = ctx.build_plan(None, L, bench.C2_GROUPS, 16384, device_count=bench.DEVICES, seed=bench.PLAN_SEED)
        plan.report()
        plan.simulate()
    ctx.synchronize()
    print("ok", ctx.launches)


if __name__ == "__main__":
    main()
