#!/usr/bin/env python3
"""FFD through the chain on a g0-like pool (lognormal lengths, cap 16384):
    HBP_TRACE=1 python tools/chain_micro.py [n] [cap]
Prints the chain trace lines of the second call."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2503_07680_b200 import abi  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
    cap = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
    rng = np.random.default_rng(1)
    L = np.clip(np.rint(rng.lognormal(7.2, 0.7, size=n)), 1, cap).astype(np.int64)
    ctx = abi.Context(0)
    for _ in range(2):
        p = ctx.pack(None, L, cap, "ffd")
    ctx.synchronize()
    print("packs", p.flat().pack_capacity.shape[0])


if __name__ == "__main__":
    main()
