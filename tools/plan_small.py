"""One 100K-sample (C1) build_plan for launch-list captures: python tools/plan_small.py [groups]"""
import sys
sys.path.insert(0, '.')
import numpy as np, bench
from paper_2503_07680_b200 import abi
lib = abi.load_library(); ctx = abi.Context(0)
L = np.maximum(bench.synth(lib, bench.C1), 128)
s, keep = abi.make_samples(None, L, "c1")
groups = [(8192, 1, 0), (32768, 4, 0), (131072, 8, 0)]
ctx.build_plan_samples(s, groups, groups[0][0], device_count=8, seed=7)
ctx.synchronize()
