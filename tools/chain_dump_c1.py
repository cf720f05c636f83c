"""Chain inputs of one C1 plan (100K, given groups) for offline analysis:
HBP_TRACE=1 HBP_CHAIN_RUNS=out python tools/chain_dump_c1.py 131072 [8192 ...]"""
import sys
sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import bench  # noqa: E402
from paper_2503_07680_b200 import abi  # noqa: E402
lib = abi.load_library()
ctx = abi.Context(0)
L = np.maximum(bench.synth(lib, bench.C1), 128)
ls = sorted(int(x) for x in sys.argv[1:]) or [131072]
p = ctx.build_plan(None, L, [(l, 1, 0) for l in ls], ls[0], device_count=8, seed=7)
print("ok", p.n_iterations)
