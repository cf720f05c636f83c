import sys, time; sys.path.insert(0, '.')
import torch, bench
from paper_2503_07680_b200 import abi
lib = abi.load_library(); ctx = abi.Context(0)
L = bench.synth(lib, bench.C4); n = len(L)
d = torch.from_numpy(L).cuda(); del L
prof = bench.c4_profile()
for k in range(6):
    torch.cuda.synchronize(); t = time.perf_counter()
    s, keep = abi.device_samples(0, d.data_ptr(), n, "c4")
    p = ctx.build_plan_samples(s, [(16384,1,53),(131072,8,53)], 16384, device_count=8, seed=1); p.report(); p.simulate(prof)
    ctx.synchronize(); print(k, round((time.perf_counter()-t)*1e3,1), "ms", torch.cuda.mem_get_info()[0]>>30, "GB free"); p = None
