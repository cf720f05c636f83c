#!/usr/bin/env python3
"""Full C5 on one GPU: 4096 candidates (512 length sets x SP{1,2,4,8} x
GC{on,off}) over the 100M-sample C4 corpus, DeepSeek-V2 cost model:
    python tools/c5_full.py [--sets K]"""
import argparse
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2503_07680_b200 import abi, sweep  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sets", type=int, default=512)
    a = ap.parse_args()
    import torch
    lib = abi.load_library()
    ctx = abi.Context(0)
    L = bench.synth(lib, bench.C4)
    d = torch.from_numpy(L).cuda()
    prof = bench.c4_profile()
    cands = sweep.make_candidates(ctx, 131072, [256, 512, 1024, 2048, 4096, 8192, 16384, 32768, 65536],
                                  bench.SWEEP_SP, prof)[:8 * a.sets]
    s, keep = abi.device_samples(0, d.data_ptr(), len(L), "c5")
    peak = [0]
    stop = threading.Event()

    def mem():
        while not stop.is_set():
            out = subprocess.run(["nvidia-smi", "--query-gpu=memory.used", "--format=csv,noheader,nounits", "-i", "0"],
                                 capture_output=True, text=True).stdout.strip()
            peak[0] = max(peak[0], int(out or 0))
            time.sleep(0.5)
    th = threading.Thread(target=mem, daemon=True)
    th.start()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    secs, best = ctx.sweep_samples(s, cands, prof, device_count=8, seed=1)
    el = time.perf_counter() - t0
    stop.set()
    print(f"W={os.environ.get('HBP_SWEEP_STREAMS', 8)} sets={a.sets}: {len(cands)} candidates in {el:.2f} s = "
          f"{len(cands) / el:.1f} cand/s, feasible {int(np.isfinite(secs).sum())}, best {best} "
          f"({secs[best] if best >= 0 else None}), peak mem {peak[0]} MiB", flush=True)


if __name__ == "__main__":
    main()
