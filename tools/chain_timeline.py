#!/usr/bin/env python3
"""Reads the first-fit chain timeline (HBP_TRACE=1 HBP_CHAIN_TL=file) and
prints, per chain launch, where the time goes: arrival of every block at
every warp, the per-step increments T(b,j) - max(T(b-1,j), T(b,j-1)), and
which steps the critical path crosses.
    python tools/chain_timeline.py file"""
import sys

import numpy as np


def launches(path):
    raw = open(path, "rb").read()
    off = 0
    while off < len(raw):
        J, nb, ffd, M = np.frombuffer(raw, np.uint32, 4, off)
        off += 16
        w = np.frombuffer(raw, np.uint64, int(J) * int(nb), off).reshape(int(J), int(nb))
        off += 8 * int(J) * int(nb)
        t = (w & np.uint64((1 << 40) - 1)).astype(np.int64)
        d = ((w >> np.uint64(40)) & np.uint64(0xffff)).astype(np.int64)
        act = (w >> np.uint64(56)).astype(np.int64)
        yield int(J), int(nb), int(ffd), int(M), t, d, act


def analyse(J, nb, ffd, M, t, d, act):
    t = t - t.min()
    print(f"== {'ffd' if ffd else 'fill'} J={J} blocks={nb} M={M}: span {t.max() / 1e3:.1f} us")
    # increments over the recurrence
    prev_b = np.full_like(t, -1)
    prev_b[:, 1:] = t[:, :-1]
    prev_j = np.full_like(t, -1)
    prev_j[1:, :] = t[:-1, :]
    ready = np.maximum(prev_b, prev_j)
    inc = np.where(ready >= 0, t - ready, 0)
    # critical path: walk back from the last cell choosing the later predecessor
    j, b = J - 1, nb - 1
    path_inc_j = 0.0
    path_inc_b = 0.0
    steps_j = steps_b = 0
    heavy = []
    while j > 0 or b > 0:
        pj = t[j - 1, b] if j > 0 else -1
        pb = t[j, b - 1] if b > 0 else -1
        if pj >= pb:
            path_inc_j += t[j, b] - pj
            steps_j += 1
            heavy.append((t[j, b] - pj, j, b, "j", int(d[j - 1, b]), int(act[j - 1, b])))
            j -= 1
        else:
            path_inc_b += t[j, b] - pb
            steps_b += 1
            heavy.append((t[j, b] - pb, j, b, "b", int(d[j, b - 1]), int(act[j, b - 1])))
            b -= 1
    print(f"  critical path: {steps_j} warp hops ({path_inc_j / 1e3:.1f} us, {path_inc_j / max(steps_j, 1):.0f} ns avg), "
          f"{steps_b} block steps ({path_inc_b / 1e3:.1f} us, {path_inc_b / max(steps_b, 1):.0f} ns avg)")
    heavy.sort(reverse=True)
    print("  heaviest path steps (ns, warp, block, kind, predecessor's serve ns, its active runs):",
          [(int(x[0]),) + x[1:] for x in heavy[:12]])
    on = act > 0
    print(f"  serve ns per (warp, block) with active runs: median {np.median(d[on]):.0f}, p99 {np.percentile(d[on], 99):.0f}, "
          f"max {d.max()}; per active run: median {np.median(d[on] / act[on]):.0f} ns; cells active {on.mean():.3f}; "
          f"sum of serve {d.sum() / 1e3:.0f} us")
    big = np.argwhere(d >= np.percentile(d[on], 99.5))
    print("  slowest cells (warp, block, serve ns, active):", [(int(a), int(b), int(d[a, b]), int(act[a, b])) for a, b in big[:10]])
    # hop latency inside vs between CTAs
    w = 16 if M > 4 else 32
    hop = t[1:, :] - t[:-1, :]
    intra = np.array([(j % w) != 0 for j in range(1, J)])
    print(f"  median hop (arrival j -> j+1): intra-CTA {np.median(hop[intra]):.0f} ns, inter-CTA {np.median(hop[~intra]):.0f} ns")
    # first warp each block reaches late: block arrival at warp 0 and at the last warp
    q = [0, nb // 4, nb // 2, 3 * nb // 4, nb - 1]
    print("  block b reaches warp 0 / J/2 / last at (us):",
          {b: (round(t[0, b] / 1e3, 1), round(t[J // 2, b] / 1e3, 1), round(t[J - 1, b] / 1e3, 1)) for b in q})


def main():
    for rec in launches(sys.argv[1]):
        analyse(*rec)


if __name__ == "__main__":
    main()
