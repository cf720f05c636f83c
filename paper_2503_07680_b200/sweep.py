"""Group auto-selection sweep.

Candidates (BASELINE.json configs 3 and 5): length set = {l_max} ∪ a subset of
the smaller candidate lengths, times an SP degree for the non-smallest groups,
times GC on/off (ckpt = AnalyticProfiler(profile).derive_ckpt(l, sp) or 0).
Each candidate's time is simulate(build_plan(corpus, groups_c)).total_seconds
(+inf when infeasible); the answer is the argmin, lowest index on ties.

Multi-GPU: candidates that share a length set share one plan, so whole length
sets are dealt to ranks (round-robin in decreasing estimated cost); every rank
evaluates its share on its own GPU, then one ncclAllGather of
(best_seconds, best_index) -- 16 bytes per rank over NVLink -- yields the
global argmin (plus an all-reduce MIN of the per-candidate seconds so every
rank holds them all). No data-path collective. On GPUs this runs in C++
(hbp_sweep_sharded over the engine's NCCL communicator, `run_sweep_nccl`);
`run_sweep` is the same dealing with a caller-supplied all_gather (gloo on
CPU hosts, tests/test_multiproc.py).
"""
from __future__ import annotations

import itertools
import math
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import abi

Candidate = Tuple[list, int]  # ([(length, sp, ckpt), ...], l_best)


def make_candidates(ctx: "abi.Context", l_max: int, smaller: Sequence[int], sps: Sequence[int],
                    profile: Optional[abi.HardwareProfile] = None) -> List[Candidate]:
    """C3/C5 candidate list: 2^len(smaller) length sets x SP x GC{on,off}, in
    (length set, sp, gc) order so candidates of one set are contiguous."""
    prof = abi.analytic_profiler(profile)
    cache = {}

    def ckpt(l, sp):
        if (l, sp) not in cache:
            try:
                cache[(l, sp)] = ctx.derive_ckpt(prof, l, sp)
            except abi.InfeasibleError:
                cache[(l, sp)] = None
        return cache[(l, sp)]

    out = []
    smaller = sorted(smaller)
    for r in range(len(smaller) + 1):
        for subset in itertools.combinations(smaller, r):
            lengths = list(subset) + [l_max]
            for sp in sps:
                for gc in (True, False):
                    groups = []
                    for i, l in enumerate(lengths):
                        s = 1 if i == 0 else sp
                        ck = ckpt(l, s) if gc else 0
                        groups.append((l, s, 0 if ck is None else ck))
                    out.append((groups, lengths[0]))
    return out


def length_set(c: Candidate) -> tuple:
    return tuple(g[0] for g in c[0])


def shard(candidates: Sequence[Candidate], rank: int, world: int) -> List[int]:
    """Indices of the candidates rank `rank` evaluates: whole length sets, dealt
    round-robin in decreasing cost (more groups and smaller groups pack more
    packs), so every plan is built exactly once across ranks."""
    sets = {}
    for i, c in enumerate(candidates):
        sets.setdefault(length_set(c), []).append(i)
    order = sorted(sets.items(), key=lambda kv: (-len(kv[0]), kv[0][0], kv[0]))
    mine = []
    for k, (_, idx) in enumerate(order):
        if k % world == rank:
            mine.extend(idx)
    return sorted(mine)


def reduce_argmin(local_best: Tuple[float, int], all_gather) -> Tuple[float, int]:
    """Combine per-rank (seconds, global index) pairs: min seconds, lowest
    index on ties, infeasible (inf) loses. `all_gather(t)` returns a list of
    per-rank (seconds, index)."""
    pairs = all_gather(local_best)
    best = (math.inf, -1)
    for sec, idx in pairs:
        if idx < 0 or not math.isfinite(sec):
            continue
        if sec < best[0] or (sec == best[0] and (best[1] < 0 or idx < best[1])):
            best = (sec, idx)
    return best


def torch_all_gather(dist, device):
    """all_gather of (float64 seconds, int64 index) over torch.distributed."""
    import torch

    def gather(pair):
        t = torch.tensor([pair[0], float(pair[1])], dtype=torch.float64, device=device)
        out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
        dist.all_gather(out, t)
        return [(float(o[0]), int(o[1])) for o in out]

    return gather


def run_sweep(ctx: "abi.Context", samples_struct, candidates: Sequence[Candidate], rank: int = 0, world: int = 1,
              all_gather=None, profile: Optional[abi.HardwareProfile] = None, **opts):
    """Evaluates this rank's share; returns (local seconds dict, global best)."""
    mine = shard(candidates, rank, world)
    secs = {}
    local = (math.inf, -1)
    if mine:
        times, best = ctx.sweep_samples(samples_struct, [candidates[i] for i in mine], profile, **opts)
        for i, t in zip(mine, times):
            secs[i] = float(t)
            if math.isfinite(t) and (t < local[0] or (t == local[0] and i < local[1])):
                local = (float(t), i)
    if world > 1 and all_gather is not None:
        return secs, reduce_argmin(local, all_gather)
    return secs, local


def engine_comm(ctx: "abi.Context", dist) -> "abi.Comm":
    """The engine's NCCL communicator for the ranks of `dist` (torch.distributed
    carries the 128-byte NCCL id from rank 0; every collective after that is
    the engine's own, on its stream)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    box = [abi.Comm.unique_id(ctx) if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    return abi.Comm(ctx, box[0], rank, world)


def run_sweep_nccl(comm: "abi.Comm", samples_struct, candidates: Sequence[Candidate],
                   profile: Optional[abi.HardwareProfile] = None, **opts):
    """hbp_sweep_sharded: (seconds of every candidate, (best seconds, best
    index), candidates this rank evaluated) -- identical on every rank."""
    secs, best, local = comm.sweep(samples_struct, candidates, profile, **opts)
    return secs, ((float(secs[best]) if best >= 0 else math.inf), best), local
