"""report / simulate of one plan sharded by data-parallel column (SURVEY.md
§8(e), BASELINE config C4's "8-rank DP sharding").

Rank r of W owns device columns [r*N/W, (r+1)*N/W) of every iteration (N =
the plan's device_count). Two exchanges, both on per-iteration vectors:

  phase 0 (local columns)  tmax, amax, busy      -> all_reduce MAX
                           tokens, pad_gap, pad_cap -> all_reduce SUM
                           sim_err (first infeasible (i, d) key) -> MIN
  phase 1 (local columns)  tgap = sum(tmax - t), agap = sum(amax - a) -> SUM
  finish (every rank)      DBR_i = tgap_i / (tmax_i * N), ABR_i likewise,
                           run-level means and simulate totals

Gaps are integers, so the all-reduced sums are exact in any order and every
rank's result is bit-identical to the single-GPU report() / simulate() of the
whole plan (hbp_eval_columns*, include/hbp_b200.h). Over NCCL the exchanges
are 6 + 2 vectors of n_iterations words.

On GPUs the whole exchange runs in C++ on the engine's stream
(hbp_eval_sharded over abi.Comm, `evaluate_nccl`). `sharded_evaluate` is the
same protocol with a caller-supplied all_reduce (gloo on CPU hosts,
tests/test_multiproc.py): the engine's kernels run on the context's stream,
torch's fills and collectives on torch's, so it synchronises at each hand-over.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional

from . import abi

MAX, SUM, MIN = "max", "sum", "min"


class EvalColumnsBufs(C.Structure):
    _fields_ = [("tmax", C.c_void_p), ("amax", C.c_void_p), ("tokens", C.c_void_p), ("pad_gap", C.c_void_p),
                ("pad_cap", C.c_void_p), ("busy", C.c_void_p), ("tgap", C.c_void_p), ("agap", C.c_void_p),
                ("sim_err", C.c_void_p)]


def columns_of(rank: int, world: int, n_devices: int):
    return rank * n_devices // world, (rank + 1) * n_devices // world


def torch_all_reduce(dist):
    """all_reduce(tensor, op) over torch.distributed (NCCL on GPUs, gloo on CPU)."""
    ops = {MAX: dist.ReduceOp.MAX, SUM: dist.ReduceOp.SUM, MIN: dist.ReduceOp.MIN}

    def reduce(t, op):
        dist.all_reduce(t, op=ops[op])

    return reduce


class ColumnBuffers:
    """The per-iteration device vectors of one rank (torch tensors)."""

    def __init__(self, n_iterations: int, device):
        import torch
        n = max(n_iterations, 1)
        self.t = {k: torch.zeros(n, dtype=torch.int64, device=device)
                  for k in ("tmax", "amax", "tokens", "pad_gap", "pad_cap", "tgap", "agap")}
        self.busy = torch.zeros(n, dtype=torch.float64, device=device)
        self.sim_err = torch.zeros(1, dtype=torch.int64, device=device)
        t = self.t
        self.c = EvalColumnsBufs(*[t[k].data_ptr() for k in ("tmax", "amax", "tokens", "pad_gap", "pad_cap")],
                                 self.busy.data_ptr(), t["tgap"].data_ptr(), t["agap"].data_ptr(),
                                 self.sim_err.data_ptr())


def _bind(lib):
    lib.hbp_eval_columns.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                     C.POINTER(EvalColumnsBufs)]
    lib.hbp_eval_columns_finish.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(EvalColumnsBufs),
                                            C.POINTER(abi.Metrics), C.POINTER(abi.SimTotals)]


def eval_phase(ctx, plan, phase: int, c0: int, c1: int, bufs: ColumnBuffers, profile=None):
    _bind(ctx.lib)
    prof = C.byref(profile) if profile is not None else None
    ctx.check(ctx.lib.hbp_eval_columns(ctx.h, plan.h, phase, c0, c1, prof, C.byref(bufs.c)))


def eval_finish(ctx, plan, bufs: ColumnBuffers, profile=None):
    _bind(ctx.lib)
    prof = C.byref(profile) if profile is not None else None
    m, st = abi.Metrics(), abi.SimTotals()
    ctx.check(ctx.lib.hbp_eval_columns_finish(ctx.h, plan.h, prof, C.byref(bufs.c), C.byref(m), C.byref(st)))
    return m, (st if profile is not None else None)


def reduce_phase0(bufs: ColumnBuffers, all_reduce):
    for k in ("tmax", "amax"):
        all_reduce(bufs.t[k], MAX)
    all_reduce(bufs.busy, MAX)
    for k in ("tokens", "pad_gap", "pad_cap"):
        all_reduce(bufs.t[k], SUM)
    all_reduce(bufs.sim_err, MIN)


def reduce_phase1(bufs: ColumnBuffers, all_reduce):
    all_reduce(bufs.t["tgap"], SUM)
    all_reduce(bufs.t["agap"], SUM)


def sharded_evaluate(ctx: "abi.Context", plan: "abi.DevicePlanHandle", rank: int, world: int,
                     all_reduce: Optional[Callable] = None, profile: Optional[abi.HardwareProfile] = None):
    """(Metrics, SimTotals or None) of `plan`, this rank evaluating its DP
    columns; `all_reduce(tensor, op)` combines across ranks (None: world 1)."""
    import torch
    v = abi.PlanView()
    ctx.check(ctx.lib.hbp_plan_view_get(ctx.h, plan.h, C.byref(v)))
    c0, c1 = columns_of(rank, world, v.device_count)
    bufs = ColumnBuffers(v.n_iterations, torch.device("cuda", torch.cuda.current_device()))
    # torch zero-filled the buffers on its current stream; the engine's kernels
    # run on the context's (non-blocking) stream
    torch.cuda.current_stream().synchronize()
    eval_phase(ctx, plan, 0, c0, c1, bufs, profile)  # returns with the context stream drained
    if all_reduce is not None and world > 1:
        reduce_phase0(bufs, all_reduce)
        torch.cuda.current_stream().synchronize()  # NCCL's all_reduce returns before it lands
    eval_phase(ctx, plan, 1, c0, c1, bufs, profile)
    if all_reduce is not None and world > 1:
        reduce_phase1(bufs, all_reduce)
        torch.cuda.current_stream().synchronize()
    return eval_finish(ctx, plan, bufs, profile)


def evaluate_nccl(comm: "abi.Comm", plan: "abi.DevicePlanHandle", profile: Optional[abi.HardwareProfile] = None):
    """hbp_eval_sharded: phases and both NCCL exchanges in C++ on the engine's stream."""
    return comm.evaluate(plan, profile)
