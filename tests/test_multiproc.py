"""World-size-2 CPU tests (gloo) of the sharded auto-selection sweep's host
logic: length-set sharding covers every candidate exactly once, keeps each
length set on one rank, and the all_gather argmin equals the single-process
argmin (lowest index on ties, infeasible candidates never win)."""
import math
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_07680_b200 import sweep


def fake_candidates():
    out = []
    for mask in range(16):
        lengths = [l for b, l in enumerate([2048, 4096, 8192, 16384]) if mask >> b & 1] + [131072]
        for sp in (1, 2, 4, 8):
            for gc in (True, False):
                out.append(([(l, 1 if i == 0 else sp, 7 if gc else 0) for i, l in enumerate(lengths)], lengths[0]))
    return out


def fake_time(i, c):
    # ties on purpose (i // 3), some infeasible
    if c[0][-1][1] == 1 and c[0][-1][2] == 0:
        return math.inf
    return 100.0 + ((i // 3) * 7919) % 97


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cands = fake_candidates()
    mine = sweep.shard(cands, rank, world)
    local = (math.inf, -1)
    for i in mine:
        t = fake_time(i, cands[i])
        if math.isfinite(t) and (t < local[0] or (t == local[0] and i < local[1])):
            local = (t, i)
    best = sweep.reduce_argmin(local, sweep.torch_all_gather(dist, "cpu"))
    q.put((rank, mine, best))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(120)
def test_sharded_sweep_argmin_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=100) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cands = fake_candidates()
    shards = {r: set(m) for r, m, _ in res}
    assert shards[0].isdisjoint(shards[1])
    assert shards[0] | shards[1] == set(range(len(cands)))
    for r in (0, 1):  # whole length sets per rank
        sets = {sweep.length_set(cands[i]) for i in shards[r]}
        other = {sweep.length_set(cands[i]) for i in shards[1 - r]}
        assert sets.isdisjoint(other)
    want = (math.inf, -1)
    for i, c in enumerate(cands):
        t = fake_time(i, c)
        if math.isfinite(t) and t < want[0]:
            want = (t, i)
    assert all(best == want for _, _, best in res)


def test_reduce_argmin_rules():
    g = lambda pairs: (lambda _x: pairs)  # noqa: E731
    assert sweep.reduce_argmin(None, g([(5.0, 7), (5.0, 3)])) == (5.0, 3)
    assert sweep.reduce_argmin(None, g([(math.inf, -1), (9.0, 4)])) == (9.0, 4)
    assert sweep.reduce_argmin(None, g([(math.inf, -1), (math.inf, -1)])) == (math.inf, -1)



# -- report / simulate sharded by DP column: the exchanges over gloo ---------

# ---------------------------------------------------------------------------
# Host restatement of the sharded evaluation's two phases over a flat plan
# (test infrastructure: checks the exchange logic over gloo on CPU).
# ---------------------------------------------------------------------------

def phase0_host(fp: object, c0: int, c1: int):
    I = len(fp.iter_group)
    out = {k: np.zeros(I, dtype=np.int64) for k in ("tmax", "amax", "tokens", "pad_gap", "pad_cap")}
    for i in range(I):
        d0, d1 = fp.iter_dev_offsets[i], fp.iter_dev_offsets[i + 1]
        for d in range(min(d0 + c0, d1), min(d0 + c1, d1)):
            q0, q1 = fp.dev_pack_offsets[d], fp.dev_pack_offsets[d + 1]
            tt = int(fp.pack_total[q0:q1].sum())
            aa = int(fp.pack_attention[q0:q1].sum())
            out["tmax"][i] = max(out["tmax"][i], tt)
            out["amax"][i] = max(out["amax"][i], aa)
            out["tokens"][i] += tt
            out["pad_gap"][i] += int((fp.pack_capacity[q0:q1] - fp.pack_total[q0:q1]).sum())
            out["pad_cap"][i] += int(fp.pack_capacity[q0:q1].sum())
    return out


def phase1_host(fp: object, c0: int, c1: int, tmax: np.ndarray, amax: np.ndarray):
    I = len(fp.iter_group)
    tg, ag = np.zeros(I, dtype=np.int64), np.zeros(I, dtype=np.int64)
    for i in range(I):
        d0, d1 = fp.iter_dev_offsets[i], fp.iter_dev_offsets[i + 1]
        for d in range(min(d0 + c0, d1), min(d0 + c1, d1)):
            q0, q1 = fp.dev_pack_offsets[d], fp.dev_pack_offsets[d + 1]
            tg[i] += tmax[i] - int(fp.pack_total[q0:q1].sum())
            ag[i] += amax[i] - int(fp.pack_attention[q0:q1].sum())
    return tg, ag


def finish_host(fp: object, red: dict, tg: np.ndarray, ag: np.ndarray):
    """Per-iteration DBR / ABR (reference operation: gap sum / (max * N))."""
    nd = np.diff(fp.iter_dev_offsets).astype(np.float64)
    dbr = tg.astype(np.float64) / (red["tmax"].astype(np.float64) * nd)
    abr = ag.astype(np.float64) / (red["amax"].astype(np.float64) * nd)
    return dbr, abr


def _eval_worker(rank, world, port, q, fp_arrays):
    import numpy as np
    import torch
    from paper_2503_07680_b200 import abi, sharded_eval as se
    from test_multiproc import phase0_host, phase1_host, finish_host
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fp = abi.FlatPlan(**fp_arrays)
    c0, c1 = se.columns_of(rank, world, fp.device_count)
    loc = phase0_host(fp, c0, c1)
    red = {}
    for k, op in (("tmax", dist.ReduceOp.MAX), ("amax", dist.ReduceOp.MAX), ("tokens", dist.ReduceOp.SUM),
                  ("pad_gap", dist.ReduceOp.SUM), ("pad_cap", dist.ReduceOp.SUM)):
        t = torch.from_numpy(loc[k].copy())
        dist.all_reduce(t, op=op)
        red[k] = t.numpy()
    tg, ag = phase1_host(fp, c0, c1, red["tmax"], red["amax"])
    tg_t, ag_t = torch.from_numpy(tg), torch.from_numpy(ag)
    dist.all_reduce(tg_t, op=dist.ReduceOp.SUM)
    dist.all_reduce(ag_t, op=dist.ReduceOp.SUM)
    dbr, abr = finish_host(fp, red, tg_t.numpy(), ag_t.numpy())
    q.put((rank, dbr, abr, int(red["tokens"].sum())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_sharded_eval_exchange_gloo():
    import sys
    import numpy as np
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    from pyoracle import Oracle
    o = Oracle("restatement")
    L = o.synth(20_000, "lognormal:7.2:0.7", 0.03, "uniform:16385:131072", 131072, 5)
    fp = o.build_plan(None, L, [(16384, 1, 28), (131072, 8, 29)], l_best=16384, device_count=8, seed=4)
    m_ref, dbr_ref, abr_ref = o.report(fp)
    arrays = {k: getattr(fp, k) for k in ("device_count", "seed", "groups", "l_best", "iter_group", "iter_dev_offsets",
                                          "dev_index", "dev_pack_offsets", "pack_capacity", "pack_total",
                                          "pack_attention", "pack_member_offsets", "member_id", "member_length")}
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_eval_worker, args=(r, world, port, q, arrays)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=150) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, dbr, abr, tokens in res:  # every rank: the reference's per-iteration values, bit for bit
        assert np.array_equal(dbr, dbr_ref) and np.array_equal(abr, abr_ref)
        assert tokens == int(np.asarray(fp.member_length).sum())
