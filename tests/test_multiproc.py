"""World-size-2 CPU tests (gloo) of the sharded auto-selection sweep's host
logic: length-set sharding covers every candidate exactly once, keeps each
length set on one rank, and the all_gather argmin equals the single-process
argmin (lowest index on ties, infeasible candidates never win)."""
import math
import os
import socket

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
