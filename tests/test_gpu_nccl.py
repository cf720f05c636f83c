"""The engine's NCCL entry points (hbp_comm_*, hbp_sweep_sharded,
hbp_eval_sharded). One GPU runs a world-1 communicator --
the collectives, the dealing and the argmin exchange execute for real -- and
must give exactly the single-GPU answers. With two or more GPUs visible, two
ranks run over NCCL and must agree with each other and with one GPU."""
import math
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2503_07680_b200 import abi, sweep

pytestmark = pytest.mark.gpu

GROUPS = [(16384, 1, 28), (131072, 8, 29)]


@pytest.fixture(scope="module")
def comm(ctx):
    c = abi.Comm(ctx, abi.Comm.unique_id(ctx), 0, 1)
    yield c
    c.close()


def test_sweep_sharded_world1_equals_sweep(ctx, comm, oracle):
    L = oracle.synth(20_000, "lognormal:8.5:1.4", 0.0, "", 131072, 42)
    L = np.maximum(L, 128)
    cands = sweep.make_candidates(ctx, 131072, [2048, 8192, 32768], [1, 4, 8])
    s, keep = abi.make_samples(None, L, "nccl")
    want, wbest = ctx.sweep_samples(s, cands, None, device_count=8, seed=7)
    got, gbest, local = sweep.run_sweep_nccl(comm, s, cands, None, device_count=8, seed=7)
    assert local == len(cands)
    assert gbest[1] == wbest
    assert np.array_equal(np.isinf(got), np.isinf(want))
    assert np.array_equal(got[np.isfinite(got)], want[np.isfinite(want)])


def test_sweep_sharded_error_is_first_in_index_order(ctx, comm, oracle):
    L = oracle.synth(5_000, "lognormal:7.2:0.7", 0.0, "", 131072, 3)
    cands = [([(8192, 1, 0), (131072, 8, 27)], 8192), ([(1024, 1, 0), (4096, 8, 0)], 1024)]  # 2nd: l_max short
    s, keep = abi.make_samples(None, L, "nccl")
    with pytest.raises(abi.ValidationError) as a:
        ctx.sweep_samples(s, cands, None, device_count=8, seed=1)
    with pytest.raises(abi.ValidationError) as b:
        comm.sweep(s, cands, None, device_count=8, seed=1)
    assert str(a.value) == str(b.value)


def test_eval_sharded_world1_bit_identical(ctx, comm, oracle):
    L = oracle.synth(200_000, "lognormal:7.2:0.7", 0.02, "uniform:16385:131072", 131072, 17)
    plan = ctx.build_plan(None, L, GROUPS, l_best=16384, device_count=8, seed=1)
    prof = abi.default_profile()
    m_ref, st_ref = plan.report(), plan.simulate(prof)
    m, st = comm.evaluate(plan, prof)
    for k in ("dbr", "pr", "abr", "cr", "ave_t"):
        assert getattr(m, k) == getattr(m_ref, k), k
    assert st.total_seconds == st_ref.total_seconds
    assert st.switch_count == st_ref.switch_count
    m2, st2 = comm.evaluate(plan, None)
    assert st2 is None and m2.abr == m_ref.abr
    tiny = abi.default_profile()
    tiny.device_memory = 25 << 30
    with pytest.raises(abi.InfeasibleError) as e1:
        plan.simulate(tiny)
    with pytest.raises(abi.InfeasibleError) as e2:
        comm.evaluate(plan, tiny)
    assert str(e1.value) == str(e2.value)


TWO_RANKS = r'''
import os, sys, json
import numpy as np
import torch, torch.distributed as dist
sys.path.insert(0, os.environ["HBP_ROOT"]); sys.path.insert(0, os.path.join(os.environ["HBP_ROOT"], "oracle"))
from paper_2503_07680_b200 import abi, sweep
from pyoracle import Oracle
rank = int(os.environ["RANK"]); torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
ctx = abi.Context(rank)
comm = sweep.engine_comm(ctx, dist)
L = np.maximum(Oracle("restatement").synth(20_000, "lognormal:8.5:1.4", 0.0, "", 131072, 42), 128)
cands = sweep.make_candidates(ctx, 131072, [2048, 8192, 32768], [1, 4, 8])
s, keep = abi.make_samples(None, L, "nccl")
secs, best, local = sweep.run_sweep_nccl(comm, s, cands, None, device_count=8, seed=7)
plan = ctx.build_plan(None, L, [(8192, 1, 11), (131072, 8, 27)], l_best=8192, device_count=8, seed=7)
m, st = comm.evaluate(plan, abi.default_profile())
print(json.dumps({"rank": rank, "best": best[1], "secs": [x if np.isfinite(x) else None for x in secs.tolist()],
                  "local": local, "abr": m.abr, "total": st.total_seconds}), flush=True)
comm.close(); ctx.close(); dist.destroy_process_group()
'''


def test_two_ranks_over_nccl(ctx, tmp_path, oracle):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (NCCL refuses two ranks on one device)")
    script = tmp_path / "two.py"
    script.write_text(TWO_RANKS)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, HBP_ROOT=root)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                          "--master-addr=127.0.0.1", "--master-port=29533", str(script)],
                         capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    import json
    rows = sorted((json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")), key=lambda r: r["rank"])
    assert len(rows) == 2
    assert rows[0]["secs"] == rows[1]["secs"] and rows[0]["best"] == rows[1]["best"]
    assert rows[0]["local"] + rows[1]["local"] == len(rows[0]["secs"])
    L = np.maximum(oracle.synth(20_000, "lognormal:8.5:1.4", 0.0, "", 131072, 42), 128)
    cands = sweep.make_candidates(ctx, 131072, [2048, 8192, 32768], [1, 4, 8])
    want, wbest = ctx.sweep(None, L, cands, device_count=8, seed=7)
    assert rows[0]["best"] == wbest
    assert [x if np.isfinite(x) else None for x in want.tolist()] == rows[0]["secs"]
    plan = ctx.build_plan(None, L, [(8192, 1, 11), (131072, 8, 27)], l_best=8192, device_count=8, seed=7)
    assert rows[0]["abr"] == rows[1]["abr"] == plan.report().abr
    assert rows[0]["total"] == rows[1]["total"] == plan.simulate().total_seconds
