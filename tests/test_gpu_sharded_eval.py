"""report / simulate sharded by DP column (paper_2503_07680_b200.sharded_eval,
hbp_eval_columns*): W ranks emulated on one GPU -- each rank's phase-0 and
phase-1 vectors combined with the all-reduce ops NCCL would apply -- must give
every metric and simulate total bit-identical to the single-GPU
report() / simulate() of the whole plan."""
import numpy as np
import pytest

from paper_2503_07680_b200 import abi, sharded_eval as se

pytestmark = pytest.mark.gpu

GROUPS = [(16384, 1, 28), (131072, 8, 29)]


def emulate(ctx, plan, world, profile):
    import torch
    v = plan.flat()
    n_it, N = len(v.iter_group), v.device_count
    dev = torch.device("cuda", 0)
    ranks = [se.ColumnBuffers(n_it, dev) for _ in range(world)]
    torch.cuda.synchronize()  # torch's zero fills before the engine's stream writes
    for r, b in enumerate(ranks):
        se.eval_phase(ctx, plan, 0, *se.columns_of(r, world, N), b, profile)
    ops = {se.MAX: torch.maximum, se.SUM: torch.add, se.MIN: torch.minimum}

    def all_reduce_over(get, op):  # what NCCL computes, written back to every rank
        acc = get(ranks[0]).clone()
        for b in ranks[1:]:
            acc = ops[op](acc, get(b))
        for b in ranks:
            get(b).copy_(acc)
        torch.cuda.synchronize()  # torch's stream before the engine's next phase

    for k, op in (("tmax", se.MAX), ("amax", se.MAX), ("tokens", se.SUM), ("pad_gap", se.SUM), ("pad_cap", se.SUM)):
        all_reduce_over(lambda b, k=k: b.t[k], op)
    all_reduce_over(lambda b: b.busy, se.MAX)
    all_reduce_over(lambda b: b.sim_err, se.MIN)
    for r, b in enumerate(ranks):
        se.eval_phase(ctx, plan, 1, *se.columns_of(r, world, N), b, profile)
    for k in ("tgap", "agap"):
        all_reduce_over(lambda b, k=k: b.t[k], se.SUM)
    return [se.eval_finish(ctx, plan, b, profile) for b in ranks]


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_eval_bit_identical(ctx, oracle, world):
    L = oracle.synth(200_000, "lognormal:7.2:0.7", 0.02, "uniform:16385:131072", 131072, 17)
    plan = ctx.build_plan(None, L, GROUPS, l_best=16384, device_count=8, seed=1)
    prof = abi.default_profile()
    m_ref, st_ref = plan.report(), plan.simulate(prof)
    for m, st in emulate(ctx, plan, world, prof):
        for k in ("dbr", "pr", "abr", "cr", "ave_t"):
            assert getattr(m, k) == getattr(m_ref, k), k
        assert st.total_seconds == st_ref.total_seconds
        assert st.switch_count == st_ref.switch_count
        assert st.gpu_days == st_ref.gpu_days


def test_sharded_eval_single_rank_and_infeasible(ctx, oracle):
    L = oracle.synth(50_000, "lognormal:7.2:0.7", 0.02, "uniform:16385:131072", 131072, 3)
    plan = ctx.build_plan(None, L, GROUPS, l_best=16384, device_count=8, seed=2)
    m, st = se.sharded_evaluate(ctx, plan, 0, 1, None, abi.default_profile())
    assert m.abr == plan.report().abr and st.total_seconds == plan.simulate().total_seconds
    tiny = abi.default_profile()
    tiny.device_memory = 25 << 30
    with pytest.raises(abi.InfeasibleError) as e1:
        plan.simulate(tiny)
    with pytest.raises(abi.InfeasibleError) as e2:
        emulate(ctx, plan, 4, tiny)
    assert str(e1.value) == str(e2.value)
