"""GPU parity of the profilers, Algorithms 1/3/4 and the candidate sweep
against the oracle restatement and the reference-generated golden answers."""
import json
import os

import numpy as np
import pytest

from paper_2503_07680_b200 import abi

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))
CANDS = [8192, 16384, 32768, 65536, 131072]
SPS = [1, 2, 4, 8, 16]


def table(name):
    return abi.table_profiler([tuple(r) for r in GOLD["profiles"][name]])


def outcome(fn):
    try:
        return ("ok", fn())
    except (abi.ValidationError, abi.InfeasibleError) as e:
        return (type(e).__name__, str(e))


def test_select_groups_golden(ctx):
    g, lb, lm = ctx.select_groups(CANDS, table("group_candidates_8b"), SPS)
    assert [list(x) for x in g] == GOLD["autoselect"]["select_groups_candidates_8b"][0]
    assert (lb, lm) == (16384, 131072)
    g, lb, lm = ctx.select_groups(CANDS, abi.analytic_profiler(), SPS)
    assert [list(x) for x in g] == GOLD["autoselect"]["select_groups_analytic_default"][0]


def test_find_best_golden(ctx):
    st = table("gc_sweep_8b")
    assert ctx.find_best_sp_ckpt(st, 32768, [2, 4, 8, 16]) == ((8, 8), 4.12)
    assert ctx.find_best_sp_ckpt(st, 131072, [2, 4, 8, 16])[0][0] == 8


def test_derive_and_memory_golden(ctx):
    an = abi.analytic_profiler()
    for key, want in GOLD["autoselect"]["analytic_derive_ckpt"].items():
        l, sp = map(int, key.split("/"))
        assert ctx.derive_ckpt(an, l, sp) == want
    for key, want in GOLD["autoselect"]["memory_used"].items():
        l, sp, ck = map(int, key.split("/"))
        assert ctx.memory_used(l, sp, ck) == want


def test_profiler_queries_match_oracle(ctx, oracle):
    rng = np.random.default_rng(1)
    for _ in range(60):
        p = abi.default_profile()
        p.per_token_activation_memory = float(rng.integers(100000, 500000))
        p.gc_memory_saving_per_layer = p.per_token_activation_memory * float(rng.uniform(0.0, 0.95)) * 4096
        p.base_memory = int((30 << 30) + rng.integers(0, 40 << 30))
        an = abi.analytic_profiler(p)
        l = int(rng.choice([1024, 4096, 16384, 65536, 131072]))
        sp = int(rng.choice([1, 2, 4, 8]))
        ck = int(rng.integers(0, 33))
        for f in ("profile_time", "profile_memory"):
            assert outcome(lambda: getattr(ctx, f)(an, l, sp, ck)) == outcome(lambda: getattr(oracle, f)(an, l, sp, ck))
        assert outcome(lambda: ctx.derive_ckpt(an, l, sp)) == outcome(lambda: oracle.derive_ckpt(an, l, sp))
        assert outcome(lambda: ctx.find_best_sp_ckpt(an, l, [1, 2, 4, 8])) == \
            outcome(lambda: oracle.find_best_sp_ckpt(an, l, [1, 2, 4, 8]))


def test_select_groups_matches_oracle_random(ctx, oracle):
    rng = np.random.default_rng(3)
    for _ in range(60):
        p = abi.default_profile()
        p.per_token_activation_memory = float(rng.integers(100000, 500000))
        p.gc_memory_saving_per_layer = p.per_token_activation_memory * float(rng.uniform(0.5, 0.95)) * 4096
        p.base_memory = int((40 << 30) + rng.integers(0, 20 << 30))
        an = abi.analytic_profiler(p)
        lens = sorted(set(int(x) for x in rng.choice([2048, 4096, 8192, 16384, 32768, 65536, 131072],
                                                     size=int(rng.integers(1, 6)))))
        sps = sorted(set(int(x) for x in rng.choice([1, 2, 4, 8, 16], size=int(rng.integers(1, 5)))))
        assert outcome(lambda: ctx.select_groups(lens, an, sps)) == \
            outcome(lambda: oracle.select_groups(lens, an, sps))


@pytest.mark.parametrize("rows,lens,sps", [
    ([(16384, 1, 28, 81604378624, 9.0), (32768, 2, 28, 82678120448, 3.0)], [16384, 32768], SPS),
    ([(8192, 1, 8, 81604378624, 2.0)], [8192], [1]),
    ([(4096, 1, 8, 81604378624, 1.5), (8192, 2, 8, 81604378624, 2.0), (16384, 4, 8, 81604378624, 9.0),
      (131072, 8, 29, 84825604096, 30.0)], [8192, 131072], SPS),
    ([(8192, 1, 8, 81604378624, 2.0), (131072, 8, 32, None, 0)], [8192, 131072], SPS),
    ([(65536, 2, 32, None, 0), (65536, 4, 32, None, 0)], [65536], [2, 4]),
])
def test_select_groups_tables(ctx, oracle, rows, lens, sps):
    t = abi.table_profiler(rows)
    assert outcome(lambda: ctx.select_groups(lens, t, sps)) == outcome(lambda: oracle.select_groups(lens, t, sps))


def test_argument_errors(ctx, oracle):
    an = abi.analytic_profiler()
    for args in [([16384, 8192], an, SPS), (CANDS, an, [1, 3]), ([], an, SPS)]:
        assert outcome(lambda: ctx.select_groups(*args)) == outcome(lambda: oracle.select_groups(*args))
    bad = abi.analytic_profiler(ckpt_min=5, ckpt_max=4)
    with pytest.raises(abi.ValidationError, match="ckpt probe bounds"):
        ctx.derive_ckpt(bad, 4096, 1)


def test_sweep_matches_oracle(ctx, oracle):
    L = oracle.synth(30_000, "lognormal:7.2:0.7", 0.03, "uniform:16385:131072", 131072, 5)
    an = abi.analytic_profiler()
    cands = []
    for ls in ([4096, 131072], [16384, 131072], [8192, 32768, 131072]):
        for sp in (4, 8):
            for gc in (True, False):
                groups = []
                for i, l in enumerate(ls):
                    s = 1 if i == 0 else sp
                    try:
                        ck = oracle.derive_ckpt(an, l, s) if gc else 0
                    except abi.InfeasibleError:
                        ck = 0
                    groups.append((l, s, ck))
                cands.append((groups, ls[0]))
    got = ctx.sweep(None, L, cands, device_count=8, seed=1)
    want = oracle.sweep(None, L, cands, device_count=8, seed=1)
    assert got[1] == want[1]
    assert np.array_equal(np.isinf(got[0]), np.isinf(want[0]))
    fin = np.isfinite(want[0])
    assert np.allclose(got[0][fin], want[0][fin], rtol=1e-12, atol=0)


def test_c3_candidates_and_sharded_sweep(ctx, oracle):
    from paper_2503_07680_b200 import sweep
    L = np.maximum(oracle.synth(20_000, "lognormal:8.5:1.4", 0.0, "", 131072, 42), 128)
    cands = sweep.make_candidates(ctx, 131072, [2048, 8192, 32768], [1, 2, 4, 8])
    assert len(cands) == 8 * 4 * 2
    an = abi.analytic_profiler()
    for groups, _ in cands:  # GC-on ckpt values are the reference profiler's
        for (l, sp, ck) in groups:
            assert ck == 0 or ck == oracle.derive_ckpt(an, l, sp)
    s, keep = abi.make_samples(None, L)
    want, wbest = oracle.sweep(None, L, cands, device_count=8, seed=7)
    merged = {}
    for rank in range(3):  # three "ranks" on one GPU: shards cover everything once
        secs, _ = sweep.run_sweep(ctx, s, cands, rank, 3, None, device_count=8, seed=7)
        assert not (set(secs) & set(merged))
        merged.update(secs)
    got = np.array([merged[i] for i in range(len(cands))])
    assert np.array_equal(np.isinf(got), np.isinf(want))
    fin = np.isfinite(want)
    assert np.allclose(got[fin], want[fin], rtol=1e-12, atol=0)
    best = min((v, i) for i, v in merged.items() if np.isfinite(v))
    assert best[1] == wbest
