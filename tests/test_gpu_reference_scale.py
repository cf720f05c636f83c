"""The GPU engine against answers the REFERENCE itself produced at the
benchmarked sizes (tests/golden/scale_golden.json, make_scale_golden.py:
oracle/_ref = proj/src compiled in place), with no restatement in between:

  C2 10M   build_plan digests (balance.cpp:207-258), report (metrics.cpp:
           107-144), simulate (sim.cpp:9-60) -- bench.py's workload
  C1 1M    the same at C1's spec
  C3       all 2048 candidates of the auto-selection sweep over C1's 100K
           corpus: per-candidate seconds, feasibility, argmin -- bench.py's
           sweep leg

Plans bit-exact (SHA-256 of every plan array); per-iteration DBR/ABR
bit-exact; run-level means and totals within 1e-9 relative (north star:
1e-6)."""
import hashlib
import json
import math
import os

import numpy as np
import pytest

from paper_2503_07680_b200 import abi, sweep

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "scale_golden.json")))
KEYS = ["iter_group", "iter_dev_offsets", "dev_index", "dev_pack_offsets", "pack_capacity", "pack_total",
        "pack_attention", "pack_member_offsets"]


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def corpus(spec):
    # the engine's generator (csrc/synth.cpp), pinned to the reference's by lengths_sha256
    from bench import synth
    L = synth(abi.load_library(), dict(count=spec["count"], short=spec["short"], long_fraction=spec["lf"],
                                       long=spec["long"], max_length=131072, seed=spec["seed"]))
    return np.maximum(L, spec["floor"])


@pytest.mark.parametrize("name", ["c1_1m", "c2_10m"])
def test_plan_vs_reference_digest(ctx, name):
    case = GOLD[name]
    L = corpus(case["spec"])
    assert digest(L) == case["lengths_sha256"]
    groups = [tuple(g) for g in case["groups"]]
    plan = ctx.build_plan(None, L, groups, l_best=case["l_best"], **case["options"])
    got = plan.flat()
    want = case["plan"]
    assert got.n_iterations == want["n_iterations"]
    assert len(got.pack_capacity) == want["n_packs"]
    for k in KEYS:
        assert digest(getattr(got, k)) == want[k], k
    ids = got.members_as_ids(None)
    assert digest(ids) == want["member_id"]
    assert digest(L[got.member_index]) == want["member_length"]
    m, dbr, abr_ = ctx.report(got)
    assert hashlib.sha256(np.concatenate([dbr, abr_]).tobytes()).hexdigest() == case["per_iteration_sha256"]
    for k, v in case["report"].items():
        assert getattr(m, k) == pytest.approx(v, rel=1e-9, abs=0), k
    st = plan.simulate(abi.default_profile())
    assert st.total_seconds == pytest.approx(case["simulate"]["total_seconds"], rel=1e-9)
    assert st.switch_count == case["simulate"]["switch_count"]


def test_c3_full_sweep_vs_reference(ctx):
    g = GOLD["c3"]
    L = corpus(g["corpus"])
    cands = sweep.make_candidates(ctx, 131072, [512, 1024, 2048, 4096, 8192, 16384, 32768, 65536], [1, 2, 4, 8])
    assert [[list(map(list, c[0])), c[1]] for c in cands] == g["candidates"]  # same ckpt from derive_ckpt
    s, keep = abi.make_samples(None, L, "c3")
    secs, best = ctx.sweep_samples(s, cands, None, **g["options"])
    want = np.array([math.inf if x == "inf" else x for x in g["seconds"]])
    assert np.array_equal(np.isinf(secs), np.isinf(want))
    fin = np.isfinite(want)
    assert int(fin.sum()) == g["feasible"] == 252
    assert np.allclose(secs[fin], want[fin], rtol=1e-12, atol=0)
    assert best == g["best_index"] == 734
    assert secs[best] == pytest.approx(g["best_seconds"], rel=1e-12)
