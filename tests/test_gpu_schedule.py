"""GPU curriculum_order / assign_runtime / write_schedule_csv (src/schedule.cpp)
against the reference: manifests and schedule CSV byte-identical (digests
the reference produced, tests/golden/make_plan_json_golden.py; byte for
byte against the compiled reference when present), error messages."""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2503_07680_b200 import abi

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "plan_json_golden.json")))
GROUPS = [(8192, 1, 0), (32768, 4, 2), (131072, 8, 27)]


def c1(oracle):
    return np.maximum(oracle.synth(20_000, "lognormal:8.5:1.4", 0.0, "", 131072, 42), 128)


@pytest.mark.parametrize("warm,cut", [(300, 1), (0, 2)])
def test_curriculum_matches_reference_digest(ctx, oracle, warm, cut):
    L = c1(oracle)
    plan = ctx.build_plan(None, L, GROUPS, l_best=8192, device_count=8, seed=7)
    cur = plan.curriculum_order(warm, cut)
    g = GOLD[f"curriculum_w{warm}_c{cut}"]
    text = cur.to_json(None, L)
    assert len(text) == g["bytes"]
    assert hashlib.sha256(text).hexdigest() == g["sha256"]
    assert hashlib.sha256(cur.schedule_csv()).hexdigest() == g["csv_sha256"]
    sp, ck, sw = cur.assign_runtime()
    assert sw == g["switch_count"]
    # a permutation of the plan's iterations: same report
    assert cur.report().abr == pytest.approx(plan.report().abr, rel=1e-12)


def test_curriculum_vs_compiled_reference(ctx, oracle):
    try:
        from pyoracle import Oracle
        ref = Oracle("reference")
    except (ImportError, FileNotFoundError, OSError):
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(2)
    L = oracle.synth(30_000, "lognormal:7.2:0.7", 0.03, "uniform:16385:131072", 131072, 31)
    ids = rng.permutation(90_000)[:30_000].astype(np.int64) - 40_000
    groups = [(16384, 1, 28), (131072, 8, 29)]
    for warm in (0, 50, 700):
        j, c, sp, ck, sw = ref.curriculum(ids, L, groups, 16384, warm, 1, device_count=4, seed=9)
        cur = ctx.build_plan(ids, L, groups, l_best=16384, device_count=4, seed=9).curriculum_order(warm, 1)
        assert cur.to_json(ids, L) == j
        assert cur.schedule_csv() == c
        gsp, gck, gsw = cur.assign_runtime()
        assert np.array_equal(gsp, sp) and np.array_equal(gck, ck) and gsw == sw
    # too few short iterations: the same message on both sides
    msgs = []
    for f in (lambda: ref.curriculum(ids, L, groups, 16384, 100000, 1, device_count=4, seed=9),
              lambda: ctx.build_plan(ids, L, groups, l_best=16384, device_count=4, seed=9).curriculum_order(100000, 1)):
        with pytest.raises(abi.ValidationError) as e:
            f()
        msgs.append(str(e.value))
    assert msgs[0] == msgs[1]


def test_curriculum_errors(ctx, oracle):
    L = c1(oracle)[:3000]
    plan = ctx.build_plan(None, L, GROUPS, l_best=8192, device_count=8, seed=7)
    with pytest.raises(abi.ValidationError, match="warmup_iterations must be >= 0"):
        plan.curriculum_order(-1, 1)
    with pytest.raises(abi.ValidationError, match="short_group_cutoff must select at least one group"):
        plan.curriculum_order(1, 4)
    with pytest.raises(abi.ValidationError, match="curriculum needs 100000 short-group iterations but the plan has only"):
        plan.curriculum_order(100000, 1)
