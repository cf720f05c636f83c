"""GPU plan manifest writer (hbp_plan_to_json) against the reference's
plan_to_json (src/io.cpp:85-110): byte-identical text, checked by SHA-256
against digests the reference itself produced (tests/golden/
make_plan_json_golden.py), and byte for byte against the compiled reference
(oracle/_ref) when it is present."""
import hashlib
import json
import os
import re

import numpy as np
import pytest

from paper_2503_07680_b200 import abi

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "plan_json_golden.json")))
TWO_LEVEL = [(16384, 1, 28), (131072, 8, 29)]
C1_GROUPS = [(8192, 1, 0), (32768, 4, 0), (131072, 8, 0)]


def cases(oracle):
    L1 = np.maximum(oracle.synth(20_000, "lognormal:8.5:1.4", 0.0, "", 131072, 42), 128)
    yield "c1_20k", None, L1, C1_GROUPS, dict(device_count=8, seed=7)
    rng = np.random.default_rng(3)
    L2 = oracle.synth(5_000, "lognormal:7.2:0.7", 0.05, "uniform:16385:131072", 131072, 9)
    ids = rng.permutation(40_000)[:5_000].astype(np.int64) - 20_000
    yield "neg_ids_5k", ids, L2, TWO_LEVEL, dict(device_count=4, seed=5)
    L3 = np.array([100, 200, 300, 16000, 40000, 5, 7, 9000], dtype=np.int64)
    yield "tiny_spill", None, L3, [(16384, 1, 0), (65536, 2, 4)], dict(device_count=3, seed=11)


@pytest.mark.parametrize("name", ["c1_20k", "neg_ids_5k", "tiny_spill"])
def test_plan_json_matches_reference_digest(ctx, oracle, name):
    for case, ids, L, groups, opts in cases(oracle):
        if case != name:
            continue
        text = ctx.build_plan(ids, L, groups, l_best=groups[0][0], **opts).to_json(ids, L)
        g = GOLD[name]
        assert len(text) == g["bytes"]
        assert text[:300].decode() == g["head"]
        assert hashlib.sha256(text).hexdigest() == g["sha256"]


def test_plan_json_bytes_vs_compiled_reference(ctx, oracle):
    try:
        from pyoracle import Oracle
        ref = Oracle("reference")
    except (ImportError, FileNotFoundError, OSError):
        pytest.skip("oracle/_ref not built")
    L = oracle.synth(30_000, "lognormal:7.2:0.7", 0.03, "uniform:16385:131072", 131072, 21)
    ids = np.arange(len(L), dtype=np.int64) * 7 - 1000
    for groups in (TWO_LEVEL, C1_GROUPS):
        want = ref.build_plan_json(ids, L, groups, l_best=groups[0][0], device_count=8, seed=3)
        got = ctx.build_plan(ids, L, groups, l_best=groups[0][0], device_count=8, seed=3).to_json(ids, L)
        if got != want:
            k = next(i for i in range(min(len(got), len(want))) if got[i] != want[i])
            raise AssertionError(f"first difference at byte {k}: {got[k-80:k+40]!r} vs {want[k-80:k+40]!r}")


def test_plan_json_buffer_too_small(ctx):
    L = np.array([100, 200, 300], dtype=np.int64)
    plan = ctx.build_plan(None, L, [(1024, 1, 0)], l_best=1024, device_count=2, seed=1)
    s, keep = abi.make_samples(None, L, "t")
    import ctypes as C
    n = C.c_int64()
    lib = ctx.lib
    lib.hbp_plan_to_json.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(abi.Samples), C.c_char_p, C.c_int64,
                                     C.POINTER(C.c_int64)]
    assert lib.hbp_plan_to_json(ctx.h, plan.h, C.byref(s), None, 0, C.byref(n)) == 0
    buf = C.create_string_buffer(8)
    assert lib.hbp_plan_to_json(ctx.h, plan.h, C.byref(s), buf, 8, C.byref(n)) == abi.HBP_ERR_VALIDATION


def batching_cases(oracle):
    L = np.maximum(oracle.synth(8_000, "lognormal:7.2:0.9", 0.0, "", 16384, 5), 1)
    yield "batching_sorted_8k", None, L, (16384, 1, 0), 8, "sorted", 0
    rng = np.random.default_rng(8)
    ids = rng.permutation(30_000)[:8_000].astype(np.int64) - 10_000
    yield "batching_random_8k", ids, L, (32768, 2, 4), 3, "random", 99


@pytest.mark.parametrize("name", ["batching_sorted_8k", "batching_random_8k"])
def test_batching_plan_matches_reference_digest(ctx, oracle, name):
    # build_batching_plan (balance.cpp:260-298) -> plan_to_json, byte-identical
    for case, ids, L, group, dc, mode, seed in batching_cases(oracle):
        if case != name:
            continue
        plan = ctx.build_batching_plan(ids, L, group, device_count=dc, mode=mode, seed=seed)
        text = plan.to_json(ids, L)
        assert len(text) == GOLD[name]["bytes"]
        assert hashlib.sha256(text).hexdigest() == GOLD[name]["sha256"]
        # the plan feeds report / simulate like any other
        assert plan.report().ave_t > 0


@pytest.mark.parametrize("mode,budget", [("sorted", 16384), ("random", 16384), ("random", 131072)])
def test_padded_batching_vs_compiled_reference(ctx, oracle, mode, budget):
    try:
        from pyoracle import Oracle
        ref = Oracle("reference")
    except (ImportError, FileNotFoundError, OSError):
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(budget)
    L = np.maximum(oracle.synth(50_000, "lognormal:7.0:1.0", 0.0, "", 16384, 13), 1)
    ids = rng.permutation(100_000)[:50_000].astype(np.int64) - 30_000
    order, off, mx = ctx.padded_batching(ids, L, budget, mode, seed=4)
    r_order, r_off, r_mx = ref.padded_batching(ids, L, budget, mode, seed=4)
    assert np.array_equal(ids[order], r_order)
    assert np.array_equal(off, r_off)
    assert np.array_equal(mx, r_mx)


def test_padded_batching_budget_error(ctx):
    with pytest.raises(abi.ValidationError, match=r"token budget 100 is below the longest sample \(300\)"):
        ctx.padded_batching(None, np.array([100, 300, 5], dtype=np.int64), 100, "sorted")


# ---- reader: hbp_plan_from_json (io.cpp:112-160) ---------------------------

PLAN_KEYS = ["iter_group", "iter_dev_offsets", "dev_index", "dev_pack_offsets", "pack_capacity", "pack_total",
             "pack_attention", "pack_member_offsets"]


@pytest.mark.parametrize("name", ["c1_20k", "neg_ids_5k", "tiny_spill"])
def test_plan_from_json_round_trip(ctx, oracle, reference, name):
    ids, L, groups, kw = next((i, l, g, k) for n, i, l, g, k in cases(oracle) if n == name)
    plan = ctx.build_plan(ids, L, groups, l_best=groups[0][0], **kw)
    text = plan.to_json(ids, L)
    back, rid, rlen = ctx.plan_from_json(text)
    a, b = plan.flat(), back.flat()
    for k in PLAN_KEYS:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    full_ids = np.arange(len(L)) if ids is None else ids
    assert np.array_equal(rid, full_ids[a.member_index]) and np.array_equal(rlen, L[a.member_index])
    assert back.to_json(rid, rlen) == text  # save / load / save is bit-exact (test_io.cpp:33-53)
    want = reference.plan_from_json(text)
    for k in PLAN_KEYS:
        assert np.array_equal(getattr(b, k), getattr(want, k)), k
    assert np.array_equal(rid, want.member_id) and np.array_equal(rlen, want.member_length)


def test_plan_from_json_curriculum_phases(ctx, oracle, reference):
    L = np.maximum(oracle.synth(20_000, "lognormal:8.5:1.4", 0.0, "", 131072, 42), 128)
    plan = ctx.build_plan(None, L, C1_GROUPS, l_best=8192, device_count=8, seed=7).curriculum_order(50, 1)
    text = plan.to_json(None, L)
    assert b'"warmup"' in text
    back, rid, rlen = ctx.plan_from_json(text)
    assert back.to_json(rid, rlen) == text


def _err(fn):
    try:
        fn()
    except (abi.ValidationError, Exception) as e:  # noqa: BLE001
        return type(e).__name__, str(e)
    return None


def test_plan_from_json_errors(ctx, oracle, reference):
    L = np.array([100, 200, 300, 16000, 40000, 5, 7, 9000], dtype=np.int64)
    text = ctx.build_plan(None, L, [(16384, 1, 0), (65536, 2, 4)], l_best=16384, device_count=3, seed=11).to_json(None, L)
    edits = [
        text.replace(b'"version": 1', b'"version": 2'),                       # unsupported version
        text.replace(b'"group": 1', b'"group": 5', 1),                        # group index out of range
        re.sub(rb'"capacity": \d+', b'"capacity": 1', text, count=1),      # pack exceeds capacity
        text.replace(b'"sp": 1', b'"sp": 0', 1),                              # groups validate
        text[: len(text) // 2],                                               # not JSON
        b"not json",
    ]
    for t in edits:
        assert t != text
        got = _err(lambda: ctx.plan_from_json(t))
        want = _err(lambda: reference.plan_from_json(t))
        assert got is not None and want is not None
        assert got[1] == want[1], (got, want)
    # valid JSON in another layout: the reference reads it (or rejects "{}"),
    # this reader refuses it as a validation error
    for t in (b"{}", json.dumps(json.loads(text)).encode()):
        got = _err(lambda: ctx.plan_from_json(t))
        assert got is not None and got[0] == "ValidationError"


@pytest.mark.parametrize("n,devices,seed", [(1, 8, 0), (3, 16, 1), (17, 5, 2), (64, 3, 3), (500, 7, 4)])
def test_plan_from_json_edge_plans(ctx, oracle, reference, n, devices, seed):
    # tiny corpora: spill tails, idle devices ("[]"), single-pack iterations
    rng = np.random.default_rng(seed)
    L = rng.integers(1, 131073, size=n).astype(np.int64)
    plan = ctx.build_plan(None, L, TWO_LEVEL, l_best=16384, device_count=devices, seed=seed)
    text = plan.to_json(None, L)
    back, rid, rlen = ctx.plan_from_json(text)
    assert back.to_json(rid, rlen) == text
    want = reference.plan_from_json(text)
    b = back.flat()
    for k in PLAN_KEYS:
        assert np.array_equal(getattr(b, k), getattr(want, k)), k
    assert np.array_equal(rid, want.member_id) and np.array_equal(rlen, want.member_length)


@pytest.mark.parametrize("mode", ["sorted", "random"])
def test_plan_from_json_batching_plan(ctx, oracle, reference, mode):
    L = oracle.synth(3_000, "lognormal:7.2:0.7", 0.05, "uniform:16385:131072", 131072, 9)
    plan = ctx.build_batching_plan(None, L, (131072, 8, 27), 4, mode, 7)
    text = plan.to_json(None, L)
    back, rid, rlen = ctx.plan_from_json(text)
    assert back.to_json(rid, rlen) == text
    want = reference.plan_from_json(text)
    assert np.array_equal(back.flat().pack_member_offsets, want.pack_member_offsets)
