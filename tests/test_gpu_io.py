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
    # valid JSON in another layout goes to the general reader (plan_json.cu)
    for t in (b"{}", b"[]", json.dumps(json.loads(text)).encode()[:-1] + b', "version": 2}'):
        got = _err(lambda: ctx.plan_from_json(t))
        want = _err(lambda: reference.plan_from_json(t))
        assert got is not None and want is not None and got[1] == want[1], (got, want)


# ---- the general reader: any JSON layout (plan_json.cu) ---------------------

def _dump(node, ind=None, sep=(", ", ": "), level=0, nl="\n"):
    """JSON text of a node tree whose objects are lists of (key, value) pairs
    (so keys can repeat and keep any order)."""
    pad = (nl + ind * (level + 1)) if ind is not None else ""
    end = (nl + ind * level) if ind is not None else ""
    item_sep = sep[0].rstrip() if ind is not None else sep[0]
    if isinstance(node, Obj):
        if not node.items:
            return "{}"
        return "{" + item_sep.join(pad + (k.text if isinstance(k, Raw) else json.dumps(k)) + sep[1] + _dump(v, ind, sep, level + 1, nl)
                                   for k, v in node.items) + end + "}"
    if isinstance(node, list):
        if not node:
            return "[]"
        return "[" + item_sep.join(pad + _dump(v, ind, sep, level + 1, nl) for v in node) + end + "]"
    if isinstance(node, Raw):
        return node.text
    return json.dumps(node)


class Obj:
    def __init__(self, items):
        self.items = list(items)


class Raw:
    def __init__(self, text):
        self.text = text


def _tree(v):
    if isinstance(v, dict):
        return Obj((k, _tree(x)) for k, x in v.items())
    if isinstance(v, list):
        return [_tree(x) for x in v]
    return v


def _walk(node, fn, path=()):
    """fn(path, obj) on every Obj (path: keys / 'i' for array elements)."""
    if isinstance(node, Obj):
        fn(path, node)
        for k, v in node.items:
            _walk(v, fn, path + (k,))
    elif isinstance(node, list):
        for v in node:
            _walk(v, fn, path + ("i",))


def _variants(text):
    doc = json.loads(text)
    yield "minified", json.dumps(doc, separators=(",", ":")).encode()
    yield "python_dumps", json.dumps(doc).encode()
    yield "indent4_crlf", json.dumps(doc, indent=4).replace("\n", "\r\n").encode()
    yield "bom_tabs", b"\xef\xbb\xbf" + _dump(_tree(doc), ind="\t").encode() + b"\n"
    yield "nul_ends_input", json.dumps(doc).encode() + b"\x00 trailing ] garbage"

    def rev(path, o):
        o.items.reverse()
    t = _tree(doc)
    _walk(t, rev)
    yield "keys_reversed", _dump(t, ind=" ").encode()

    def dup_and_unknown(path, o):
        keys = [k for k, _ in o.items]
        if "capacity" in keys:  # a pack: an earlier capacity, unknown members, extra sample elements
            o.items.insert(0, ("capacity", 0))
            o.items.insert(1, ("samples", [[1, 2, 3]]))
            o.items.append(("note", Obj([("x", [[1, 2], [3]]), ("cap", "no")])))
            for k, v in o.items:
                if k == "samples" and isinstance(v, list) and v and len(v[0]) == 2:
                    for smp in v:
                        smp.extend(["extra", Obj([("k", [1, [2]])]), None])
        elif "devices" in keys:  # an iteration: an earlier devices and group, unknown members
            o.items.insert(0, ("devices", [[Obj([("capacity", 1), ("samples", [[0, 5]])])]]))
            o.items.insert(0, ("group", "not read"))
            o.items.append(("meta", [Obj([("devs", [])]), [[[]]]]))
        elif "iterations" in keys:  # the root: an unknown member and an earlier iterations
            o.items.insert(0, ("iterations", [Obj([("group", 99)])]))
            o.items.append(("comment", "r\u00e9sum\u00e9 \\ \" ok"))
    t = _tree(doc)
    _walk(t, dup_and_unknown)
    yield "duplicates_unknown_extra", _dump(t, ind="  ").encode()

    def numbers(path, o):
        for i, (k, v) in enumerate(o.items):
            if k == "capacity":
                o.items[i] = (k, Raw(f"{v}.0"))
            if k == "samples":
                o.items[i] = (k, [[Raw(f"{a}e0"), Raw(f"{b * 10}E-1")] for a, b in v])
            if k == "group":
                o.items[i] = (Raw('"gr\\u006fup"'), Raw("true" if v == 1 else "false") if v in (0, 1) else v)
    t = _tree(doc)
    _walk(t, numbers)
    yield "floats_bools_escaped_keys", _dump(t).encode()


@pytest.mark.parametrize("name", ["c1_20k", "neg_ids_5k", "tiny_spill"])
def test_plan_from_json_any_layout(ctx, oracle, reference, name):
    ids, L, groups, kw = next((i, l, g, k) for n, i, l, g, k in cases(oracle) if n == name)
    text = ctx.build_plan(ids, L, groups, l_best=groups[0][0], **kw).to_json(ids, L)
    for vname, t in _variants(text.decode()):
        want = reference.plan_from_json(t)
        back, rid, rlen = ctx.plan_from_json(t)
        b = back.flat()
        for k in PLAN_KEYS:
            assert np.array_equal(getattr(b, k), getattr(want, k)), (vname, k)
        assert np.array_equal(rid, want.member_id) and np.array_equal(rlen, want.member_length), vname
        assert b.device_count == want.device_count and b.seed == want.seed, vname


def _same_error(ctx, reference, t):
    got = _err(lambda: ctx.plan_from_json(t))
    want = _err(lambda: reference.plan_from_json(t))
    assert got is not None and want is not None, (t[:200], got, want)
    assert got[1] == want[1], (t[:200], got, want)
    if want[1].startswith("[json.exception"):  # nlohmann's own exception: RuntimeError on both sides
        assert got[0] == "JsonError", got
    else:
        assert got[0] == want[0] == "ValidationError", (got, want)


def test_plan_from_json_general_errors(ctx, reference):
    L = np.array([100, 200, 300, 16000, 40000, 5, 7, 9000], dtype=np.int64)
    doc = json.loads(ctx.build_plan(None, L, [(16384, 1, 0), (65536, 2, 4)], l_best=16384, device_count=3,
                                    seed=11).to_json(None, L))
    base = json.dumps(doc)

    def edit(f):
        d = json.loads(base)
        f(d)
        return json.dumps(d).encode()

    def it0(d):
        return d["iterations"][0]

    def pk0(d):
        return next(p for it in d["iterations"] for dev in it["devices"] for p in dev)
    semantic = [
        edit(lambda d: pk0(d).__setitem__("capacity", "16384")),            # type_error 302
        edit(lambda d: it0(d).pop("phase")),                                 # out_of_range 403
        edit(lambda d: it0(d).pop("group")),
        edit(lambda d: it0(d).pop("devices")),
        edit(lambda d: pk0(d).pop("samples")),
        edit(lambda d: pk0(d).pop("capacity")),
        edit(lambda d: pk0(d)["samples"].__setitem__(0, [5])),               # out_of_range 401
        edit(lambda d: pk0(d)["samples"].__setitem__(0, [])),
        edit(lambda d: pk0(d)["samples"].__setitem__(0, {"a": 1})),          # type_error 304
        edit(lambda d: pk0(d)["samples"].__setitem__(0, ["x", 5])),          # type_error 302
        edit(lambda d: pk0(d)["samples"].__setitem__(0, [1, None])),
        edit(lambda d: pk0(d)["samples"].__setitem__(0, 7)),
        edit(lambda d: it0(d).__setitem__("phase", 3)),
        edit(lambda d: it0(d).__setitem__("group", 9)),                      # group range (ValidationError)
        edit(lambda d: it0(d).__setitem__("group", -1)),
        edit(lambda d: it0(d).__setitem__("group", [1])),
        edit(lambda d: pk0(d).__setitem__("capacity", 1)),                   # pack exceeds its capacity
        edit(lambda d: it0(d)["devices"].__setitem__(0, 5)),
        edit(lambda d: it0(d)["devices"].__setitem__(0, [3])),
        edit(lambda d: d.__setitem__("iterations", 5)),
        edit(lambda d: d["iterations"].append(4)),
        edit(lambda d: d.pop("iterations")),
        edit(lambda d: d.pop("seed")),
        edit(lambda d: d.__setitem__("device_count", "3")),
        edit(lambda d: d["groups"]["groups"][0].__setitem__("sp", 0)),
        edit(lambda d: d.__setitem__("version", 2)),
        edit(lambda d: d.pop("version")),
        b"[]", b"{}", b"7", b'"plan"', b"null",
    ]
    invalid = [base[:-1], base + ",", base + " 1", base.replace(": ", " ", 1), base.replace("]", "}", 1),
               base.replace("[", "{", 1), base.replace(", ", ",,", 1), base.replace("]]", "],]", 1),
               base.replace('"phase"', '"ph\\xase"', 1), base.replace('"phase"', '"ph\tase"', 1),
               base.replace('"phase"', '"\\ud800"', 1), base.replace("1", "01", 1), base.replace("100", "1.", 1),
               base.replace("100", "-", 1), base.replace("100", "1e", 1), base.replace("100", "+100", 1),
               base.replace("null", "nul") if "null" in base else base.replace("[", "[nul,", 1),
               base.replace("[", "[tru,", 1), base.replace("[", "[True,", 1), base.replace('"seed"', "seed", 1),
               "", "   ", base.replace('"', "'", 2), "\x00" + base, "\xef\xbb" + base]
    for t in semantic:
        _same_error(ctx, reference, t)
    for t in invalid:
        tb = t.encode() if isinstance(t, str) else t
        _same_error(ctx, reference, tb)


def test_plan_from_json_object_where_array_is_iterated(ctx, reference):
    """nlohmann iterates an object's values (key order) where the reference
    range-fors over devices / packs / samples; this reader refuses that
    layout with a validation error instead (known gaps)."""
    L = np.array([100, 200, 300], dtype=np.int64)
    d = json.loads(ctx.build_plan(None, L, [(16384, 1, 0)], l_best=16384, device_count=2, seed=1).to_json(None, L))
    d["iterations"][0]["devices"] = {"a": d["iterations"][0]["devices"][0], "b": d["iterations"][0]["devices"][1]}
    t = json.dumps(d).encode()
    reference.plan_from_json(t)  # the reference reads it
    got = _err(lambda: ctx.plan_from_json(t))
    assert got is not None and got[0] == "ValidationError" and "GPU reader" in got[1]


def test_plan_from_json_fuzzed(ctx, reference):
    """Byte-level mutations of a small manifest in a non-canonical layout:
    the reader accepts exactly what the reference accepts, with the same plan,
    and otherwise fails with the same message."""
    L = np.array([100, 200, 300, 16000, 40000, 5, 7, 9000, 1, 2], dtype=np.int64)
    base = json.dumps(json.loads(ctx.build_plan(None, L, [(16384, 1, 0), (65536, 2, 4)], l_best=16384,
                                                device_count=3, seed=11).to_json(None, L))).encode()
    rng = np.random.default_rng(2026)
    alphabet = b' \t\r\n{}[]:,"\\-+.0123456789eEtrufalsn\x00\xc3\xa9u'
    agree = 0
    for _ in range(400):
        t = bytearray(base)
        for _ in range(int(rng.integers(1, 3))):
            op, i = int(rng.integers(0, 3)), int(rng.integers(0, len(t)))
            ch = alphabet[int(rng.integers(0, len(alphabet)))]
            if op == 0:
                t[i] = ch
            elif op == 1:
                t.insert(i, ch)
            elif len(t) > 1:
                del t[i]
        t = bytes(t)
        want = _err(lambda: reference.plan_from_json(t))
        if want is None:
            back, rid, rlen = ctx.plan_from_json(t)
            w = reference.plan_from_json(t)
            b = back.flat()
            for k in PLAN_KEYS:
                assert np.array_equal(getattr(b, k), getattr(w, k)), (t, k)
            assert np.array_equal(rid, w.member_id) and np.array_equal(rlen, w.member_length), t
            agree += 1
        else:
            got = _err(lambda: ctx.plan_from_json(t))
            assert got is not None and got[1] == want[1], (t, got, want)
    assert agree > 20  # some mutations keep a valid manifest (white space, digits)


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
