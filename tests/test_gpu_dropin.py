"""The reference's public APIs, unchanged, running on the B200 engine:

* the C++ API (include/hbp/*.hpp) through tests/cpp/test_dropin.cpp, a port
  of the reference test suite's known answers linked like hbp_core;
* the Python module (paper_2503_07680_b200.hbp == reference `hbp`), checked
  against the oracle restatement on the same inputs.
"""
import json
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_golden.json")))


def test_cpp_dropin_suite():
    exe = os.path.join(ROOT, "tests", "cpp", "test_dropin")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.fixture(scope="module")
def hbp():
    from paper_2503_07680_b200 import hbp as mod
    return mod


def groups_obj(hbp, groups, l_best):
    return hbp.HierarchicalGroups([hbp.GroupConfig(l, hbp.RuntimeConfig(sp, ck)) for (l, sp, ck) in groups],
                                  l_best, groups[-1][0])


def test_python_build_plan_matches_oracle(hbp, oracle):
    L = oracle.synth(30_000, "lognormal:7.2:0.7", 0.03, "uniform:16385:131072", 131072, 9)
    groups = [(16384, 1, 27), (131072, 8, 27)]
    plan = hbp.build_plan(hbp.SampleSet(L.tolist()), groups_obj(hbp, groups, 16384), device_count=8, seed=3)
    want = oracle.build_plan(None, L, groups, l_best=16384, device_count=8, seed=3)
    got_members = [s.id for it in plan.iterations for d in it.devices for p in d.packs for s in p.samples]
    assert got_members == want.member_id.tolist()
    assert [it.group_index for it in plan.iterations] == want.iter_group.tolist()
    rep = hbp.report(plan)
    m = oracle.report(want)[0]
    assert rep.abr == pytest.approx(m.abr, rel=1e-12) and rep.cr == m.cr and rep.pr == m.pr
    sim = hbp.simulate(plan, hbp.HardwareProfile(), "hbp")
    assert sim.total_seconds == pytest.approx(oracle.simulate(want)[0].total_seconds, rel=1e-12)


def test_python_select_groups_table(hbp, tmp_path):
    rows = GOLD["profiles"]["group_candidates_8b"]
    path = tmp_path / "group_candidates_8b.csv"
    path.write_text("length,sp,ckpt,memory_bytes,iter_seconds\n" + "".join(
        f"{l},{sp},{ck},{'oom' if mem is None else mem},{sec}\n" for l, sp, ck, mem, sec in rows))
    t = hbp.TableProfiler.from_csv_file(str(path))
    g = hbp.select_groups([8192, 16384, 32768, 65536, 131072], t, [1, 2, 4, 8, 16])
    assert [(x.length, x.config.sp, x.config.ckpt) for x in g.groups] == \
        [tuple(x) for x in GOLD["autoselect"]["select_groups_candidates_8b"][0]]


def test_python_exceptions(hbp):
    with pytest.raises(ValueError, match="non-positive length 0"):
        hbp.SampleSet([1, 0])
    with pytest.raises(ValueError, match="sample 1"):
        hbp.pack(hbp.SampleSet([3, 9, 2]), 4, "ffd")
    tiny = hbp.HardwareProfile()
    tiny.device_memory = 25 << 30
    L = [1000] * 64
    plan = hbp.build_plan(hbp.SampleSet(L), groups_obj(hbp, [(16384, 1, 0)], 16384), device_count=2)
    with pytest.raises(RuntimeError, match="iteration 0"):
        hbp.simulate(plan, tiny)


def test_python_pack_strategies(hbp, oracle):
    rng = np.random.default_rng(5)
    L = rng.integers(1, 978, size=500)
    for kind in ["isf", "random", "ffd", "ffs", "bfs", "spfhp"]:
        got = hbp.pack(hbp.SampleSet(L.tolist()), 1024, kind, 77)
        want = oracle.pack(None, L, 1024, kind, seed=77)
        ids = [s.id for p in got.packs for s in p.samples]
        assert ids == want.member_id.tolist(), kind


def test_python_load_lengths(hbp, tmp_path):
    # ingest.hpp:22 / py_hbp.cpp:74-78: load_lengths(path, format="jsonl")
    p = tmp_path / "c.jsonl"
    p.write_bytes(b'{"id":7,"length":10}\n\n{"length":20}\n')
    s = hbp.load_lengths(str(p))
    assert [(x.id, x.length) for x in s.samples] == [(7, 10), (1, 20)] and s.source == str(p)
    q = tmp_path / "c.csv"
    q.write_bytes(b"name,length\na,3\nb,4\n")
    assert hbp.load_lengths(str(q), "csv").lengths == [3, 4]
    r = tmp_path / "c.txt"
    r.write_bytes(b"10\nnonsense\n30\n")
    with pytest.raises(ValueError, match="line 2: not an integer length: 'nonsense'"):
        hbp.load_lengths(str(r), "raw-lengths")
    with pytest.raises(OSError, match="cannot open corpus file"):
        hbp.load_lengths(str(tmp_path / "missing.txt"), "raw")
    with pytest.raises(ValueError, match="unknown corpus format: xml"):
        hbp.load_lengths(str(r), "xml")


def test_python_plan_manifest(hbp, tmp_path):
    # Plan.to_json / Plan.from_json / write_plan / read_plan (py_hbp.cpp:300-305, 423-424)
    L = [100, 200, 300, 16000, 40000, 5, 7, 9000] * 50
    plan = hbp.build_plan(hbp.SampleSet(L), groups_obj(hbp, [(16384, 1, 0), (65536, 2, 4)], 16384), device_count=3,
                          seed=11)
    text = plan.to_json()
    back = hbp.Plan.from_json(text)
    assert back.to_json() == text and len(back.iterations) == len(plan.iterations)
    assert [[[s.id for p in d.packs for s in p.samples] for d in it.devices] for it in back.iterations] == \
        [[[s.id for p in d.packs for s in p.samples] for d in it.devices] for it in plan.iterations]
    assert hbp.report(back).abr == hbp.report(plan).abr
    path = tmp_path / "plan.json"
    hbp.write_plan(plan, str(path))
    assert path.read_bytes() == text.encode()
    assert hbp.read_plan(str(path)).to_json() == text
    with pytest.raises(OSError, match="cannot open file"):
        hbp.read_plan(str(tmp_path / "missing.json"))
    with pytest.raises(ValueError, match="bad plan manifest"):
        hbp.Plan.from_json("not json")


def test_python_curriculum_and_runtime(hbp, reference):
    # curriculum_order / assign_runtime (py_hbp.cpp:350-370) through the
    # facade: same iteration order, phases and switch count as the reference
    import numpy as np
    L = np.maximum(reference.synth(20_000, "lognormal:8.5:1.4", 0.0, "", 131072, 42), 128)
    groups = [(8192, 1, 0), (32768, 4, 0), (131072, 8, 0)]
    plan = hbp.build_plan(hbp.SampleSet(L.tolist()), groups_obj(hbp, groups, 8192), device_count=8, seed=7)
    cur = hbp.curriculum_order(plan, hbp.CurriculumSpec(50, 1))
    assert sum(1 for it in cur.iterations if str(it.phase).endswith("Warmup")) == 50
    jt, ct, sp, ck, sw = reference.curriculum(None, L, groups, 8192, 50, 1, device_count=8, seed=7)
    assert cur.to_json().encode() == jt  # same order, phases and packs as the reference
    per_it, switches = hbp.assign_runtime(cur)
    assert [rc.sp for rc in per_it] == sp.tolist() and [rc.ckpt for rc in per_it] == ck.tolist() and switches == sw
    assert len(per_it) == len(cur.iterations)
    assert all(rc.sp == groups[it.group_index][1] for rc, it in zip(per_it, cur.iterations))
    changes = sum(1 for a, b in zip(per_it, per_it[1:]) if (a.sp, a.ckpt) != (b.sp, b.ckpt))
    assert switches == changes
    with pytest.raises(ValueError):
        hbp.curriculum_order(plan, hbp.CurriculumSpec(10 ** 6, 1))
