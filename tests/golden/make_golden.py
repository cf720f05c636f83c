#!/usr/bin/env python3
"""Regenerates tests/golden/*.json from the REFERENCE itself.

Runs the reference planner compiled in place (oracle/_ref/libhbp_ref.so,
built by `make -C oracle` from /root/reference/proj/src) and reads the
reference's data fixtures (/root/reference/proj/data/profiles). The JSON it
writes pins the oracle restatement (tests/test_oracle.py) and the CUDA
engine (tests/test_gpu_*.py) on machines where /root/reference is absent.

    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_2503_07680_b200 import abi  # noqa: E402
from pyoracle import Oracle  # noqa: E402

REF_DATA = "/root/reference/proj/data/profiles"

PLAN_KEYS = ["iter_group", "iter_dev_offsets", "dev_index", "dev_pack_offsets", "pack_capacity",
             "pack_total", "pack_attention", "pack_member_offsets", "member_id", "member_length"]


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def plan_digests(p) -> dict:
    return {k: digest(getattr(p, k)) for k in PLAN_KEYS} | {
        "n_iterations": int(p.n_iterations), "n_packs": int(len(p.pack_capacity)),
        "n_members": int(len(p.member_id))}


def main():
    ref = Oracle("reference")
    out = {}
    # ---- reference data fixtures (cost-model inputs) -----------------------
    with open(os.path.join(REF_DATA, "group_candidates_8b.csv")) as f:
        cand_rows = abi.parse_table_csv(f.read())
    with open(os.path.join(REF_DATA, "gc_sweep_8b.csv")) as f:
        sweep_rows = abi.parse_table_csv(f.read())
    with open(os.path.join(REF_DATA, "analytic_default.json")) as f:
        analytic = json.load(f)
    out["profiles"] = {"group_candidates_8b": cand_rows, "gc_sweep_8b": sweep_rows,
                       "analytic_default": analytic}

    # ---- auto-selection known answers --------------------------------------
    ka = {}
    t = abi.table_profiler(cand_rows)
    ka["select_groups_candidates_8b"] = ref.select_groups([8192, 16384, 32768, 65536, 131072], t, [1, 2, 4, 8, 16])
    an = abi.analytic_profiler()
    ka["select_groups_analytic_default"] = ref.select_groups([8192, 16384, 32768, 65536, 131072], an, [1, 2, 4, 8, 16])
    st = abi.table_profiler(sweep_rows)
    ka["find_best_32k"] = ref.find_best_sp_ckpt(st, 32768, [2, 4, 8, 16])
    ka["find_best_128k"] = ref.find_best_sp_ckpt(st, 131072, [2, 4, 8, 16])
    derive = {}
    for l in [512, 1024, 2048, 4096, 8192, 16384, 32768, 65536, 131072]:
        for sp in [1, 2, 4, 8]:
            try:
                derive[f"{l}/{sp}"] = ref.derive_ckpt(an, l, sp)
            except Exception as e:  # noqa: BLE001
                derive[f"{l}/{sp}"] = f"{type(e).__name__}: {e}"
    ka["analytic_derive_ckpt"] = derive
    mem = {}
    for l in [4096, 16384, 32768, 131072]:
        for sp in [1, 2, 8]:
            for ck in [0, 16, 32]:
                mem[f"{l}/{sp}/{ck}"] = ref.memory_used(l, sp, ck)
    ka["memory_used"] = mem
    out["autoselect"] = ka

    # ---- plans: digests of the reference output ------------------------------
    plans = {}
    cases = [
        ("c1_100k", dict(count=100_000, short="lognormal:8.5:1.4", lf=0.0, long="", seed=42, floor=128),
         # ckpt = AnalyticProfiler(defaults).derive_ckpt(l, sp)
         [(8192, 1, 11), (32768, 4, 11), (131072, 8, 27)], 8192, dict(device_count=8, seed=7)),
        ("c2_shape_300k", dict(count=300_000, short="lognormal:7.2:0.7", lf=0.02, long="uniform:16385:131072",
                               seed=20250515, floor=1),
         [(16384, 1, 28), (131072, 8, 28)], 16384, dict(device_count=8, seed=1)),
        ("hybrid_20k_random_batching", dict(count=20_000, short="lognormal:7.2:0.7", lf=0.03,
                                            long="uniform:16385:131072", seed=11, floor=1),
         [(16384, 1, 28), (131072, 8, 29)], 16384, dict(device_count=4, seed=7, balance_batching=False)),
        ("hybrid_5k_ffd", dict(count=5_000, short="lognormal:7.2:0.7", lf=0.03, long="uniform:16385:131072",
                               seed=3, floor=1),
         [(16384, 1, 28), (131072, 8, 29)], 16384, dict(device_count=4, seed=1, strategy="ffd")),
    ]
    for name, spec, groups, l_best, opts in cases:
        L = np.maximum(ref.synth(spec["count"], spec["short"], spec["lf"], spec["long"], 131072, spec["seed"]),
                       spec["floor"])
        p = ref.build_plan(None, L, groups, l_best=l_best, **opts)
        m, dbr, abr_ = ref.report(p)
        try:
            s = ref.simulate(p)[0]
            sim = {"total_seconds": s.total_seconds, "gpu_days": s.gpu_days, "switch_count": s.switch_count}
        except abi.InfeasibleError as e:
            sim = {"error": str(e)}
        plans[name] = {"spec": spec, "groups": groups, "l_best": l_best, "options": opts,
                       "lengths_sha256": digest(L), "plan": plan_digests(p),
                       "report": {k: getattr(m, k) for k in ("dbr", "pr", "abr", "cr", "ave_t")},
                       "per_iteration_sha256": hashlib.sha256(np.concatenate([dbr, abr_]).tobytes()).hexdigest(),
                       "simulate": sim}
    out["plans"] = plans

    # ---- packing known answers ----------------------------------------------
    pk = {}
    rng = np.random.default_rng(2024)
    for kind in ["random", "isf", "ffs", "ffd", "bfs", "spfhp"]:
        L = rng.integers(1, 978, size=120)
        p = ref.pack(None, L, 1024, kind, seed=12345)
        pk[kind] = {"lengths": L.tolist(), "pack_member_offsets": p.pack_member_offsets.tolist(),
                    "member_id": p.member_id.tolist()}
    out["pack"] = pk
    with open(os.path.join(HERE, "reference_golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", os.path.join(HERE, "reference_golden.json"))


if __name__ == "__main__":
    main()
