"""TEST INFRASTRUCTURE ONLY: ctypes access to the two oracle libraries.

    Oracle("restatement")  -> oracle/liboracle_hbp.so  (plain-C restatement)
    Oracle("reference")    -> oracle/_ref/libhbp_ref.so (reference compiled in place)

Both export the ABI of oracle/oracle.h. Imported only by tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs.
"""
from __future__ import annotations

import ctypes as C
import os
import sys
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from paper_2503_07680_b200 import abi  # noqa: E402  (structs only)

PATHS = {
    "restatement": os.path.join(HERE, "liboracle_hbp.so"),
    "reference": os.path.join(HERE, "_ref", "libhbp_ref.so"),
}


class OraclePlan(C.Structure):
    _fields_ = [("device_count", C.c_int32), ("seed", C.c_uint64),
                ("n_iterations", C.c_int64), ("n_devices", C.c_int64),
                ("n_packs", C.c_int64), ("n_members", C.c_int64),
                ("iter_group", C.POINTER(C.c_int32)),
                ("iter_dev_offsets", C.POINTER(C.c_int64)),
                ("dev_index", C.POINTER(C.c_int32)),
                ("dev_pack_offsets", C.POINTER(C.c_int64)),
                ("pack_capacity", C.POINTER(C.c_int64)),
                ("pack_total", C.POINTER(C.c_int64)),
                ("pack_attention", C.POINTER(C.c_int64)),
                ("pack_member_offsets", C.POINTER(C.c_int64)),
                ("member_id", C.POINTER(C.c_int64)),
                ("member_length", C.POINTER(C.c_int64))]


def available(kind: str) -> bool:
    return os.path.exists(PATHS[kind])


def _arr(p, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(p, shape=(n,)).astype(dtype, copy=True)


class Oracle:
    def __init__(self, kind: str = "restatement"):
        path = PATHS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run make -C oracle)")
        self.kind = kind
        self.lib = C.CDLL(path)
        self.lib.oracle_plan_free.argtypes = [C.POINTER(OraclePlan)]
        self.err = C.create_string_buffer(8192)

    # -- helpers -----------------------------------------------------------
    def _check(self, rc: int) -> None:
        abi.raise_status(rc, self.err.value.decode("utf-8", "backslashreplace"))

    def _take(self, p: C.POINTER(OraclePlan), groups=None, l_best=None) -> abi.FlatPlan:
        o = p.contents
        ni, nd, npk, nm = o.n_iterations, o.n_devices, o.n_packs, o.n_members
        fp = abi.FlatPlan(
            device_count=o.device_count, seed=o.seed,
            groups=list(groups) if groups else [], l_best=l_best or 0,
            iter_group=_arr(o.iter_group, ni, np.int32),
            iter_dev_offsets=_arr(o.iter_dev_offsets, ni + 1, np.int64),
            dev_index=_arr(o.dev_index, nd, np.int32),
            dev_pack_offsets=_arr(o.dev_pack_offsets, nd + 1, np.int64),
            pack_capacity=_arr(o.pack_capacity, npk, np.int64),
            pack_total=_arr(o.pack_total, npk, np.int64),
            pack_attention=_arr(o.pack_attention, npk, np.int64),
            pack_member_offsets=_arr(o.pack_member_offsets, npk + 1, np.int64),
            member_id=_arr(o.member_id, nm, np.int64),
            member_length=_arr(o.member_length, nm, np.int64))
        self.lib.oracle_plan_free(p)
        return fp

    @staticmethod
    def _ids(ids, n):
        if ids is None:
            return None
        return np.ascontiguousarray(ids, dtype=np.int64)

    # -- ABI -----------------------------------------------------------------
    def synth(self, count: int, short_dist: str, long_fraction: float = 0.0,
              long_dist: str = "", max_length: int = 131072, seed: int = 0) -> np.ndarray:
        out = np.zeros(count, dtype=np.int64)
        rc = self.lib.oracle_synth_lengths(C.c_int64(count), short_dist.encode(),
                                           C.c_double(long_fraction), long_dist.encode(),
                                           C.c_int64(max_length), C.c_uint64(seed),
                                           abi.ptr(out, C.c_int64), self.err, len(self.err))
        self._check(rc)
        return out

    def shuffle_positions(self, seed: int, m: int) -> np.ndarray:
        out = np.zeros(max(m, 1), dtype=np.uint32)
        self.lib.oracle_shuffle_positions(C.c_uint64(seed & (2**64 - 1)), C.c_int64(m), abi.ptr(out, C.c_uint32))
        return out[:m]

    def validate(self, ids, lengths) -> None:
        lengths = np.ascontiguousarray(lengths, dtype=np.int64)
        ids = self._ids(ids, len(lengths))
        rc = self.lib.oracle_validate(abi.ptr(ids, C.c_int64), abi.ptr(lengths, C.c_int64),
                                      C.c_int64(len(lengths)), self.err, len(self.err))
        self._check(rc)

    def fingerprint(self, ids, lengths):
        lengths = np.ascontiguousarray(lengths, dtype=np.int64)
        ids = self._ids(ids, len(lengths))
        h, c, t = C.c_uint64(), C.c_int64(), C.c_int64()
        self.lib.oracle_fingerprint(abi.ptr(ids, C.c_int64), abi.ptr(lengths, C.c_int64),
                                    C.c_int64(len(lengths)), C.byref(h), C.byref(c), C.byref(t))
        return h.value, c.value, t.value

    def group_data(self, ids, lengths, groups: Sequence[tuple], l_best=None) -> abi.FlatPlan:
        lengths = np.ascontiguousarray(lengths, dtype=np.int64)
        ids = self._ids(ids, len(lengths))
        g, keep = abi.make_groups(groups, l_best)
        out = C.POINTER(OraclePlan)()
        rc = self.lib.oracle_group_data(abi.ptr(ids, C.c_int64), abi.ptr(lengths, C.c_int64),
                                        C.c_int64(len(lengths)), C.byref(g), C.byref(out),
                                        self.err, len(self.err))
        self._check(rc)
        return self._take(out)

    def pack(self, ids, lengths, capacity: int, strategy: str = "isf", seed: int = 0,
             isf_iterations: int = 8, isf_fill_threshold: float = 0.98) -> abi.FlatPlan:
        lengths = np.ascontiguousarray(lengths, dtype=np.int64)
        ids = self._ids(ids, len(lengths))
        st = abi.Strategy(abi.STRATEGIES[strategy], isf_iterations, isf_fill_threshold)
        out = C.POINTER(OraclePlan)()
        rc = self.lib.oracle_pack(abi.ptr(ids, C.c_int64), abi.ptr(lengths, C.c_int64),
                                  C.c_int64(len(lengths)), C.c_int64(capacity), C.byref(st),
                                  C.c_uint64(seed & (2**64 - 1)), C.byref(out), self.err, len(self.err))
        self._check(rc)
        return self._take(out)

    def _to_oracle(self, fp: abi.FlatPlan):
        keep = []

        def col(a, dt):
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a.ctypes.data_as(C.POINTER(C.c_int64 if dt == np.int64 else C.c_int32))

        o = OraclePlan()
        o.device_count = fp.device_count
        o.seed = fp.seed
        o.n_iterations = len(fp.iter_group)
        o.n_devices = len(fp.dev_index)
        o.n_packs = len(fp.pack_capacity)
        o.n_members = int(fp.pack_member_offsets[-1]) if o.n_packs else 0
        o.iter_group = col(fp.iter_group, np.int32)
        o.iter_dev_offsets = col(fp.iter_dev_offsets, np.int64)
        o.dev_index = col(fp.dev_index, np.int32)
        o.dev_pack_offsets = col(fp.dev_pack_offsets, np.int64)
        o.pack_capacity = col(fp.pack_capacity, np.int64)
        o.pack_total = col(fp.pack_total, np.int64)
        o.pack_attention = col(fp.pack_attention, np.int64)
        o.pack_member_offsets = col(fp.pack_member_offsets, np.int64)
        o.member_id = col(fp.member_id, np.int64)
        o.member_length = col(fp.member_length, np.int64)
        return o, keep

    def greedy_fill(self, packs: abi.FlatPlan, pools: abi.FlatPlan):
        a, ka = self._to_oracle(packs)
        b, kb = self._to_oracle(pools)
        op, oq = C.POINTER(OraclePlan)(), C.POINTER(OraclePlan)()
        rc = self.lib.oracle_greedy_fill(C.byref(a), C.byref(b), C.byref(op), C.byref(oq),
                                         self.err, len(self.err))
        self._check(rc)
        return self._take(op), self._take(oq)

    def balance_batching(self, packs: abi.FlatPlan, device_count: int, group_index: int = 0,
                         sp_comm: bool = False, random: bool = False, seed: int = 0):
        a, ka = self._to_oracle(packs)
        out = C.POINTER(OraclePlan)()
        rc = self.lib.oracle_balance_batching(C.byref(a), C.c_int32(device_count),
                                              C.c_int32(group_index), C.c_int32(int(sp_comm)),
                                              C.c_int32(int(random)), C.c_uint64(seed),
                                              C.byref(out), self.err, len(self.err))
        self._check(rc)
        return self._take(out)

    def build_plan(self, ids, lengths, groups: Sequence[tuple], l_best=None, **opts) -> abi.FlatPlan:
        lengths = np.ascontiguousarray(lengths, dtype=np.int64)
        ids = self._ids(ids, len(lengths))
        g, keep = abi.make_groups(groups, l_best)
        o = abi.make_options(**opts)
        out = C.POINTER(OraclePlan)()
        rc = self.lib.oracle_build_plan(abi.ptr(ids, C.c_int64), abi.ptr(lengths, C.c_int64),
                                        C.c_int64(len(lengths)), C.byref(g), C.byref(o),
                                        C.byref(out), self.err, len(self.err))
        self._check(rc)
        return self._take(out, groups, g.l_best)

    def plan_from_json(self, text: bytes) -> abi.FlatPlan:
        """plan_from_json(text) in the reference (reference kind only); member ids / lengths in the plan."""
        out = C.POINTER(OraclePlan)()
        rc = self.lib.oracle_plan_from_json(C.c_char_p(text), C.c_int64(len(text)), C.byref(out), self.err,
                                            len(self.err))
        self._check(rc)
        return self._take(out)

    def build_plan_json(self, ids, lengths, groups: Sequence[tuple], l_best=None, **opts) -> bytes:
        """The reference's plan_to_json text of its build_plan (reference kind only)."""
        lengths = np.ascontiguousarray(lengths, dtype=np.int64)
        ids = self._ids(ids, len(lengths))
        g, keep = abi.make_groups(groups, l_best)
        o = abi.make_options(**opts)
        out = C.c_void_p()
        n = C.c_int64()
        rc = self.lib.oracle_build_plan_json(abi.ptr(ids, C.c_int64), abi.ptr(lengths, C.c_int64),
                                             C.c_int64(len(lengths)), C.byref(g), C.byref(o),
                                             C.byref(out), C.byref(n), self.err, len(self.err))
        self._check(rc)
        text = C.string_at(out, n.value)
        self.lib.oracle_free_text.argtypes = [C.c_void_p]
        self.lib.oracle_free_text(out)
        return text

    def build_batching_plan_json(self, ids, lengths, group: tuple, device_count: int, mode: str,
                                 seed: int = 0) -> bytes:
        """plan_to_json(build_batching_plan(...)) of the reference (reference kind only)."""
        lengths = np.ascontiguousarray(lengths, dtype=np.int64)
        ids = self._ids(ids, len(lengths))
        out, n = C.c_void_p(), C.c_int64()
        rc = self.lib.oracle_build_batching_plan_json(
            abi.ptr(ids, C.c_int64), abi.ptr(lengths, C.c_int64), C.c_int64(len(lengths)), C.c_int64(group[0]),
            C.c_int32(group[1]), C.c_int32(group[2]), C.c_int32(device_count), C.c_int32(0 if mode == "sorted" else 1),
            C.c_uint64(seed), C.byref(out), C.byref(n), self.err, len(self.err))
        self._check(rc)
        text = C.string_at(out, n.value)
        self.lib.oracle_free_text.argtypes = [C.c_void_p]
        self.lib.oracle_free_text(out)
        return text

    def padded_batching(self, ids, lengths, budget: int, mode: str, seed: int = 0):
        """(order ids, batch offsets, batch max) of sorted_/random_batching (reference kind only)."""
        lengths = np.ascontiguousarray(lengths, dtype=np.int64)
        ids = self._ids(ids, len(lengths))
        n = len(lengths)
        order = np.zeros(max(n, 1), dtype=np.int64)
        off = np.zeros(n + 1, dtype=np.int64)
        mx = np.zeros(max(n, 1), dtype=np.int64)
        nb = C.c_int64()
        rc = self.lib.oracle_padded_batching(abi.ptr(ids, C.c_int64), abi.ptr(lengths, C.c_int64), C.c_int64(n),
                                             C.c_int64(budget), C.c_int32(0 if mode == "sorted" else 1),
                                             C.c_uint64(seed), abi.ptr(order, C.c_int64), abi.ptr(off, C.c_int64),
                                             abi.ptr(mx, C.c_int64), C.byref(nb), self.err, len(self.err))
        self._check(rc)
        b = nb.value
        return order[:n], off[:b + 1], mx[:b]

    def curriculum(self, ids, lengths, groups, l_best, warmup: int, cutoff: int, **opts):
        """(manifest, schedule csv, sp[], ckpt[], switch_count) of curriculum_order(build_plan(...))
        in the reference (reference kind only)."""
        lengths = np.ascontiguousarray(lengths, dtype=np.int64)
        ids = self._ids(ids, len(lengths))
        g, keep = abi.make_groups(groups, l_best)
        o = abi.make_options(**opts)
        j, jn, c, cn = C.c_void_p(), C.c_int64(), C.c_void_p(), C.c_int64()
        cap = len(lengths) + 1
        sp = np.zeros(cap, dtype=np.int32)
        ck = np.zeros(cap, dtype=np.int32)
        sw = C.c_int64()
        rc = self.lib.oracle_curriculum(abi.ptr(ids, C.c_int64), abi.ptr(lengths, C.c_int64), C.c_int64(len(lengths)),
                                        C.byref(g), C.byref(o), C.c_int32(warmup), C.c_int32(cutoff), C.byref(j),
                                        C.byref(jn), C.byref(c), C.byref(cn), abi.ptr(sp, C.c_int32),
                                        abi.ptr(ck, C.c_int32), C.byref(sw), self.err, len(self.err))
        self._check(rc)
        jt, ct = C.string_at(j, jn.value), C.string_at(c, cn.value)
        self.lib.oracle_free_text.argtypes = [C.c_void_p]
        self.lib.oracle_free_text(j)
        self.lib.oracle_free_text(c)
        ni = ct.count(b"\n") - 1
        return jt, ct, sp[:ni], ck[:ni], sw.value

    def load_lengths(self, text: bytes, fmt: str, source: str = "corpus"):
        """(ids, lengths) of load_lengths(istream, format, source) in the reference (reference kind only)."""
        cap = len(text) // 2 + 2
        lens = np.zeros(cap, dtype=np.int64)
        ids = np.zeros(cap, dtype=np.int64)
        n = C.c_int64()
        code = {"jsonl": 0, "csv": 1, "raw-lengths": 2, "raw": 2}[fmt]
        rc = self.lib.oracle_load_lengths(C.c_char_p(text), C.c_int64(len(text)), C.c_int32(code),
                                          source.encode(), abi.ptr(lens, C.c_int64), abi.ptr(ids, C.c_int64),
                                          C.c_int64(cap), C.byref(n), self.err, len(self.err))
        self._check(rc)
        return ids[:n.value], lens[:n.value]

    def report(self, plan: abi.FlatPlan):
        v = plan.view()
        m = abi.Metrics()
        ni = plan.n_iterations
        dbr = np.zeros(max(ni, 1))
        abr_ = np.zeros(max(ni, 1))
        rc = self.lib.oracle_report(C.byref(v), C.byref(m), abi.ptr(dbr, C.c_double),
                                    abi.ptr(abr_, C.c_double), self.err, len(self.err))
        self._check(rc)
        return m, dbr[:ni], abr_[:ni]

    def simulate(self, plan: abi.FlatPlan, profile: Optional[abi.HardwareProfile] = None):
        v = plan.view()
        prof = profile if profile is not None else abi.default_profile()
        st = abi.SimTotals()
        ni, nd = plan.n_iterations, len(plan.dev_index)
        it = np.zeros(max(ni, 1))
        dc, dm, di = (np.zeros(max(nd, 1)) for _ in range(3))
        rc = self.lib.oracle_simulate(C.byref(v), C.byref(prof), C.byref(st), abi.ptr(it, C.c_double),
                                      abi.ptr(dc, C.c_double), abi.ptr(dm, C.c_double),
                                      abi.ptr(di, C.c_double), self.err, len(self.err))
        self._check(rc)
        return st, it[:ni], dc[:nd], dm[:nd], di[:nd]

    def memory_used(self, length, sp, ckpt, profile=None) -> int:
        prof = profile if profile is not None else abi.default_profile()
        out = C.c_int64()
        rc = self.lib.oracle_memory_used(C.c_int64(length), C.c_int32(sp), C.c_int32(ckpt),
                                         C.byref(prof), C.byref(out), self.err, len(self.err))
        self._check(rc)
        return out.value

    def iter_time(self, caps, totals, attns, sp, ckpt, profile=None) -> float:
        prof = profile if profile is not None else abi.default_profile()
        caps, totals, attns = (np.ascontiguousarray(a, dtype=np.int64) for a in (caps, totals, attns))
        out = C.c_double()
        rc = self.lib.oracle_iter_time(abi.ptr(caps, C.c_int64), abi.ptr(totals, C.c_int64),
                                       abi.ptr(attns, C.c_int64), C.c_int64(len(caps)),
                                       C.c_int32(sp), C.c_int32(ckpt), C.byref(prof), C.byref(out),
                                       self.err, len(self.err))
        self._check(rc)
        return out.value

    def profile_time(self, profiler, length, sp, ckpt) -> float:
        out = C.c_double()
        rc = self.lib.oracle_profile_time(C.byref(profiler), C.c_int64(length), C.c_int32(sp),
                                          C.c_int32(ckpt), C.byref(out), self.err, len(self.err))
        self._check(rc)
        return out.value

    def profile_memory(self, profiler, length, sp, ckpt) -> int:
        out = C.c_int64()
        rc = self.lib.oracle_profile_memory(C.byref(profiler), C.c_int64(length), C.c_int32(sp),
                                            C.c_int32(ckpt), C.byref(out), self.err, len(self.err))
        self._check(rc)
        return out.value

    def derive_ckpt(self, profiler, length, sp) -> int:
        out = C.c_int32()
        rc = self.lib.oracle_derive_ckpt(C.byref(profiler), C.c_int64(length), C.c_int32(sp),
                                         C.byref(out), self.err, len(self.err))
        self._check(rc)
        return out.value

    def greedy_profile_ckpt(self, profiler, length, sp, ckpt_min, ckpt_max) -> int:
        out = C.c_int32()
        rc = self.lib.oracle_greedy_profile_ckpt(C.byref(profiler), C.c_int64(length), C.c_int32(sp),
                                                 C.c_int32(ckpt_min), C.c_int32(ckpt_max),
                                                 C.byref(out), self.err, len(self.err))
        self._check(rc)
        return out.value

    def find_best_sp_ckpt(self, profiler, length, sps):
        arr = np.ascontiguousarray(sps, dtype=np.int32)
        sp, ck, sec = C.c_int32(), C.c_int32(), C.c_double()
        rc = self.lib.oracle_find_best_sp_ckpt(C.byref(profiler), C.c_int64(length),
                                               abi.ptr(arr, C.c_int32), C.c_int32(len(arr)),
                                               C.byref(sp), C.byref(ck), C.byref(sec),
                                               self.err, len(self.err))
        self._check(rc)
        return (sp.value, ck.value), sec.value

    def select_groups(self, lengths, profiler, sps):
        ls = np.ascontiguousarray(lengths, dtype=np.int64)
        sp = np.ascontiguousarray(sps, dtype=np.int32)
        out = (abi.GroupConfig * 4)()
        n, lb, lm = C.c_int32(), C.c_int64(), C.c_int64()
        rc = self.lib.oracle_select_groups(abi.ptr(ls, C.c_int64), C.c_int32(len(ls)),
                                           C.byref(profiler), abi.ptr(sp, C.c_int32),
                                           C.c_int32(len(sp)), out, C.byref(n), C.byref(lb),
                                           C.byref(lm), self.err, len(self.err))
        self._check(rc)
        return [(out[i].length, out[i].sp, out[i].ckpt) for i in range(n.value)], lb.value, lm.value

    def sweep(self, ids, lengths, candidates: Sequence[tuple], profile=None, **opts):
        """candidates: [(groups[(l,sp,ck)...], l_best)]."""
        lengths = np.ascontiguousarray(lengths, dtype=np.int64)
        ids = self._ids(ids, len(lengths))
        flat, offs, lbs = [], [0], []
        for groups, lb in candidates:
            flat.extend(groups)
            offs.append(len(flat))
            lbs.append(lb)
        garr = (abi.GroupConfig * len(flat))(*[abi.GroupConfig(*g) for g in flat])
        offs = np.array(offs, dtype=np.int64)
        lbs = np.array(lbs, dtype=np.int64)
        prof = profile if profile is not None else abi.default_profile()
        o = abi.make_options(**opts)
        out = np.zeros(len(candidates))
        best = C.c_int64()
        rc = self.lib.oracle_sweep(abi.ptr(ids, C.c_int64), abi.ptr(lengths, C.c_int64),
                                   C.c_int64(len(lengths)), garr, abi.ptr(offs, C.c_int64),
                                   abi.ptr(lbs, C.c_int64), C.c_int64(len(candidates)),
                                   C.byref(o), C.byref(prof), abi.ptr(out, C.c_double),
                                   C.byref(best), self.err, len(self.err))
        self._check(rc)
        return out, best.value
