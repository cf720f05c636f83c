"""ctypes mirror of include/hbp_b200.h plus numpy helpers.

This is the thin Python side of the C-ABI seam: structs, the library loader
and conversions between numpy arrays and the flat plan layout. The compute
lives in libhbp_b200.so (CUDA, sm_100a); when that library is missing the
loader raises -- there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

# the engine's contexts, side streams and sweep workers are independent
# streams; with the default 8 hardware queues they serialise. Effective when
# set before the process creates its CUDA context (import this first).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhbp_b200.so")
# A/B builds only (tools/): another copy of the library, e.g. variants/<name>/libhbp_b200.so
LIB_PATH = os.environ.get("HBP_LIB_OVERRIDE", LIB_PATH)

HBP_OK, HBP_ERR_VALIDATION, HBP_ERR_INFEASIBLE, HBP_ERR_IO, HBP_ERR_CUDA, HBP_ERR_JSON = 0, 2, 3, 4, 5, 6
STRATEGIES = {"random": 0, "isf": 1, "ffs": 2, "ffd": 3, "bfs": 4, "spfhp": 5}
HBP_MEM_HOST, HBP_MEM_DEVICE = 0, 1


class ValidationError(ValueError):
    """hbp::ValidationError (errors.hpp:17-20) -> ValueError, py_hbp.cpp:49-50."""


class InfeasibleError(RuntimeError):
    """hbp::InfeasibleError (errors.hpp:23-26) -> RuntimeError, py_hbp.cpp:51-52."""


class HbpIoError(OSError):
    """hbp::IoError (errors.hpp:29-32) -> OSError, py_hbp.cpp:53."""


class CudaError(RuntimeError):
    """A CUDA / internal failure of the engine (status 5)."""


class JsonError(RuntimeError):
    """nlohmann::json::exception (a manifest key / type error, status 6): the
    reference's module has no mapping for it, so pybind11 raises RuntimeError."""


def raise_status(code: int, msg: str) -> None:
    if code == HBP_OK:
        return
    if code == HBP_ERR_VALIDATION:
        raise ValidationError(msg)
    if code == HBP_ERR_INFEASIBLE:
        raise InfeasibleError(msg)
    if code == HBP_ERR_IO:
        raise HbpIoError(msg)
    if code == HBP_ERR_JSON:
        raise JsonError(msg)
    raise CudaError(msg)


class GroupConfig(C.Structure):
    _fields_ = [("length", C.c_int64), ("sp", C.c_int32), ("ckpt", C.c_int32)]


class Groups(C.Structure):
    _fields_ = [("groups", C.POINTER(GroupConfig)), ("count", C.c_int32),
                ("l_best", C.c_int64), ("l_max", C.c_int64)]


class Strategy(C.Structure):
    _fields_ = [("kind", C.c_int32), ("isf_iterations", C.c_int32),
                ("isf_fill_threshold", C.c_double)]


class PlanOptions(C.Structure):
    _fields_ = [("strategy", Strategy), ("device_count", C.c_int32),
                ("balance_batching", C.c_int32), ("greedy_fill", C.c_int32),
                ("seed", C.c_uint64)]


class HardwareProfile(C.Structure):
    _fields_ = [("per_token_linear_cost", C.c_double),
                ("per_token2_attention_cost", C.c_double),
                ("sp_comm_cost", C.c_double),
                ("gc_recompute_factor", C.c_double),
                ("fixed_iteration_cost", C.c_double),
                ("layer_count", C.c_int32),
                ("base_memory", C.c_int64),
                ("per_token_activation_memory", C.c_double),
                ("gc_memory_saving_per_layer", C.c_double),
                ("reference_length", C.c_int64),
                ("device_memory", C.c_int64)]


def default_profile() -> HardwareProfile:
    """HardwareProfile{} defaults, costmodel.hpp:32-43."""
    return HardwareProfile(2.5e-4, 1.5e-9, 1.6e-5, 1.0 / 3.0, 0.0, 32, 24 << 30,
                           300000.0, 300000.0 * 0.75 * 4096.0, 4096, 80 << 30)


class Samples(C.Structure):
    _fields_ = [("ids", C.POINTER(C.c_int64)), ("lengths", C.POINTER(C.c_int64)),
                ("n", C.c_int64), ("memory", C.c_int32), ("source", C.c_char_p)]


def make_samples(ids: Optional[np.ndarray], lengths: np.ndarray, source: str = "python"):
    """Host-memory hbp_samples over numpy arrays. Returns (struct, keepalive)."""
    lengths = np.ascontiguousarray(lengths, dtype=np.int64)
    ids = None if ids is None else np.ascontiguousarray(ids, dtype=np.int64)
    src = source.encode()
    s = Samples(ptr(ids, C.c_int64), ptr(lengths, C.c_int64), len(lengths), HBP_MEM_HOST, src)
    return s, (ids, lengths, src)


def device_samples(ids_ptr: int, lengths_ptr: int, n: int, source: str = "device"):
    """hbp_samples over device pointers (e.g. torch tensors' data_ptr())."""
    src = source.encode()
    s = Samples(C.cast(C.c_void_p(ids_ptr), C.POINTER(C.c_int64)) if ids_ptr else C.POINTER(C.c_int64)(),
                C.cast(C.c_void_p(lengths_ptr), C.POINTER(C.c_int64)), n, HBP_MEM_DEVICE, src)
    return s, (src,)


class PlanView(C.Structure):
    _fields_ = [("device_count", C.c_int32), ("seed", C.c_uint64), ("groups", Groups),
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
                ("member_index", C.POINTER(C.c_int32)),
                ("iter_phase", C.POINTER(C.c_int8))]


class Metrics(C.Structure):
    _fields_ = [("dbr", C.c_double), ("pr", C.c_double), ("abr", C.c_double),
                ("cr", C.c_double), ("ave_t", C.c_double)]


class SimTotals(C.Structure):
    _fields_ = [("total_seconds", C.c_double), ("gpu_days", C.c_double),
                ("switch_count", C.c_int32), ("device_count", C.c_int32),
                ("metrics", Metrics)]


class ProfileRow(C.Structure):
    _fields_ = [("length", C.c_int64), ("sp", C.c_int32), ("ckpt", C.c_int32),
                ("memory_bytes", C.c_int64), ("seconds", C.c_double), ("oom", C.c_int32)]


class Profiler(C.Structure):
    _fields_ = [("kind", C.c_int32), ("profile", HardwareProfile),
                ("ckpt_min", C.c_int32), ("ckpt_max", C.c_int32),
                ("rows", C.POINTER(ProfileRow)), ("n_rows", C.c_int64),
                ("device_memory", C.c_int64)]


def analytic_profiler(profile: Optional[HardwareProfile] = None, ckpt_min: int = 0,
                      ckpt_max: int = -1) -> Profiler:
    p = Profiler()
    p.kind = 0
    p.profile = profile if profile is not None else default_profile()
    p.ckpt_min, p.ckpt_max = ckpt_min, ckpt_max
    p.device_memory = 80 << 30
    return p


def table_profiler(rows: Sequence[tuple], device_memory: int = 80 << 30) -> Profiler:
    """rows: (length, sp, ckpt, memory_bytes | None for oom, seconds)."""
    arr = (ProfileRow * max(1, len(rows)))()
    for i, (l, sp, ck, mem, sec) in enumerate(rows):
        arr[i] = ProfileRow(l, sp, ck, 0 if mem is None else mem, sec, 1 if mem is None else 0)
    p = Profiler()
    p.kind = 1
    p.profile = default_profile()
    p.rows = arr
    p.n_rows = len(rows)
    p.device_memory = device_memory
    p._keep = arr  # keep the row array alive with the struct
    return p


def parse_table_csv(text: str) -> list:
    """TableProfiler::from_csv row format (costmodel.cpp:144-209)."""
    rows, header = [], False
    for line in text.splitlines():
        if not line.strip(" \t\r") or line[0] == "#":
            continue
        cells = [c.strip(" \t\r") for c in line.split(",")]
        if not header and cells and cells[0] == "length":
            header = True
            continue
        mem = None if cells[3] == "oom" else int(cells[3])
        rows.append((int(cells[0]), int(cells[1]), int(cells[2]), mem,
                     0.0 if mem is None else float(cells[4])))
    return rows


def make_groups(groups: Sequence[tuple], l_best: Optional[int] = None):
    """groups: [(length, sp, ckpt), ...] ascending. Returns (Groups, keepalive)."""
    arr = (GroupConfig * len(groups))(*[GroupConfig(l, s, c) for (l, s, c) in groups])
    g = Groups(arr, len(groups), groups[0][0] if l_best is None else l_best, groups[-1][0])
    return g, arr


def make_options(strategy: str = "isf", device_count: int = 4, seed: int = 0,
                 balance_batching: bool = True, greedy_fill: bool = True,
                 isf_iterations: int = 8, isf_fill_threshold: float = 0.98) -> PlanOptions:
    return PlanOptions(Strategy(STRATEGIES[strategy], isf_iterations, isf_fill_threshold),
                       device_count, int(bool(balance_batching)), int(bool(greedy_fill)),
                       C.c_uint64(seed & ((1 << 64) - 1)).value)


def ptr(a: Optional[np.ndarray], ctype):
    if a is None:
        return C.POINTER(ctype)()
    return a.ctypes.data_as(C.POINTER(ctype))


@dataclass
class FlatPlan:
    """A plan in the flat CSR layout of hbp_plan_view (numpy arrays)."""
    device_count: int
    seed: int
    groups: list  # [(length, sp, ckpt)]
    l_best: int
    iter_group: np.ndarray
    iter_dev_offsets: np.ndarray
    dev_index: np.ndarray
    dev_pack_offsets: np.ndarray
    pack_capacity: np.ndarray
    pack_total: np.ndarray
    pack_attention: np.ndarray
    pack_member_offsets: np.ndarray
    member_index: Optional[np.ndarray] = None   # product plans: index into input
    member_id: Optional[np.ndarray] = None      # oracle plans: sample ids
    member_length: Optional[np.ndarray] = None
    _keep: list = field(default_factory=list, repr=False)

    @property
    def n_iterations(self) -> int:
        return int(self.iter_group.shape[0])

    def view(self) -> PlanView:
        g, arr = make_groups(self.groups, self.l_best)
        cols = {k: np.ascontiguousarray(getattr(self, k)) for k in (
            "iter_group", "iter_dev_offsets", "dev_index", "dev_pack_offsets",
            "pack_capacity", "pack_total", "pack_attention", "pack_member_offsets")}
        cols["iter_group"] = cols["iter_group"].astype(np.int32, copy=False)
        cols["dev_index"] = cols["dev_index"].astype(np.int32, copy=False)
        for k in cols:
            if k not in ("iter_group", "dev_index"):
                cols[k] = cols[k].astype(np.int64, copy=False)
        mi = None if self.member_index is None else np.ascontiguousarray(self.member_index, dtype=np.int32)
        v = PlanView()
        v.device_count = self.device_count
        v.seed = C.c_uint64(self.seed & ((1 << 64) - 1)).value
        v.groups = g
        v.n_iterations = cols["iter_group"].shape[0]
        v.n_devices = cols["dev_index"].shape[0]
        v.n_packs = cols["pack_capacity"].shape[0]
        v.n_members = int(cols["pack_member_offsets"][-1]) if v.n_packs else 0
        v.iter_group = ptr(cols["iter_group"], C.c_int32)
        v.iter_dev_offsets = ptr(cols["iter_dev_offsets"], C.c_int64)
        v.dev_index = ptr(cols["dev_index"], C.c_int32)
        v.dev_pack_offsets = ptr(cols["dev_pack_offsets"], C.c_int64)
        v.pack_capacity = ptr(cols["pack_capacity"], C.c_int64)
        v.pack_total = ptr(cols["pack_total"], C.c_int64)
        v.pack_attention = ptr(cols["pack_attention"], C.c_int64)
        v.pack_member_offsets = ptr(cols["pack_member_offsets"], C.c_int64)
        v.member_index = ptr(mi, C.c_int32)
        v._keep = (arr, cols, mi)
        return v

    def members_as_ids(self, ids: Optional[np.ndarray]) -> np.ndarray:
        if self.member_id is not None:
            return self.member_id
        idx = self.member_index.astype(np.int64)
        return idx if ids is None else ids[idx]


# ---------------------------------------------------------------------------
# engine library
# ---------------------------------------------------------------------------

_LIB = None


def load_library() -> C.CDLL:
    """Loads libhbp_b200.so (built in-tree). Raises when it is missing:
    there is no CPU implementation to fall back to."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing; build it with __graft_entry__.build()")
        lib = C.CDLL(LIB_PATH)
        lib.hbp_last_error.restype = C.c_char_p
        lib.hbp_last_error.argtypes = [C.c_void_p]
        lib.hbp_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        lib.hbp_ctx_destroy.argtypes = [C.c_void_p]
        lib.hbp_ctx_launch_count.restype = C.c_int64
        lib.hbp_ctx_launch_count.argtypes = [C.c_void_p]
        lib.hbp_ctx_stream.restype = C.c_void_p
        lib.hbp_ctx_stream.argtypes = [C.c_void_p]
        _LIB = lib
    return _LIB


class Context:
    """One engine context (one CUDA stream) on `device`."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        rc = self.lib.hbp_ctx_create(device, C.byref(h))
        if rc != HBP_OK:
            raise CudaError(f"hbp_ctx_create({device}) failed with status {rc}")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.hbp_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc: int) -> None:
        if rc != HBP_OK:
            raise_status(rc, self.lib.hbp_last_error(self.h).decode("utf-8", "backslashreplace"))

    @property
    def launches(self) -> int:
        return int(self.lib.hbp_ctx_launch_count(self.h))

    def synchronize(self) -> None:
        self.check(self.lib.hbp_ctx_synchronize(self.h))

    # -- hot path (include/hbp_b200.h) -------------------------------------
    def validate(self, ids, lengths, source: str = "python") -> None:
        s, keep = make_samples(ids, lengths, source)
        self.check(self.lib.hbp_validate(self.h, C.byref(s)))

    def group_data(self, ids, lengths, groups, l_best=None):
        s, keep = make_samples(ids, lengths)
        g, garr = make_groups(groups, l_best)
        off = np.zeros(len(groups) + 1, dtype=np.int64)
        mem = np.zeros(max(1, len(keep[1])), dtype=np.int32)
        self.check(self.lib.hbp_group_data(self.h, C.byref(s), C.byref(g), ptr(off, C.c_int64),
                                           ptr(mem, C.c_int32)))
        return off, mem[:len(keep[1])]

    def _plan(self, handle, groups, l_best) -> "DevicePlanHandle":
        return DevicePlanHandle(self, handle, groups, l_best)

    def pack(self, ids, lengths, capacity: int, strategy: str = "isf", seed: int = 0,
             isf_iterations: int = 8, isf_fill_threshold: float = 0.98) -> "DevicePlanHandle":
        s, keep = make_samples(ids, lengths)
        st = Strategy(STRATEGIES[strategy], isf_iterations, isf_fill_threshold)
        h = C.c_void_p()
        self.check(self.lib.hbp_pack(self.h, C.byref(s), C.c_int64(capacity), C.byref(st),
                                     C.c_uint64(seed & (2**64 - 1)), C.byref(h)))
        return self._plan(h, [], 0)

    def build_plan(self, ids, lengths, groups, l_best=None, source: str = "python", **opts) -> "DevicePlanHandle":
        s, keep = make_samples(ids, lengths, source)
        return self.build_plan_samples(s, groups, l_best, **opts)

    def build_batching_plan(self, ids, lengths, group: tuple, device_count: int = 4, mode: str = "sorted",
                            seed: int = 0) -> "DevicePlanHandle":
        """hbp::build_batching_plan (balance.cpp:260-298) on the GPU."""
        s, keep = make_samples(ids, lengths, "python")
        h = C.c_void_p()
        self.lib.hbp_build_batching_plan.argtypes = [C.c_void_p, C.POINTER(Samples), GroupConfig, C.c_int32,
                                                     C.c_int32, C.c_uint64, C.POINTER(C.c_void_p)]
        self.check(self.lib.hbp_build_batching_plan(self.h, C.byref(s), GroupConfig(*group), C.c_int32(device_count),
                                                    C.c_int32(0 if mode == "sorted" else 1),
                                                    C.c_uint64(seed & (2**64 - 1)), C.byref(h)))
        return self._plan(h, [group], group[0])

    CORPUS_FORMATS = {"jsonl": 0, "csv": 1, "raw-lengths": 2, "raw": 2}

    def load_lengths(self, text: bytes, fmt: str, source: str = "corpus", device_out=None, with_ids=False):
        """hbp::load_lengths(istream, format, source) on the GPU (jsonl, csv,
        raw-lengths): the lengths as int64 numpy ((ids, lengths) with
        with_ids), or written into the torch int64 CUDA tensor `device_out`
        (returns the count)."""
        if fmt not in self.CORPUS_FORMATS:
            raise ValidationError("unknown corpus format: " + fmt)
        cap = len(text) // 2 + 1 if device_out is None else device_out.numel()
        n = C.c_int64()
        self.lib.hbp_load_lengths.argtypes = [C.c_void_p, C.c_char_p, C.c_int64, C.c_int32, C.c_char_p, C.c_void_p,
                                              C.c_void_p, C.c_int64, C.c_int32, C.POINTER(C.c_int64)]
        ids = None
        if device_out is None:
            out = np.empty(max(cap, 1), dtype=np.int64)  # written up to the count; no fill
            dst, mem = out.ctypes.data, 0
            if with_ids:
                ids = np.empty(max(cap, 1), dtype=np.int64)
        else:
            dst, mem = device_out.data_ptr(), 1
        self.check(self.lib.hbp_load_lengths(self.h, text, C.c_int64(len(text)), C.c_int32(self.CORPUS_FORMATS[fmt]),
                                             source.encode(), C.c_void_p(ids.ctypes.data if ids is not None else None),
                                             C.c_void_p(dst), C.c_int64(cap), C.c_int32(mem), C.byref(n)))
        if device_out is not None:
            return n.value
        return (ids[:n.value], out[:n.value]) if with_ids else out[:n.value]

    def padded_batching(self, ids, lengths, token_budget: int, mode: str = "sorted", seed: int = 0):
        """hbp::sorted_batching / random_batching on the GPU: (order as input
        indices, batch offsets into order, batch max lengths)."""
        s, keep = make_samples(ids, lengths, "python")
        n = len(lengths)
        order = np.zeros(max(n, 1), dtype=np.int32)
        off = np.zeros(n + 1, dtype=np.int64)
        mx = np.zeros(max(n, 1), dtype=np.int64)
        nb = C.c_int64()
        self.lib.hbp_padded_batching.argtypes = [C.c_void_p, C.POINTER(Samples), C.c_int64, C.c_int32, C.c_uint64,
                                                 C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                                 C.POINTER(C.c_int64)]
        self.check(self.lib.hbp_padded_batching(self.h, C.byref(s), C.c_int64(token_budget),
                                                C.c_int32(0 if mode == "sorted" else 1), C.c_uint64(seed & (2**64 - 1)),
                                                ptr(order, C.c_int32), ptr(off, C.c_int64), ptr(mx, C.c_int64),
                                                C.byref(nb)))
        b = nb.value
        return order[:n], off[:b + 1], mx[:b]

    def plan_from_json(self, text: bytes):
        """hbp::plan_from_json on the GPU: (DevicePlanHandle, ids, lengths) --
        the plan's member_index indexes the manifest's samples (ids, lengths)."""
        self.lib.hbp_plan_from_json.argtypes = [C.c_void_p, C.c_char_p, C.c_int64, C.POINTER(C.c_void_p),
                                                C.POINTER(C.c_int64)]
        self.lib.hbp_plan_members.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        h = C.c_void_p()
        m = C.c_int64()
        self.check(self.lib.hbp_plan_from_json(self.h, text, C.c_int64(len(text)), C.byref(h), C.byref(m)))
        v = PlanView()
        self.check(self.lib.hbp_plan_view_get(self.h, h, C.byref(v)))
        groups = [(v.groups.groups[k].length, v.groups.groups[k].sp, v.groups.groups[k].ckpt)
                  for k in range(v.groups.count)]
        plan = self._plan(h, groups, v.groups.l_best)
        ids = np.zeros(max(m.value, 1), dtype=np.int64)
        lens = np.zeros(max(m.value, 1), dtype=np.int64)
        self.check(self.lib.hbp_plan_members(self.h, h, C.c_void_p(ids.ctypes.data), C.c_void_p(lens.ctypes.data)))
        return plan, ids[:m.value], lens[:m.value]

    def build_plan_samples(self, s: Samples, groups, l_best=None, **opts) -> "DevicePlanHandle":
        g, garr = make_groups(groups, l_best)
        o = make_options(**opts)
        h = C.c_void_p()
        self.check(self.lib.hbp_build_plan(self.h, C.byref(s), C.byref(g), C.byref(o), C.byref(h)))
        return self._plan(h, groups, g.l_best)

    def report(self, plan: FlatPlan):
        v = plan.view()
        m = Metrics()
        ni = plan.n_iterations
        dbr = np.zeros(max(ni, 1))
        abr_ = np.zeros(max(ni, 1))
        self.check(self.lib.hbp_report(self.h, C.byref(v), C.byref(m), ptr(dbr, C.c_double),
                                       ptr(abr_, C.c_double)))
        return m, dbr[:ni], abr_[:ni]

    def simulate(self, plan: FlatPlan, profile: Optional[HardwareProfile] = None):
        v = plan.view()
        prof = profile if profile is not None else default_profile()
        st = SimTotals()
        ni, nd = plan.n_iterations, len(plan.dev_index)
        it = np.zeros(max(ni, 1))
        dc, dm, di = (np.zeros(max(nd, 1)) for _ in range(3))
        self.check(self.lib.hbp_simulate(self.h, C.byref(v), C.byref(prof), C.byref(st), ptr(it, C.c_double),
                                         ptr(dc, C.c_double), ptr(dm, C.c_double), ptr(di, C.c_double)))
        return st, it[:ni], dc[:nd], dm[:nd], di[:nd]

    def memory_used(self, length, sp, ckpt, profile=None) -> int:
        prof = profile if profile is not None else default_profile()
        out = C.c_int64()
        self.check(self.lib.hbp_memory_used(self.h, C.c_int64(length), C.c_int32(sp), C.c_int32(ckpt),
                                            C.byref(prof), C.byref(out)))
        return out.value

    # -- cost model / auto-selection -----------------------------------------
    def profile_time(self, profiler: Profiler, length, sp, ckpt) -> float:
        out = C.c_double()
        self.check(self.lib.hbp_profiler_time(self.h, C.byref(profiler), C.c_int64(length), C.c_int32(sp),
                                              C.c_int32(ckpt), C.byref(out)))
        return out.value

    def profile_memory(self, profiler: Profiler, length, sp, ckpt) -> int:
        out = C.c_int64()
        self.check(self.lib.hbp_profiler_memory(self.h, C.byref(profiler), C.c_int64(length), C.c_int32(sp),
                                                C.c_int32(ckpt), C.byref(out)))
        return out.value

    def derive_ckpt(self, profiler: Profiler, length, sp) -> int:
        out = C.c_int32()
        self.check(self.lib.hbp_profiler_derive_ckpt(self.h, C.byref(profiler), C.c_int64(length), C.c_int32(sp),
                                                     C.byref(out)))
        return out.value

    def greedy_profile_ckpt(self, profiler: Profiler, length, sp, ckpt_min, ckpt_max) -> int:
        out = C.c_int32()
        self.check(self.lib.hbp_greedy_profile_ckpt(self.h, C.byref(profiler), C.c_int64(length), C.c_int32(sp),
                                                    C.c_int32(ckpt_min), C.c_int32(ckpt_max), C.byref(out)))
        return out.value

    def find_best_sp_ckpt(self, profiler: Profiler, length, sps):
        arr = np.ascontiguousarray(sps, dtype=np.int32)
        sp, ck, sec = C.c_int32(), C.c_int32(), C.c_double()
        self.check(self.lib.hbp_find_best_sp_ckpt(self.h, C.byref(profiler), C.c_int64(length),
                                                  ptr(arr, C.c_int32), C.c_int32(len(arr)), C.byref(sp),
                                                  C.byref(ck), C.byref(sec)))
        return (sp.value, ck.value), sec.value

    def select_groups(self, lengths, profiler: Profiler, sps):
        ls = np.ascontiguousarray(lengths, dtype=np.int64)
        sp = np.ascontiguousarray(sps, dtype=np.int32)
        out = (GroupConfig * 4)()
        n, lb, lm = C.c_int32(), C.c_int64(), C.c_int64()
        self.check(self.lib.hbp_select_groups(self.h, ptr(ls, C.c_int64), C.c_int32(len(ls)), C.byref(profiler),
                                              ptr(sp, C.c_int32), C.c_int32(len(sp)), out, C.byref(n),
                                              C.byref(lb), C.byref(lm)))
        return [(out[i].length, out[i].sp, out[i].ckpt) for i in range(n.value)], lb.value, lm.value

    def sweep(self, ids, lengths, candidates, profile: Optional[HardwareProfile] = None, **opts):
        """candidates: [(groups[(l, sp, ckpt)...], l_best)] -> (seconds[], best index)."""
        s, keep = make_samples(ids, lengths)
        return self.sweep_samples(s, candidates, profile, **opts)

    def sweep_samples(self, s: Samples, candidates, profile: Optional[HardwareProfile] = None, **opts):
        garr, offs, lbs = flatten_candidates(candidates)
        prof = profile if profile is not None else default_profile()
        o = make_options(**opts)
        out = np.zeros(max(1, len(candidates)))
        best = C.c_int64()
        self.check(self.lib.hbp_sweep(self.h, C.byref(s), garr, ptr(offs, C.c_int64), ptr(lbs, C.c_int64),
                                      C.c_int64(len(candidates)), C.byref(o), C.byref(prof),
                                      ptr(out, C.c_double), C.byref(best)))
        return out[:len(candidates)], best.value

    def greedy_fill(self, pack_offsets, pack_capacity, ids, lengths, pool_offsets, pool_ids, pool_lengths):
        """hbp_greedy_fill (balance.cpp:46-101): per pack, in pick order, the
        flattened pool indices it takes; and which pool samples stay."""
        class PacksIn(C.Structure):
            _fields_ = [("n_packs", C.c_int64), ("pack_offsets", C.c_void_p), ("pack_capacity", C.c_void_p),
                        ("ids", C.c_void_p), ("lengths", C.c_void_p)]
        po, pc = (np.ascontiguousarray(x, dtype=np.int64) for x in (pack_offsets, pack_capacity))
        pi, pl = (np.ascontiguousarray(x, dtype=np.int64) for x in (ids, lengths))
        qo, qi, ql = (np.ascontiguousarray(x, dtype=np.int64) for x in (pool_offsets, pool_ids, pool_lengths))
        packs = PacksIn(len(pc), po.ctypes.data, pc.ctypes.data, pi.ctypes.data, pl.ctypes.data)
        m = int(qo[-1]) if len(qo) else 0
        off = np.zeros(len(pc) + 1, np.int64)
        added = np.zeros(max(m, 1), np.int64)
        keep = np.zeros(max(m, 1), np.uint8)
        self.lib.hbp_greedy_fill.argtypes = [C.c_void_p, C.POINTER(PacksIn), C.c_int32, C.c_void_p, C.c_void_p,
                                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        self.check(self.lib.hbp_greedy_fill(self.h, C.byref(packs), len(qo) - 1, qo.ctypes.data, qi.ctypes.data,
                                            ql.ctypes.data, off.ctypes.data, added.ctypes.data, keep.ctypes.data))
        return off, added[:off[-1]], keep[:m].astype(bool)

    # -- stage hooks (include/hbp_b200_testing.h) --------------------------
    def shuffle_positions(self, seed: int, m: int) -> np.ndarray:
        out = np.zeros(max(m, 1), dtype=np.uint32)
        self.check(self.lib.hbp_test_shuffle_positions(self.h, C.c_uint64(seed & (2**64 - 1)),
                                                       C.c_int64(m), ptr(out, C.c_uint32)))
        return out[:m]

    def scan_u32(self, a: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint32)
        out = np.zeros(max(len(a), 1), dtype=np.uint64)
        self.check(self.lib.hbp_test_scan_u32(self.h, ptr(a, C.c_uint32), C.c_int64(len(a)),
                                              ptr(out, C.c_uint64)))
        return out[:len(a)]

    def radix_sort(self, keys: np.ndarray, values: np.ndarray, bits: int, descending: bool = False):
        k = np.ascontiguousarray(keys, dtype=np.uint32).copy()
        v = np.ascontiguousarray(values, dtype=np.uint32).copy()
        self.check(self.lib.hbp_test_radix_sort(self.h, ptr(k, C.c_uint32), ptr(v, C.c_uint32),
                                                C.c_int64(len(k)), C.c_int32(bits), C.c_int32(int(descending))))
        return k, v


def flatten_candidates(candidates):
    """[(groups[(l, sp, ck)...], l_best)] -> (GroupConfig array, offsets, l_best) of the C-ABI."""
    flat, offs, lbs = [], [0], []
    for groups, lb in candidates:
        flat.extend(groups)
        offs.append(len(flat))
        lbs.append(lb)
    garr = (GroupConfig * max(1, len(flat)))(*[GroupConfig(*g) for g in flat])
    return garr, np.array(offs, dtype=np.int64), np.array(lbs, dtype=np.int64)


COMM_ID_BYTES = 128


class Comm:
    """The engine's NCCL communicator (hbp_comm_*, include/hbp_b200.h): the
    multi-GPU sweep and the DP-column sharded report/simulate run their
    exchanges as NCCL collectives on the context's stream, in C++."""

    def __init__(self, ctx: "Context", uid: bytes, rank: int, world: int):
        lib = ctx.lib
        lib.hbp_comm_create.argtypes = [C.c_void_p, C.c_char_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]
        lib.hbp_comm_destroy.argtypes = [C.c_void_p]
        self.ctx, self.rank, self.world = ctx, rank, world
        h = C.c_void_p()
        ctx.check(lib.hbp_comm_create(ctx.h, uid, rank, world, C.byref(h)))
        self.h = h

    @staticmethod
    def unique_id(ctx: "Context") -> bytes:
        buf = C.create_string_buffer(COMM_ID_BYTES)
        ctx.lib.hbp_comm_unique_id.argtypes = [C.c_void_p, C.c_char_p]
        ctx.check(ctx.lib.hbp_comm_unique_id(ctx.h, buf))
        return buf.raw

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.hbp_comm_destroy(self.h)
            self.h = None

    def sweep(self, s: Samples, candidates, profile: Optional[HardwareProfile] = None, **opts):
        """(seconds[n] on every rank, global argmin, candidates evaluated here)."""
        lib = self.ctx.lib
        garr, offs, lbs = flatten_candidates(candidates)
        prof = profile if profile is not None else default_profile()
        o = make_options(**opts)
        out = np.zeros(max(1, len(candidates)))
        best, local = C.c_int64(), C.c_int64()
        lib.hbp_sweep_sharded.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64),
                                          C.POINTER(C.c_int64)]
        self.ctx.check(lib.hbp_sweep_sharded(self.ctx.h, self.h, C.byref(s), garr, offs.ctypes.data,
                                             lbs.ctypes.data, len(candidates), C.byref(o), C.byref(prof),
                                             out.ctypes.data, C.byref(best), C.byref(local)))
        return out[:len(candidates)], best.value, local.value

    def evaluate(self, plan: "DevicePlanHandle", profile: Optional[HardwareProfile] = None):
        """(Metrics, SimTotals or None): report / simulate by DP column."""
        lib = self.ctx.lib
        lib.hbp_eval_sharded.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        m, st = Metrics(), SimTotals()
        self.ctx.check(lib.hbp_eval_sharded(self.ctx.h, self.h, plan.h,
                                            C.byref(profile) if profile is not None else None, C.byref(m),
                                            C.byref(st)))
        return m, (st if profile is not None else None)


class DevicePlanHandle:
    """A plan resident in HBM (hbp_plan*). `.flat()` copies it to host."""

    def __init__(self, ctx: Context, handle: C.c_void_p, groups, l_best):
        self.ctx, self.h, self.groups, self.l_best = ctx, handle, list(groups), l_best

    def __del__(self):
        try:
            if self.h:
                self.ctx.lib.hbp_plan_free(self.h)
                self.h = None
        except Exception:
            pass

    def flat(self) -> FlatPlan:
        v = PlanView()
        self.ctx.check(self.ctx.lib.hbp_plan_view_get(self.ctx.h, self.h, C.byref(v)))

        def arr(p, n, dt):
            if n == 0:
                return np.zeros(0, dtype=dt)
            return np.ctypeslib.as_array(p, shape=(n,)).astype(dt, copy=True)

        ni, nd, npk, nm = v.n_iterations, v.n_devices, v.n_packs, v.n_members
        return FlatPlan(device_count=v.device_count, seed=v.seed, groups=self.groups, l_best=self.l_best,
                        iter_group=arr(v.iter_group, ni, np.int32),
                        iter_dev_offsets=arr(v.iter_dev_offsets, ni + 1, np.int64),
                        dev_index=arr(v.dev_index, nd, np.int32),
                        dev_pack_offsets=arr(v.dev_pack_offsets, nd + 1, np.int64),
                        pack_capacity=arr(v.pack_capacity, npk, np.int64),
                        pack_total=arr(v.pack_total, npk, np.int64),
                        pack_attention=arr(v.pack_attention, npk, np.int64),
                        pack_member_offsets=arr(v.pack_member_offsets, npk + 1, np.int64),
                        member_index=arr(v.member_index, nm, np.int32))

    def to_json(self, ids: Optional[np.ndarray], lengths: np.ndarray) -> bytes:
        """hbp::plan_to_json of this plan (src/io.cpp:85-110), written on the GPU;
        ids / lengths: the corpus the plan was built from (host arrays)."""
        s, keep = make_samples(ids, lengths, "json")
        n = C.c_int64()
        lib = self.ctx.lib
        lib.hbp_plan_to_json.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(Samples), C.c_char_p, C.c_int64,
                                         C.POINTER(C.c_int64)]
        self.ctx.check(lib.hbp_plan_to_json(self.ctx.h, self.h, C.byref(s), None, 0, C.byref(n)))
        buf = np.empty(max(1, n.value), dtype=np.uint8)  # no zero fill
        self.ctx.check(lib.hbp_plan_to_json(self.ctx.h, self.h, C.byref(s), buf.ctypes.data_as(C.c_char_p), n.value,
                                            C.byref(n)))
        return buf[:n.value].tobytes()

    def curriculum_order(self, warmup_iterations: int = 500, short_group_cutoff: int = 1) -> "DevicePlanHandle":
        """hbp::curriculum_order (schedule.cpp:10-63) on the GPU: a new device plan."""
        lib = self.ctx.lib
        h = C.c_void_p()
        lib.hbp_curriculum_order.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]
        self.ctx.check(lib.hbp_curriculum_order(self.ctx.h, self.h, warmup_iterations, short_group_cutoff,
                                                C.byref(h)))
        return DevicePlanHandle(self.ctx, h, self.groups, self.l_best)

    def assign_runtime(self):
        """hbp::assign_runtime: (sp[], ckpt[], switch_count)."""
        lib = self.ctx.lib
        n = self.flat().iter_group.shape[0]
        sp = np.zeros(max(n, 1), dtype=np.int32)
        ck = np.zeros(max(n, 1), dtype=np.int32)
        sw = C.c_int64()
        lib.hbp_assign_runtime.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                           C.POINTER(C.c_int64)]
        self.ctx.check(lib.hbp_assign_runtime(self.ctx.h, self.h, ptr(sp, C.c_int32), ptr(ck, C.c_int32),
                                              C.byref(sw)))
        return sp[:n], ck[:n], sw.value

    def schedule_csv(self) -> bytes:
        """hbp::write_schedule_csv text, written on the GPU."""
        lib = self.ctx.lib
        n = C.c_int64()
        lib.hbp_schedule_csv.argtypes = [C.c_void_p, C.c_void_p, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)]
        self.ctx.check(lib.hbp_schedule_csv(self.ctx.h, self.h, None, 0, C.byref(n)))
        buf = np.empty(max(1, n.value), dtype=np.uint8)
        self.ctx.check(lib.hbp_schedule_csv(self.ctx.h, self.h, buf.ctypes.data_as(C.c_char_p), n.value,
                                            C.byref(n)))
        return buf[:n.value].tobytes()

    def report(self):
        m = Metrics()
        self.ctx.check(self.ctx.lib.hbp_report_plan(self.ctx.h, self.h, C.byref(m), C.POINTER(C.c_double)(),
                                                    C.POINTER(C.c_double)()))
        return m

    def simulate(self, profile: Optional[HardwareProfile] = None) -> SimTotals:
        prof = profile if profile is not None else default_profile()
        st = SimTotals()
        self.ctx.check(self.ctx.lib.hbp_simulate_plan(self.ctx.h, self.h, C.byref(prof), C.byref(st),
                                                      C.POINTER(C.c_double)()))
        return st
