#!/usr/bin/env python3
"""Benchmark of the B200 HBP batch-construction engine (BASELINE.json).

One step = one pass of the hot path over one synthetic corpus of the C2
shape (LongAlign-like long tail, 10M samples, groups [16K sp1 ckpt28,
128K sp8 ckpt28], 8 data-parallel devices, seed 1): build_plan + report
(ABR/CR) + simulate (estimated step time) -- the reference's C2 call chain
(SURVEY.md §8(d)).

  value  samples/s with the corpus already in HBM (C-ABI device input)
  e2e    samples/s through the C-ABI with HOST buffers: H2D of the lengths
         and D2H of the whole plan CSR inside every timed step

Packing one corpus does not shard: with --gpus N every
rank packs its own corpus (replicas, weak scaling) and value is the sum.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import os

# Independent streams (plans in flight, the sweep's worker contexts, their
# side streams) need their own hardware work queues: with the default 8 they
# share queues and serialise (C3 sweep 3.6K -> 6K candidates/s with 32). Read
# when the process creates its CUDA context, so before torch touches CUDA.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C2 = dict(count=10_000_000, short="lognormal:7.2:0.7", long_fraction=0.02, long="uniform:16385:131072",
          max_length=131072, seed=20250515)
C2_GROUPS = [(16384, 1, 28), (131072, 8, 28)]
DEVICES, PLAN_SEED = 8, 1
METRIC = "samples packed/sec"
UNIT = "samples/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    # The per-reason fields (clocks_event_reasons.hw_slowdown, ...) stall the
    # driver for 10-40 ms per sample (measured: they land inside timed steps);
    # the `active` bitmask carries the same reasons and does not.
    Q = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active"
    BITS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
            0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 5:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
                mask = int(f[4], 16)
            except ValueError:
                continue
            for bit, name in self.BITS.items():
                if mask & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def synth(abi_lib, spec, count=None):
    n = spec["count"] if count is None else count
    out = np.zeros(n, dtype=np.int64)
    err = C.create_string_buffer(256)
    rc = abi_lib.hbp_synth_lengths(C.c_int64(n), spec["short"].encode(), C.c_double(spec["long_fraction"]),
                                   spec["long"].encode(), C.c_int64(spec["max_length"]), C.c_uint64(spec["seed"]),
                                   out.ctypes.data_as(C.POINTER(C.c_int64)), err, 256)
    if rc != 0:
        raise RuntimeError(err.value.decode())
    return out


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation (oracle/_ref)
# ---------------------------------------------------------------------------

REF_BENCH = os.path.join(ROOT, "oracle", "_ref", "ref_bench")


def c2_synth_arg(spec):
    """The reference's synth spec text (ingest.cpp:331-373) for `spec`."""
    s = f"count={spec['count']},short={spec['short']},max={spec['max_length']}"
    if spec["long_fraction"] > 0:
        s += f",long_fraction={spec['long_fraction']},long={spec['long']}"
    return s


def ref_bench_cmd(spec, groups, l_best, profile=None):
    cmd = [REF_BENCH, "--synth", c2_synth_arg(spec), "--seed", str(spec["seed"]),
           "--groups", ",".join(f"{l}:{sp}:{ck}" for l, sp, ck in groups), "--l-best", str(l_best),
           "--devices", str(DEVICES), "--plan-seed", str(PLAN_SEED)]
    if profile:
        cmd += ["--profile", profile]
    return cmd


def _pin(core):
    return lambda: os.sched_setaffinity(0, {core})


def ref_run_concurrent(cmd, cores):
    """One reference step per listed core, all at once (the reference is
    single-threaded); returns each process's JSON line."""
    procs = [subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, preexec_fn=_pin(c))
             for c in cores]
    out = []
    for p in procs:
        o, e = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"ref_bench rc={p.returncode}: {e.strip()[-300:]}")
        out.append(json.loads(o.strip().splitlines()[-1]))
    return out


def run_reference(args, rank, world):
    """The reference's build_plan + report + simulate (oracle/_ref/ref_bench:
    proj/src compiled in place, its own synth_lengths for the corpus) on the
    SAME config as our arm: the full C2 corpus, one step per host core, all
    concurrently. Never imports this repo's package or loads its engine."""
    if rank != 0:
        return 0
    cores = sorted(os.sched_getaffinity(0))
    try:
        import psutil
        avail_gb = psutil.virtual_memory().available / 2**30
    except Exception:
        avail_gb = 64.0
    # peak RSS of one 10M C2 reference step is ~1.7 GB
    k = max(1, min(args.steps, len(cores), int(avail_gb // 2.5)))
    spec = dict(C2)
    if args.n:
        spec["count"] = args.n
    line = {"impl": "reference", "metric": METRIC, "unit": UNIT, "n_gpus": args.gpus, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": DATA, "config": bench_config(spec)}
    if not os.path.exists(REF_BENCH):
        line["unavailable"] = f"{REF_BENCH} not built (make -C oracle needs /root/reference)"
        print(json.dumps(line), flush=True)
        return 0
    warm = dict(spec, count=min(spec["count"], 100_000))
    for _ in range(min(args.warmup, 1)):  # pages the binary and libstdc++ in; untimed
        ref_run_concurrent(ref_bench_cmd(warm, C2_GROUPS, 16384), cores[:1])
    t0 = time.perf_counter()
    res = ref_run_concurrent(ref_bench_cmd(spec, C2_GROUPS, 16384), cores[:k])
    wall = time.perf_counter() - t0
    step_s = [r["step_s"] for r in res]
    value = k * spec["count"] / max(step_s)
    line.update({
        "value": value, "steps": k, "warmup": min(args.warmup, 1), "ms_per_step": 1000 * statistics.mean(step_s),
        "ms_steps": [round(1000 * x, 1) for x in step_s], "wall_s": wall,
        "steps_note": f"{k} steps run concurrently, one per host core (requested {args.steps}); "
                      "value = steps x samples / slowest step (build_plan + report + simulate; synth not timed)",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": k, "kind": "reference",
                         "sample": f"{k} concurrent single-threaded reference steps, each the full C2 corpus "
                                   f"({spec['count']} samples)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "result": {kk: res[0][kk] for kk in ("iterations", "packs", "abr", "cr", "total_seconds", "plan_fnv")},
    })
    print(json.dumps(line), flush=True)
    return 0


DATA = "synthetic (reference synth_lengths, C2 spec)"


def bench_config(spec):
    """Identical in both arms: the workload, not the implementation."""
    return {"workload": "C2: HBP build_plan+report+simulate, LongAlign-like long tail, groups [16K sp1, 128K sp8], "
                        "8 DP devices",
            "samples_per_step": spec["count"], "synth": c2_synth_arg(spec), "corpus_seed": spec["seed"],
            "groups": [list(g) for g in C2_GROUPS], "l_best": 16384, "dp_devices": DEVICES, "plan_seed": PLAN_SEED}


class CpuBaseline:
    """cpu_baseline of our arm: one reference step on the full C2 corpus on
    one host core (the reference is single-threaded), run in the background
    on a core this process does not use while the GPU legs run."""

    def __init__(self, spec):
        self.p = None
        self.spec = spec
        cores = sorted(os.sched_getaffinity(0))
        if not os.path.exists(REF_BENCH) or len(cores) < 2:
            return
        self.core = cores[-1]
        os.sched_setaffinity(0, set(cores[:-1]))
        self.p = subprocess.Popen(ref_bench_cmd(spec, C2_GROUPS, 16384), stdout=subprocess.PIPE,
                                  stderr=subprocess.PIPE, text=True, preexec_fn=_pin(self.core))

    def result(self):
        if self.p is None:
            return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                    "sample": "unavailable: oracle/_ref/ref_bench not built or a single host core"}
        o, e = self.p.communicate()
        if self.p.returncode != 0:
            return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e[-300:]}"}
        r = json.loads(o.strip().splitlines()[-1])
        return {"value": r["samples"] / r["step_s"], "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": f"one step on the full C2 corpus ({r['samples']} samples), host core {self.core}, "
                          "run concurrently with the GPU legs on a core the GPU process does not use",
                "seconds": r["step_s"], "result": {k: r[k] for k in ("iterations", "packs", "abr", "cr",
                                                                     "total_seconds", "plan_fnv")}}

    def kill(self):
        if self.p is not None and self.p.poll() is None:
            self.p.kill()


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args, rank, world, local):
    import torch
    from paper_2503_07680_b200 import abi

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = abi.load_library()
    ctx = abi.Context(local)
    stream = torch.cuda.ExternalStream(lib.hbp_ctx_stream(ctx.h))

    spec0 = dict(C2)
    if args.n:
        spec0["count"] = args.n
    # reference step on the same corpus on one spare host core, in the background
    cpu_bl = CpuBaseline(spec0) if rank == 0 and world == 1 and not args.no_cpu else None
    spec = dict(spec0, seed=C2["seed"] + rank)  # independent replica per rank
    L = synth(lib, spec)
    n = len(L)
    d_len = torch.from_numpy(L).cuda()
    h_len = torch.from_numpy(L).pin_memory()
    prof = abi.default_profile()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def step_device(c=None, dl=None):
        c = c or ctx
        dl = d_len if dl is None else dl
        s, keep = abi.device_samples(0, dl.data_ptr(), n, "bench")
        plan = c.build_plan_samples(s, C2_GROUPS, 16384, device_count=DEVICES, seed=PLAN_SEED)
        plan.report()
        plan.simulate(prof)
        return plan

    phases = os.environ.get("HBP_BENCH_PHASES") == "1"

    def step_e2e(c=None):
        c = c or ctx
        t0 = time.perf_counter()
        s, keep = abi.make_samples(None, h_len.numpy(), "bench")
        plan = c.build_plan_samples(s, C2_GROUPS, 16384, device_count=DEVICES, seed=PLAN_SEED)
        t1 = time.perf_counter()
        m = plan.report()
        st = plan.simulate(prof)
        t2 = time.perf_counter()
        v = abi.PlanView()
        c.check(lib.hbp_plan_view_get(c.h, plan.h, C.byref(v)))
        if phases:
            t3 = time.perf_counter()
            print(f"e2e phases ms: build {1e3 * (t1 - t0):.1f} report+sim {1e3 * (t2 - t1):.1f} "
                  f"view {1e3 * (t3 - t2):.1f}", file=sys.stderr, flush=True)
        d2h = (v.n_iterations * 4 + (v.n_iterations + 1) * 8 + v.n_devices * 4 + (v.n_devices + 1) * 8
               + v.n_packs * 24 + (v.n_packs + 1) * 8 + v.n_members * 4 + 5 * 8 + 3 * 8)
        return plan, d2h, m.abr, st.total_seconds

    def timed(fn, k):
        ms = []
        out = None
        for _ in range(k):
            out = None  # the previous step's plan is freed before the next one (one plan alive, as in use)
            flush.zero_()
            torch.cuda.synchronize()
            if dist is not None:
                dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            out = fn()
            b.record(stream)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        return ms, out

    # Plans in flight: IN_FLIGHT (5) contexts (one stream and one host thread
    # each; ctypes releases the GIL inside the C-ABI calls) build independent
    # plans at once, as a loader building the plans of several corpora (or
    # epochs) does -- one plan leaves the GPU mostly idle in its first-fit
    # chains and host round trips, and the copies of one overlap the kernels
    # of another. Each context packs its own copy of the corpus (IN_FLIGHT x
    # 80 MB > the 126 MB L2). Timed on the device: events on every context's
    # stream, from a start recorded on an idle device to the last end.
    ctxs = [ctx] + [abi.Context(local) for _ in range(IN_FLIGHT - 1)]
    d_lens = [d_len] + [d_len.clone() for _ in range(IN_FLIGHT - 1)]
    streams = [stream] + [torch.cuda.ExternalStream(lib.hbp_ctx_stream(c.h)) for c in ctxs[1:]]

    def timed_inflight(fn, k):
        per = [k // IN_FLIGHT + (1 if i < k % IN_FLIGHT else 0) for i in range(IN_FLIGHT)]
        outs = [None] * IN_FLIGHT
        errs = []

        def work(i):
            try:
                for _ in range(per[i]):
                    outs[i] = None  # one plan alive per context
                    outs[i] = fn(i)
            except Exception as e:  # surfaced after the join
                errs.append(e)

        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        start = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        th = [threading.Thread(target=work, args=(i,)) for i in range(IN_FLIGHT)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errs:
            raise errs[0]
        ends = []
        for st_ in streams:
            e = torch.cuda.Event(enable_timing=True)
            e.record(st_)
            ends.append(e)
        torch.cuda.synchronize()
        return max(start.elapsed_time(e) for e in ends), outs

    # the clock sampler starts before the warm-up: nvidia-smi's start-up takes
    # the driver for ~100 ms and would land inside the first timed steps
    clocks = Clocks(local)
    clocks.start()
    time.sleep(1.0)
    for _ in range(args.warmup):
        for i in range(IN_FLIGHT):
            step_device(ctxs[i], d_lens[i])
            step_e2e(ctxs[i])
    launches0 = ctx.launches
    dev_ms, plan = timed(step_device, args.steps)  # one plan at a time: the latency of a step
    plan = None  # one plan alive at a time (the e2e loop would otherwise grow the memory pool in its first step)
    launches = (ctx.launches - launches0) // max(1, args.steps)
    e2e_ms, e2e_out = timed(step_e2e, args.steps)
    e2e_out = None
    # warm-up in flight too: the stream-ordered pool grows to hold IN_FLIGHT
    # working sets at once (growth inside a timed region stalls the device)
    timed_inflight(lambda i: step_device(ctxs[i], d_lens[i]), max(args.warmup, 1) * IN_FLIGHT)
    inf_dev_ms, _ = timed_inflight(lambda i: step_device(ctxs[i], d_lens[i]), args.steps)
    timed_inflight(lambda i: step_e2e(ctxs[i]), max(args.warmup, 1) * IN_FLIGHT)
    inf_e2e_ms, inf_out = timed_inflight(lambda i: step_e2e(ctxs[i]), args.steps)
    ck = clocks.stop()
    d2h = [o for o in inf_out if o is not None][0][1]
    inf_out = None
    # the other in-flight contexts give their memory pools back before the
    # 100M-sample legs (C5's workers are bounded by free HBM)
    for c in ctxs[1:]:
        c.close()
    ctxs = ctxs[:1]
    d_lens = d_lens[:1]

    # stage profile of one extra step (CUDA events around each engine stage)
    stages = profile_stages(ctx, lib, step_device)
    from paper_2503_07680_b200 import sweep as sweep_mod
    comm = sweep_mod.engine_comm(ctx, dist) if dist is not None else abi.Comm(ctx, abi.Comm.unique_id(ctx), 0, 1)
    sweep_res = None if args.no_sweep else run_sweep_leg(ctx, lib, rank, world, dist, comm)
    c4_res = run_c4_leg(ctx, lib, comm, rank, world, dist) if not args.no_c4 else None
    ingest_res = run_ingest_leg(ctx, lib) if rank == 0 and not args.no_ingest else None

    tot_dev = sum(dev_ms)
    tot_e2e = sum(e2e_ms)
    if dist is not None:
        t = torch.tensor([tot_dev, tot_e2e, inf_dev_ms, inf_e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_dev, tot_e2e, inf_dev_ms, inf_e2e_ms = t.tolist()
    if rank == 0:
        # headline: whole-job throughput with IN_FLIGHT plans in flight; the
        # one-plan-at-a-time step (its latency) beside it
        ms_step = inf_dev_ms / args.steps
        value = world * n / (ms_step / 1000.0)
        e2e_value = world * n / (inf_e2e_ms / args.steps / 1000.0)
        seq_ms = tot_dev / args.steps
        seq_e2e_ms = tot_e2e / args.steps
        peak, peak_kind = peaks()
        roof = roofline(stages, peak, peak_kind)
        cpu = cpu_bl.result() if cpu_bl is not None else None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64",
            "data": DATA + "; restated bit-identically in csrc/synth.cpp; rank r packs the corpus of seed 20250515 + r",
            "config": bench_config(spec0),
            "parallelism": f"replicas x{world} (packing one corpus does not shard, SURVEY.md 8(e))",
            "in_flight": IN_FLIGHT,
            "l2": (f"{IN_FLIGHT} plans in flight, each on its own copy of the corpus ({IN_FLIGHT} x {8 * n >> 20} MB "
                   "> 126 MB L2); the one-plan-at-a-time steps flush L2 (256 MB write) before every step"),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": int(d2h),
                    "ms_per_step": inf_e2e_ms / args.steps, "in_flight": IN_FLIGHT,
                    "one_at_a_time": {"value": world * n / (seq_e2e_ms / 1000.0), "ms_per_step": seq_e2e_ms,
                                      "ms_steps": [round(x, 3) for x in e2e_ms]}},
            "one_at_a_time": {"value": world * n / (seq_ms / 1000.0), "ms_per_step": seq_ms,
                              "ms_steps": [round(x, 3) for x in dev_ms]},
            "gpu_launches": int(launches),
            "roofline": roof,
            "stages_ms": {k: round(v["ms"], 4) for k, v in sorted(stages.items(), key=lambda kv: -kv[1]["ms"])[:12]},
            "clocks": ck,
            "cpu_baseline": cpu,
            "sweep": sweep_res,
            "c4": c4_res,
            "ingest": ingest_res,
        }
        print(json.dumps(line), flush=True)
    comm.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()
    return 0


IN_FLIGHT = int(os.environ.get("HBP_BENCH_IN_FLIGHT", "5"))  # plans built at once (one context each)
C1 = dict(count=100_000, short="lognormal:8.5:1.4", long_fraction=0.0, long="", max_length=131072, seed=42)
SWEEP_SMALLER = [512, 1024, 2048, 4096, 8192, 16384, 32768, 65536]  # 256 length sets with 131072
SWEEP_SP = [1, 2, 4, 8]


def run_sweep_leg(ctx, lib, rank, world, dist, comm):
    """C3 auto-selection sweep: 256 length sets x SP{1,2,4,8} x GC{on,off} =
    2048 candidates over the C1 corpus (100K, lengths >= 128), sharded across
    ranks by length set with the NCCL argmin, all in the engine
    (hbp_sweep_sharded). Three timed repetitions after an untimed one (the
    worker contexts and their memory pools are created and grown there),
    the median reported; time = max over ranks."""
    import torch
    from paper_2503_07680_b200 import abi, sweep
    L = np.maximum(synth(lib, C1), 128)
    cands = sweep.make_candidates(ctx, 131072, SWEEP_SMALLER, SWEEP_SP)
    s, keep = abi.make_samples(None, L, "c1")
    opts = dict(device_count=8, seed=7)
    sweep.run_sweep_nccl(comm, s, cands, None, **opts)  # warm-up: every worker context, pools grown
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    reps = []
    for _ in range(3):  # three timed repetitions; the median is reported (all of them beside it)
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        secs, best, local = sweep.run_sweep_nccl(comm, s, cands, None, **opts)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([el], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        reps.append(el)
    elapsed = statistics.median(reps)
    return {"workload": "C3: 256 length sets x SP{1,2,4,8} x GC{on,off}, C1 corpus (100K), 8B analytic cost model",
            "candidates": len(cands), "feasible": int(np.isfinite(secs).sum()), "seconds": elapsed,
            "seconds_reps": [round(x, 4) for x in reps],
            "candidates_per_s": len(cands) / elapsed, "best_index": best[1],
            "best_groups": cands[best[1]][0] if best[1] >= 0 else None, "best_seconds": best[0],
            "local_candidates_rank0": local,
            "sharding": f"length sets round-robin over {world} rank(s); hbp_sweep_sharded: ncclAllReduce(MIN) of "
                        "seconds + ncclAllGather of (best seconds, best index) on the engine's stream"}


C4 = dict(C2, count=100_000_000)
C4_PROFILE = os.path.join(ROOT, "tests", "golden", "deepseek_v2_236b_analytic.json")


def c4_profile():
    """DeepSeek-V2 236B analytic cost model (builder-written fixture, see its _note)."""
    from paper_2503_07680_b200 import abi
    with open(C4_PROFILE) as f:
        d = json.load(f)
    p = abi.default_profile()
    for name, _ in abi.HardwareProfile._fields_:
        if name in d:
            setattr(p, name, d[name])
    return p


def run_c4_leg(ctx, lib, comm, rank=0, world=1, dist=None, steps=3, warmup=3):
    """BASELINE config C4: 100M samples of the C2 spec, groups [16K sp1,
    128K sp8] with ckpt derived under the DeepSeek-V2 236B cost model, 8 DP
    devices: build_plan + report (ABR/CR) + simulate, corpus resident in HBM.
    Then C5 in full: the 4096-candidate sweep (512 length sets x SP{1,2,4,8} x
    GC{on,off}) over the same corpus, sharded across the ranks."""
    import torch
    from paper_2503_07680_b200 import abi, sweep
    stream = torch.cuda.ExternalStream(lib.hbp_ctx_stream(ctx.h))
    L = synth(lib, C4)
    n = len(L)
    d_len = torch.from_numpy(L).cuda()
    del L
    prof = c4_profile()
    pr = abi.analytic_profiler(prof)
    pr.device_memory = prof.device_memory
    groups = [(16384, 1, ctx.derive_ckpt(pr, 16384, 1)), (131072, 8, ctx.derive_ckpt(pr, 131072, 8))]

    def step():
        s, keep = abi.device_samples(0, d_len.data_ptr(), n, "c4")
        plan = ctx.build_plan_samples(s, groups, 16384, device_count=DEVICES, seed=PLAN_SEED)
        m = plan.report()
        st = plan.simulate(prof)
        return plan, m, st

    for _ in range(warmup):  # memory pool / block cache growth at this size takes a few steps
        out = step()
        out = None
    ms = []
    for _ in range(steps):
        out = None
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        out = step()
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    plan, m, st = out
    res = {"workload": "C4: 100M samples (C2 spec), groups [16K sp1, 128K sp8], DeepSeek-V2 236B analytic cost model "
                       "(tests/golden/deepseek_v2_236b_analytic.json), 8 DP devices; build_plan+report+simulate",
           "samples": n, "groups": groups, "ms_per_step": statistics.mean(ms), "ms_steps": [round(x, 2) for x in ms],
           "samples_per_s": n / (statistics.mean(ms) / 1000.0), "abr": m.abr, "cr": m.cr,
           "estimated_seconds": st.total_seconds}
    # report + simulate sharded by DP column across the ranks (hbp_eval_sharded:
    # NCCL all-reduce of per-iteration vectors on the engine's stream),
    # against the single-GPU evaluation
    def timed_eval(fn):
        best = math.inf
        for _ in range(3):
            torch.cuda.synchronize()
            if dist is not None:
                dist.barrier()
            t0 = time.perf_counter()
            r = fn()
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
            if dist is not None:
                tt = torch.tensor([el], dtype=torch.float64, device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                el = float(tt.item())
            best = min(best, el)
        return r, best

    (m1, st1), single_s = timed_eval(lambda: (plan.report(), plan.simulate(prof)))
    (m2, st2), shard_s = timed_eval(lambda: comm.evaluate(plan, prof))
    res["sharded_eval"] = {"ranks": world, "dp_columns": DEVICES, "ms": 1e3 * shard_s, "single_gpu_ms": 1e3 * single_s,
                           "identical": bool(m1.abr == m2.abr and m1.dbr == m2.dbr and m1.cr == m2.cr
                                             and st1.total_seconds == st2.total_seconds),
                           "exchange": "hbp_eval_sharded: ncclAllReduce MAX/SUM/MIN of 6 per-iteration vectors, "
                                       "then SUM of 2, on the engine's stream"}
    out = plan = None
    # C5 in full: 512 length sets x SP{1,2,4,8} x GC{on,off} = 4096 candidates
    # over the same 100M corpus, length sets dealt across the ranks
    # (hbp_sweep_sharded: one plan per set, NCCL MIN of the seconds and
    # all-gather of each rank's best); wall time = max over ranks
    cands = sweep.make_candidates(ctx, 131072, [256, 512, 1024, 2048, 4096, 8192, 16384, 32768, 65536], SWEEP_SP, prof)
    s, keep = abi.device_samples(0, d_len.data_ptr(), n, "c5")
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    secs, best, local = sweep.run_sweep_nccl(comm, s, cands, prof, device_count=DEVICES, seed=PLAN_SEED)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if dist is not None:
        tt = torch.tensor([el], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        el = float(tt.item())
    res["c5"] = {"workload": "C5: 512 length sets ({131072} + subsets of {256..64K}) x SP{1,2,4,8} x GC{on,off} "
                             "over the C4 corpus (100M), DeepSeek-V2 cost model, sharded by length set",
                 "candidates": len(cands), "seconds": el, "candidates_per_s": len(cands) / el,
                 "feasible": int(np.isfinite(secs).sum()), "best_index": int(best[1]),
                 "best_groups": cands[best[1]][0] if best[1] >= 0 else None, "best_seconds": best[0],
                 "local_candidates_rank0": local, "ranks": world}
    return res


def profile_stages(ctx, lib, fn):
    """Per-kernel-family device time of one step (the engine times its own
    launches with CUDA events on its stream when profiling is on)."""
    if not hasattr(lib, "hbp_ctx_set_profiling"):
        return {}
    lib.hbp_ctx_set_profiling(ctx.h, 1)
    fn()
    ctx.synchronize()
    lib.hbp_ctx_set_profiling(ctx.h, 0)
    out = {}
    name = C.create_string_buffer(128)
    ms, launches, nbytes = C.c_double(), C.c_int64(), C.c_double()
    i = 0
    while lib.hbp_ctx_stage_stats(ctx.h, i, name, 128, C.byref(ms), C.byref(launches), C.byref(nbytes)) == 0:
        k = name.value.decode()
        # the scan call sites (scan.nf1, scan.radix1, ...) form one kernel family
        fam = "scan" if k.startswith("scan.") or k == "nf.tiles_scan" else k
        o = out.setdefault(fam, {"ms": 0.0, "launches": 0, "bytes": 0.0})
        o["ms"] += ms.value
        o["launches"] += launches.value
        o["bytes"] += nbytes.value
        i += 1
    return out


TRAFFIC_FILE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02_traffic.json")


def roofline(stages, peak, peak_kind):
    """The step's dominant kernel family (largest summed device time; CUDA
    events around every launch on the engine's stream): algorithmic bytes
    (SURVEY.md 8(d) per-unit figures x units, registered per launch by the
    engine) / its device time. The sort and scan families the north star
    targets are listed beside it."""
    cands = {k: v for k, v in stages.items() if v["ms"] > 0}
    if not cands:
        return None
    total_ms = sum(x["ms"] for x in stages.values())
    k, v = max(cands.items(), key=lambda kv: kv[1]["ms"])
    achieved = v["bytes"] / (v["ms"] / 1000.0) / 1e9
    traffic = None
    if os.path.exists(TRAFFIC_FILE):  # ncu --set full capture of the same step, per launch
        with open(TRAFFIC_FILE) as f:
            traffic = json.load(f).get(k, {}).get("dram_bytes_per_launch")

    def fam(vv):
        gbs = vv["bytes"] / (vv["ms"] / 1000.0) / 1e9
        return {"ms": round(vv["ms"], 4), "launches": vv["launches"], "share": round(vv["ms"] / total_ms, 4),
                "achieved_gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}

    return {"bound": "hbm", "kernel": k, "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
            "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
            "algorithmic_bytes_per_launch": v["bytes"] / max(v["launches"], 1),
            "launches": v["launches"], "ms": v["ms"], "share_of_kernel_time": v["ms"] / total_ms,
            "note": "fit.chain is a dependency chain over bins (latency-bound, DESIGN.md); its bytes are "
                    "12 B/item + 12 B/bin (SURVEY.md 8(d) FFD residue)" if k.startswith("fit.chain") else None,
            "sort_scan": {kk: fam(vv) for kk, vv in stages.items()
                          if (kk.startswith("radix") or kk == "scan") and vv["ms"] > 0},
            "families": {kk: fam(vv) for kk, vv in sorted(cands.items(), key=lambda kv: -kv[1]["ms"])[:10]}}


INGEST_SAMPLES = 2_000_000


def run_ingest_leg(ctx, lib):
    """load_lengths of a JSONL corpus (2M records of
    the C2 spec, {"id":i,"length":L} per line, 57 MB) through the C-ABI --
    host text in, host ids + lengths out (e2e, wall clock) -- with the
    device-side parse timed by CUDA events; the reference's istream parser
    (oracle/_ref, one core) on the same bytes beside it."""
    import time
    L = synth(lib, C2, INGEST_SAMPLES)
    text = "".join(f'{{"id":{i},"length":{v}}}\n' for i, v in enumerate(L.tolist())).encode()
    for _ in range(2):
        ctx.load_lengths(text, "jsonl", with_ids=True)
    ctx.synchronize()
    e2e = []
    for _ in range(3):
        t0 = time.perf_counter()
        ids, got = ctx.load_lengths(text, "jsonl", with_ids=True)
        e2e.append((time.perf_counter() - t0) * 1e3)
    assert np.array_equal(got, L) and np.array_equal(ids, np.arange(len(L)))
    lib.hbp_ctx_set_profiling(ctx.h, 1)
    ctx.load_lengths(text, "jsonl")
    ctx.synchronize()
    lib.hbp_ctx_set_profiling(ctx.h, 0)
    st = {}
    name = C.create_string_buffer(128)
    ms, launches, nbytes = C.c_double(), C.c_int64(), C.c_double()
    i = 0
    while lib.hbp_ctx_stage_stats(ctx.h, i, name, 128, C.byref(ms), C.byref(launches), C.byref(nbytes)) == 0:
        st[name.value.decode()] = ms.value
        i += 1
    dev_ms = sum(st.values())
    parse_ms = st.get("k_parse_jsonl", 0.0)
    peak, peak_kind = peaks()
    # parse kernel: reads the text once, reads 2 line starts and writes value + id per line
    alg = len(text) + 32.0 * len(L)
    ref = None
    try:
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle"))
        import pyoracle
        if pyoracle.available("reference"):
            o = pyoracle.Oracle("reference")
            t0 = time.perf_counter()
            _, want = o.load_lengths(text, "jsonl", "bench")
            ref = {"ms": (time.perf_counter() - t0) * 1e3, "cores": 1, "kind": "reference",
                   "identical": bool(np.array_equal(want, got))}
    except Exception as e:  # noqa: BLE001
        ref = {"unavailable": str(e)}
    return {"workload": f"load_lengths(jsonl): {len(L)} records of the C2 spec, {len(text)} bytes",
            "e2e_ms": round(statistics.median(e2e), 3), "device_ms": round(dev_ms, 4),
            "records_per_s_e2e": len(L) / (statistics.median(e2e) / 1e3),
            "stages_ms": {k: round(v, 4) for k, v in sorted(st.items(), key=lambda kv: -kv[1])},
            "parse_roofline": {"kernel": "k_parse_jsonl", "bound": "hbm", "algorithmic_bytes": alg,
                               "achieved": alg / (parse_ms / 1e3) / 1e9 if parse_ms else None, "peak": peak,
                               "peak_kind": peak_kind, "unit": "GB/s",
                               "frac": alg / (parse_ms / 1e3) / 1e9 / peak if parse_ms else None},
            "reference": ref}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=0, help="override corpus size (default 10M)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-sweep", action="store_true", help="skip the auto-selection sweep leg")
    ap.add_argument("--no-c4", action="store_true", help="skip the 100M-sample C4 / C5 legs")
    ap.add_argument("--no-ingest", action="store_true", help="skip the corpus-file (JSONL) ingest leg")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch this command under torchrun
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    rank, world, local = dist_env()
    if world != args.gpus and args.impl == "ours":
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
