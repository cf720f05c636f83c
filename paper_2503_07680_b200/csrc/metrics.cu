// metrics.cu — report() and simulate() over a flat plan in HBM.
//
// Reference: dbr / abr / report (src/metrics.cpp:22-144), device_work /
// iter_time (src/costmodel.cpp:55-104), simulate (src/sim.cpp:9-60) and
// switch_count (src/schedule.cpp:67-79). One thread owns one iteration and
// walks its devices in order, so every per-iteration DBR / ABR / time is
// computed with the reference's operation order (bit-identical). The
// run-level sums -- mean DBR / ABR, CR's token sums, the total time -- are
// warp-level reductions of fixed shape (per thread, the block's last five
// levels and the final one by warp shuffles, three cross-warp levels in
// shared memory): deterministic, and within 1e-15 relative of the
// reference's sequential sums. Integer sums (tokens, comm, padding) are exact.
#include "costmodel.cuh"
#include "metrics.cuh"

namespace hbp_b200 {

namespace {

constexpr int EB = 256;
constexpr int EG = 148 * 4;

struct Partial {
    double dbr, abr, seconds;
    unsigned long long tokens, comm, pad_gap, pad_cap, switches;
};

struct EvalArgs {
    PlanArrays p;
    const hbp_group_config* groups;
    int ng;
    bool simulate;
    hbp_hardware_profile prof;
    double* out_dbr;
    double* out_abr;
    double* out_secs;
    double* out_dcomp;
    double* out_dcomm;
    double* out_didle;
    Partial* partials;
    unsigned long long* report_err;  // key = 2*i + (abr ? 1 : 0); kind in err_kind
    unsigned long long* sim_err;     // key = (i << 20) | d
};

__device__ __forceinline__ void add_partial(Partial& a, const Partial& b) {
    a.dbr += b.dbr;
    a.abr += b.abr;
    a.seconds += b.seconds;
    a.tokens += b.tokens;
    a.comm += b.comm;
    a.pad_gap += b.pad_gap;
    a.pad_cap += b.pad_cap;
    a.switches += b.switches;
}

// Fixed-order block reduction of the per-thread partials: the pairing
// s[t] += s[t + w] for w = EB/2 .. 1, the three cross-warp levels through
// shared memory, the last five inside warp 0 by shuffles (same pairs, same
// operand order: deterministic and identical wherever it runs).
__device__ __forceinline__ Partial shfl_down_partial(const Partial& p, int o) {
    Partial q;
    q.dbr = __shfl_down_sync(0xffffffffu, p.dbr, o);
    q.abr = __shfl_down_sync(0xffffffffu, p.abr, o);
    q.seconds = __shfl_down_sync(0xffffffffu, p.seconds, o);
    q.tokens = __shfl_down_sync(0xffffffffu, p.tokens, o);
    q.comm = __shfl_down_sync(0xffffffffu, p.comm, o);
    q.pad_gap = __shfl_down_sync(0xffffffffu, p.pad_gap, o);
    q.pad_cap = __shfl_down_sync(0xffffffffu, p.pad_cap, o);
    q.switches = __shfl_down_sync(0xffffffffu, p.switches, o);
    return q;
}

__device__ __forceinline__ void block_reduce_partial(Partial acc, Partial* out) {
    __shared__ Partial s[EB];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int w = EB / 2; w >= 32; w >>= 1) {
        if (threadIdx.x < static_cast<unsigned>(w)) add_partial(s[threadIdx.x], s[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x < 32) {
        Partial v = s[threadIdx.x];
        for (int o = 16; o > 0; o >>= 1) {
            const Partial q = shfl_down_partial(v, o);
            if (threadIdx.x < static_cast<unsigned>(o)) add_partial(v, q);
        }
        if (threadIdx.x == 0) *out = v;
    }
}

__global__ void __launch_bounds__(EB) k_eval(EvalArgs a) {
    Partial acc{0, 0, 0, 0, 0, 0, 0, 0};
    const PlanArrays& P = a.p;
    for (i64 i = blockIdx.x * static_cast<i64>(EB) + threadIdx.x; i < P.I; i += static_cast<i64>(gridDim.x) * EB) {
        const i64 d0 = P.iter_dev_offsets[i], d1 = P.iter_dev_offsets[i + 1];
        const int g = P.iter_group[i];
        const hbp_group_config cfg = a.groups[g];
        if (i > 0) {
            const hbp_group_config prev = a.groups[P.iter_group[i - 1]];
            if (prev.sp != cfg.sp || prev.ckpt != cfg.ckpt) acc.switches += 1;
        }
        const double nd = static_cast<double>(d1 - d0);
        if (d1 == d0) {
            atomicMin(a.report_err, static_cast<unsigned long long>(2 * i));  // "dbr: no devices"
            continue;
        }
        int64_t tmax = 0, amax = 0, tokens = 0;
        for (i64 d = d0; d < d1; ++d) {
            int64_t t = 0, at = 0;
            for (i64 k = P.dev_pack_offsets[d]; k < P.dev_pack_offsets[d + 1]; ++k) {
                t += P.pack_total[k];
                at += P.pack_attention[k];
                acc.pad_gap += static_cast<unsigned long long>(P.pack_capacity[k] - P.pack_total[k]);
                acc.pad_cap += static_cast<unsigned long long>(P.pack_capacity[k]);
            }
            tmax = t > tmax ? t : tmax;
            amax = at > amax ? at : amax;
            tokens += t;
        }
        acc.tokens += static_cast<unsigned long long>(tokens);
        if (cfg.sp > 1) acc.comm += static_cast<unsigned long long>(tokens);
        double dbr = 0.0, abr = 0.0;
        if (tmax == 0) {
            atomicMin(a.report_err, static_cast<unsigned long long>(2 * i));
        } else if (amax == 0) {
            atomicMin(a.report_err, static_cast<unsigned long long>(2 * i + 1));
        } else {
            double gt = 0.0, ga = 0.0;
            for (i64 d = d0; d < d1; ++d) {
                int64_t t = 0, at = 0;
                for (i64 k = P.dev_pack_offsets[d]; k < P.dev_pack_offsets[d + 1]; ++k) {
                    t += P.pack_total[k];
                    at += P.pack_attention[k];
                }
                gt = __dadd_rn(gt, static_cast<double>(tmax - t));
                ga = __dadd_rn(ga, static_cast<double>(amax - at));
            }
            dbr = __ddiv_rn(gt, __dmul_rn(static_cast<double>(tmax), nd));
            abr = __ddiv_rn(ga, __dmul_rn(static_cast<double>(amax), nd));
        }
        if (a.out_dbr) a.out_dbr[i] = dbr;
        if (a.out_abr) a.out_abr[i] = abr;
        acc.dbr += dbr;
        acc.abr += abr;
        if (!a.simulate) continue;
        double imax = 0.0;
        for (i64 d = d0; d < d1; ++d) {
            int64_t padded = 0, attn = 0, maxcap = 0;
            for (i64 k = P.dev_pack_offsets[d]; k < P.dev_pack_offsets[d + 1]; ++k) {
                const int64_t cap = P.pack_capacity[k];
                padded += cap;
                attn += P.pack_attention[k];
                const int64_t pad = cap - P.pack_total[k];
                attn += pad * pad;
                maxcap = cap > maxcap ? cap : maxcap;
            }
            double busy = 0.0;
            if (padded != 0) {
                bool bad = cfg.sp < 1 || cfg.ckpt < 0 || cfg.ckpt > a.prof.layer_count;
                if (!bad) bad = cm_memory_used(maxcap, cfg.sp, cfg.ckpt, a.prof) > a.prof.device_memory;
                if (bad) {
                    atomicMin(a.sim_err, (static_cast<unsigned long long>(i) << 20) | static_cast<unsigned long long>(d - d0));
                } else {
                    busy = cm_iter_time(padded, attn, cfg.sp, cfg.ckpt, a.prof);
                }
            }
            const double comm = padded != 0 ? cm_comm(padded, cfg.sp, a.prof) : (cfg.sp > 1 ? 0.0 : 0.0);
            if (a.out_dcomm) a.out_dcomm[d] = comm;
            if (a.out_dcomp) a.out_dcomp[d] = __dsub_rn(busy, comm);
            imax = busy > imax ? busy : imax;
        }
        if (a.out_didle) {
            for (i64 d = d0; d < d1; ++d) {
                // idle = max - (compute + comm)  (sim.cpp:49-52)
                a.out_didle[d] = __dsub_rn(imax, __dadd_rn(a.out_dcomp[d], a.out_dcomm[d]));
            }
        }
        if (a.out_secs) a.out_secs[i] = imax;
        acc.seconds += imax;
    }
    // block reduction in fixed order
    block_reduce_partial(acc, a.partials + blockIdx.x);
}

// Fixed-order final reduction of the block partials by one warp: lane l
// sums partials l, l + 32, ... in order, then a fixed butterfly.
__device__ __forceinline__ Partial shfl_xor_partial(const Partial& p, int o) {
    Partial q;
    q.dbr = __shfl_xor_sync(0xffffffffu, p.dbr, o);
    q.abr = __shfl_xor_sync(0xffffffffu, p.abr, o);
    q.seconds = __shfl_xor_sync(0xffffffffu, p.seconds, o);
    q.tokens = __shfl_xor_sync(0xffffffffu, p.tokens, o);
    q.comm = __shfl_xor_sync(0xffffffffu, p.comm, o);
    q.pad_gap = __shfl_xor_sync(0xffffffffu, p.pad_gap, o);
    q.pad_cap = __shfl_xor_sync(0xffffffffu, p.pad_cap, o);
    q.switches = __shfl_xor_sync(0xffffffffu, p.switches, o);
    return q;
}

__global__ void k_eval_final(const Partial* __restrict__ partials, int n, Partial* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    Partial acc{0, 0, 0, 0, 0, 0, 0, 0};
    for (int b = lane; b < n; b += 32) add_partial(acc, partials[b]);
    for (int o = 1; o < 32; o <<= 1) {  // lanes l and l ^ o hold the same pair after each step: order fixed
        const Partial q = shfl_xor_partial(acc, o);
        if (lane & o) {
            Partial t = q;
            add_partial(t, acc);
            acc = t;
        } else {
            add_partial(acc, q);
        }
    }
    if (threadIdx.x == 0) *out = acc;
}

}  // namespace

void eval_plan(Ctx& c, const PlanArrays& p, int32_t device_count, const std::vector<hbp_group_config>& groups,
               const hbp_hardware_profile* profile, EvalOut& out, double* d_dbr, double* d_abr, double* d_secs,
               double* d_dcomp, double* d_dcomm, double* d_didle) {
    cudaStream_t s = c.stream;
    if (profile) {
        const int pc = cm_profile_check(*profile);
        if (pc) fail_validation(cm_profile_message(pc));
        if (p.I == 0) fail_validation("simulate: empty plan");
    }
    if (p.I == 0) fail_validation("metrics report: empty plan");
    for (const auto& it : groups) (void)it;
    DevBuf<hbp_group_config> dg(groups.size(), s);
    CUDA_CHECK(cudaMemcpyAsync(dg.p, groups.data(), sizeof(hbp_group_config) * groups.size(), cudaMemcpyHostToDevice, s));
    DevBuf<Partial> partials(EG + 1, s);
    DevBuf<unsigned long long> errs(2, s);
    CUDA_CHECK(cudaMemsetAsync(errs.p, 0xff, sizeof(unsigned long long) * 2, s));
    // idle needs compute / comm scratch even if the caller did not ask for them
    DevBuf<double> tmp_comp, tmp_comm;
    if (d_didle && !d_dcomp) {
        tmp_comp.alloc(static_cast<size_t>(p.D), s);
        d_dcomp = tmp_comp.p;
    }
    if (d_didle && !d_dcomm) {
        tmp_comm.alloc(static_cast<size_t>(p.D), s);
        d_dcomm = tmp_comm.p;
    }
    EvalArgs a{p, dg.p, static_cast<int>(groups.size()), profile != nullptr,
               profile ? *profile : hbp_hardware_profile{}, d_dbr, d_abr, d_secs, d_dcomp, d_dcomm, d_didle,
               partials.p, errs.p, errs.p + 1};
    const int grid = static_cast<int>(std::min<i64>(EG, (p.I + EB - 1) / EB));
    LAUNCH(k_eval, grid, EB, 0, s, a);
    LAUNCH(k_eval_final, 1, 32, 0, s, partials.p, grid, partials.p + EG);
    const auto e = read_vector(c, errs.p, 2);
    if (e[0] != ~0ull) {
        const i64 i = static_cast<i64>(e[0] >> 1);
        const bool abr = e[0] & 1;
        // distinguish "no devices" from "all zero" for the DBR case
        const auto offs = read_vector(c, p.iter_dev_offsets + i, 2);
        if (!abr && offs[1] == offs[0]) fail_validation("dbr: no devices");
        fail_validation(abr ? "abr undefined: all devices carry zero attention"
                            : "dbr undefined: all devices carry zero tokens");
    }
    if (profile && e[1] != ~0ull) {
        const i64 i = static_cast<i64>(e[1] >> 20);
        const i64 dd = static_cast<i64>(e[1] & 0xfffff);
        const int g = read_vector(c, p.iter_group + i, 1)[0];
        const hbp_group_config cfg = groups.at(static_cast<size_t>(g));
        if (cfg.sp < 1) fail_validation("sp must be >= 1");
        if (cfg.ckpt < 0 || cfg.ckpt > profile->layer_count) fail_validation("ckpt must lie in [0, layer_count]");
        const i64 d = read_vector(c, p.iter_dev_offsets + i, 1)[0] + dd;
        const auto po = read_vector(c, p.dev_pack_offsets + d, 2);
        const auto caps = read_vector(c, p.pack_capacity + po[0], static_cast<size_t>(po[1] - po[0]));
        int64_t maxcap = 0;
        for (auto v : caps) maxcap = v > maxcap ? v : maxcap;
        const int64_t used = cm_memory_used(maxcap, cfg.sp, cfg.ckpt, *profile);
        fail_infeasible("iteration " + std::to_string(i) + ": configuration sp=" + std::to_string(cfg.sp) +
                        " ckpt=" + std::to_string(cfg.ckpt) + " at length " + std::to_string(maxcap) + " requires " +
                        std::to_string(used) + " bytes, " + std::to_string(profile->device_memory) + " available");
    }
    const Partial tot = read_scalar(c, partials.p + EG);
    const double ni = static_cast<double>(p.I);
    const double total = static_cast<double>(tot.tokens);
    const double comm = static_cast<double>(tot.comm);
    const double pad_gap = static_cast<double>(tot.pad_gap);
    const double pad_cap = static_cast<double>(tot.pad_cap);
    out.m.dbr = tot.dbr / ni;
    out.m.abr = tot.abr / ni;
    out.m.cr = total > 0.0 ? comm / total : 0.0;
    out.m.pr = pad_cap > 0.0 ? pad_gap / pad_cap : 0.0;
    out.m.ave_t = total / (ni * static_cast<double>(device_count));
    out.total_seconds = tot.seconds;
    out.switch_count = static_cast<int32_t>(tot.switches);
}

// ---------------------------------------------------------------------------
// Evaluation sharded by data-parallel column: the rank
// owning device columns [c0, c1) of every iteration computes their maxima,
// sums and simulated busy times (phase 0), then -- after an all-reduce MAX
// of the maxima -- their gaps to the maxima (phase 1); after an all-reduce
// SUM of the gaps every rank finishes identically. Gaps are integers, so
// their sum is exact in any order and DBR / ABR per iteration, and the
// run-level reduction (same grid, same order as k_eval), are bit-identical
// to the single-GPU report / simulate.
// ---------------------------------------------------------------------------

namespace {

struct ColArgs {
    PlanArrays p;
    const hbp_group_config* groups;
    bool simulate;
    hbp_hardware_profile prof;
    int32_t c0, c1;
    hbp_eval_columns_bufs b;
};

__global__ void __launch_bounds__(EB) k_cols_phase0(ColArgs a) {
    const PlanArrays& P = a.p;
    for (i64 i = blockIdx.x * static_cast<i64>(EB) + threadIdx.x; i < P.I; i += static_cast<i64>(gridDim.x) * EB) {
        const i64 d0 = P.iter_dev_offsets[i], d1 = P.iter_dev_offsets[i + 1];
        const hbp_group_config cfg = a.groups[P.iter_group[i]];
        const i64 lo = d0 + a.c0 < d1 ? d0 + a.c0 : d1, hi = d0 + a.c1 < d1 ? d0 + a.c1 : d1;
        int64_t tmax = 0, amax = 0, tokens = 0, pg = 0, pc = 0;
        double imax = 0.0;
        for (i64 d = lo; d < hi; ++d) {
            int64_t t = 0, at = 0, padded = 0, attn = 0, maxcap = 0;
            for (i64 k = P.dev_pack_offsets[d]; k < P.dev_pack_offsets[d + 1]; ++k) {
                const int64_t cap = P.pack_capacity[k], tot = P.pack_total[k];
                t += tot;
                at += P.pack_attention[k];
                pg += cap - tot;
                pc += cap;
                padded += cap;
                attn += P.pack_attention[k] + (cap - tot) * (cap - tot);
                maxcap = cap > maxcap ? cap : maxcap;
            }
            tmax = t > tmax ? t : tmax;
            amax = at > amax ? at : amax;
            tokens += t;
            if (a.simulate && padded != 0) {
                bool bad = cfg.sp < 1 || cfg.ckpt < 0 || cfg.ckpt > a.prof.layer_count;
                if (!bad) bad = cm_memory_used(maxcap, cfg.sp, cfg.ckpt, a.prof) > a.prof.device_memory;
                if (bad) {
                    atomicMin(reinterpret_cast<unsigned long long*>(a.b.sim_err),
                              (static_cast<unsigned long long>(i) << 20) | static_cast<unsigned long long>(d - d0));
                } else {
                    const double busy = cm_iter_time(padded, attn, cfg.sp, cfg.ckpt, a.prof);
                    imax = busy > imax ? busy : imax;
                }
            }
        }
        a.b.tmax[i] = tmax;
        a.b.amax[i] = amax;
        a.b.tokens[i] = tokens;
        a.b.pad_gap[i] = pg;
        a.b.pad_cap[i] = pc;
        if (a.b.busy) a.b.busy[i] = imax;
    }
}

__global__ void __launch_bounds__(EB) k_cols_phase1(ColArgs a) {
    const PlanArrays& P = a.p;
    for (i64 i = blockIdx.x * static_cast<i64>(EB) + threadIdx.x; i < P.I; i += static_cast<i64>(gridDim.x) * EB) {
        const i64 d0 = P.iter_dev_offsets[i], d1 = P.iter_dev_offsets[i + 1];
        const i64 lo = d0 + a.c0 < d1 ? d0 + a.c0 : d1, hi = d0 + a.c1 < d1 ? d0 + a.c1 : d1;
        const int64_t tmax = a.b.tmax[i], amax = a.b.amax[i];
        int64_t tg = 0, ag = 0;
        for (i64 d = lo; d < hi; ++d) {
            int64_t t = 0, at = 0;
            for (i64 k = P.dev_pack_offsets[d]; k < P.dev_pack_offsets[d + 1]; ++k) {
                t += P.pack_total[k];
                at += P.pack_attention[k];
            }
            tg += tmax - t;
            ag += amax - at;
        }
        a.b.tgap[i] = tg;
        a.b.agap[i] = ag;
    }
}

// the run-level accumulation of k_eval over the reduced per-iteration values
__global__ void __launch_bounds__(EB) k_cols_finish(ColArgs a, Partial* partials, unsigned long long* report_err) {
    Partial acc{0, 0, 0, 0, 0, 0, 0, 0};
    const PlanArrays& P = a.p;
    for (i64 i = blockIdx.x * static_cast<i64>(EB) + threadIdx.x; i < P.I; i += static_cast<i64>(gridDim.x) * EB) {
        const i64 d0 = P.iter_dev_offsets[i], d1 = P.iter_dev_offsets[i + 1];
        const hbp_group_config cfg = a.groups[P.iter_group[i]];
        if (i > 0) {
            const hbp_group_config prev = a.groups[P.iter_group[i - 1]];
            if (prev.sp != cfg.sp || prev.ckpt != cfg.ckpt) acc.switches += 1;
        }
        const double nd = static_cast<double>(d1 - d0);
        if (d1 == d0) {
            atomicMin(report_err, static_cast<unsigned long long>(2 * i));
            continue;
        }
        const int64_t tmax = a.b.tmax[i], amax = a.b.amax[i], tokens = a.b.tokens[i];
        acc.pad_gap += static_cast<unsigned long long>(a.b.pad_gap[i]);
        acc.pad_cap += static_cast<unsigned long long>(a.b.pad_cap[i]);
        acc.tokens += static_cast<unsigned long long>(tokens);
        if (cfg.sp > 1) acc.comm += static_cast<unsigned long long>(tokens);
        double dbr = 0.0, abr = 0.0;
        if (tmax == 0) {
            atomicMin(report_err, static_cast<unsigned long long>(2 * i));
        } else if (amax == 0) {
            atomicMin(report_err, static_cast<unsigned long long>(2 * i + 1));
        } else {
            dbr = __ddiv_rn(static_cast<double>(a.b.tgap[i]), __dmul_rn(static_cast<double>(tmax), nd));
            abr = __ddiv_rn(static_cast<double>(a.b.agap[i]), __dmul_rn(static_cast<double>(amax), nd));
        }
        acc.dbr += dbr;
        acc.abr += abr;
        if (a.simulate) acc.seconds += a.b.busy[i];
    }
    block_reduce_partial(acc, partials + blockIdx.x);
}

}  // namespace

void eval_columns(Ctx& c, const PlanArrays& p, const std::vector<hbp_group_config>& groups,
                  const hbp_hardware_profile* profile, int phase, int32_t c0, int32_t c1,
                  const hbp_eval_columns_bufs& b) {
    cudaStream_t s = c.stream;
    if (profile) {
        const int pc = cm_profile_check(*profile);
        if (pc) fail_validation(cm_profile_message(pc));
    }
    if (p.I == 0) fail_validation("metrics report: empty plan");
    DevBuf<hbp_group_config> dg(groups.size(), s);
    CUDA_CHECK(cudaMemcpyAsync(dg.p, groups.data(), sizeof(hbp_group_config) * groups.size(), cudaMemcpyHostToDevice, s));
    ColArgs a{p, dg.p, profile != nullptr, profile ? *profile : hbp_hardware_profile{}, c0, c1, b};
    const int grid = static_cast<int>(std::min<i64>(EG, (p.I + EB - 1) / EB));
    if (phase == 0) {
        if (b.sim_err) CUDA_CHECK(cudaMemsetAsync(b.sim_err, 0x7f, sizeof(int64_t), s));  // "none" = large
        LAUNCH(k_cols_phase0, grid, EB, 0, s, a);
    } else {
        LAUNCH(k_cols_phase1, grid, EB, 0, s, a);
    }
    CUDA_CHECK(cudaStreamSynchronize(s));
}

void eval_columns_finish(Ctx& c, const PlanArrays& p, int32_t device_count,
                         const std::vector<hbp_group_config>& groups, const hbp_hardware_profile* profile,
                         const hbp_eval_columns_bufs& b, EvalOut& out) {
    cudaStream_t s = c.stream;
    if (p.I == 0) fail_validation("metrics report: empty plan");
    DevBuf<hbp_group_config> dg(groups.size(), s);
    CUDA_CHECK(cudaMemcpyAsync(dg.p, groups.data(), sizeof(hbp_group_config) * groups.size(), cudaMemcpyHostToDevice, s));
    DevBuf<Partial> partials(EG + 1, s);
    DevBuf<unsigned long long> errs(1, s);
    CUDA_CHECK(cudaMemsetAsync(errs.p, 0xff, sizeof(unsigned long long), s));
    ColArgs a{p, dg.p, profile != nullptr, profile ? *profile : hbp_hardware_profile{}, 0, 0, b};
    const int grid = static_cast<int>(std::min<i64>(EG, (p.I + EB - 1) / EB));
    LAUNCH(k_cols_finish, grid, EB, 0, s, a, partials.p, errs.p);
    LAUNCH(k_eval_final, 1, 32, 0, s, partials.p, grid, partials.p + EG);
    const auto e = read_vector(c, errs.p, 1);
    if (e[0] != ~0ull) {
        const i64 i = static_cast<i64>(e[0] >> 1);
        const bool abr = e[0] & 1;
        const auto offs = read_vector(c, p.iter_dev_offsets + i, 2);
        if (!abr && offs[1] == offs[0]) fail_validation("dbr: no devices");
        fail_validation(abr ? "abr undefined: all devices carry zero attention"
                            : "dbr undefined: all devices carry zero tokens");
    }
    if (profile && b.sim_err) {
        const int64_t key = read_vector(c, b.sim_err, 1)[0];
        if (key != 0x7f7f7f7f7f7f7f7fll) {
            const i64 i = static_cast<i64>(static_cast<u64>(key) >> 20);
            const i64 dd = static_cast<i64>(static_cast<u64>(key) & 0xfffff);
            const int g = read_vector(c, p.iter_group + i, 1)[0];
            const hbp_group_config cfg = groups.at(static_cast<size_t>(g));
            if (cfg.sp < 1) fail_validation("sp must be >= 1");
            if (cfg.ckpt < 0 || cfg.ckpt > profile->layer_count) fail_validation("ckpt must lie in [0, layer_count]");
            const i64 d = read_vector(c, p.iter_dev_offsets + i, 1)[0] + dd;
            const auto po = read_vector(c, p.dev_pack_offsets + d, 2);
            const auto caps = read_vector(c, p.pack_capacity + po[0], static_cast<size_t>(po[1] - po[0]));
            int64_t maxcap = 0;
            for (auto v : caps) maxcap = v > maxcap ? v : maxcap;
            const int64_t used = cm_memory_used(maxcap, cfg.sp, cfg.ckpt, *profile);
            fail_infeasible("iteration " + std::to_string(i) + ": configuration sp=" + std::to_string(cfg.sp) +
                            " ckpt=" + std::to_string(cfg.ckpt) + " at length " + std::to_string(maxcap) +
                            " requires " + std::to_string(used) + " bytes, " + std::to_string(profile->device_memory) +
                            " available");
        }
    }
    const Partial tot = read_scalar(c, partials.p + EG);
    const double ni = static_cast<double>(p.I);
    const double total = static_cast<double>(tot.tokens);
    const double comm = static_cast<double>(tot.comm);
    const double pad_gap = static_cast<double>(tot.pad_gap);
    const double pad_cap = static_cast<double>(tot.pad_cap);
    out.m.dbr = tot.dbr / ni;
    out.m.abr = tot.abr / ni;
    out.m.cr = total > 0.0 ? comm / total : 0.0;
    out.m.pr = pad_cap > 0.0 ? pad_gap / pad_cap : 0.0;
    out.m.ave_t = total / (ni * static_cast<double>(device_count));
    out.total_seconds = tot.seconds;
    out.switch_count = static_cast<int32_t>(tot.switches);
}

}  // namespace hbp_b200
