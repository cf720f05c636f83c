// metrics.cu — report() and simulate() over a flat plan in HBM.
//
// Reference: dbr / abr / report (src/metrics.cpp:22-144), device_work /
// iter_time (src/costmodel.cpp:55-104), simulate (src/sim.cpp:9-60) and
// switch_count (src/schedule.cpp:67-79). One thread owns one iteration and
// walks its devices in order, so every per-iteration DBR / ABR / time is
// computed with the reference's operation order (bit-identical). The
// run-level sums use a fixed-shape reduction (per-thread, per-block, then
// one block in order): deterministic, and within 1e-15 relative of the
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
    __shared__ Partial s[EB];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int w = EB / 2; w > 0; w >>= 1) {
        if (threadIdx.x < static_cast<unsigned>(w)) add_partial(s[threadIdx.x], s[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) a.partials[blockIdx.x] = s[0];
}

__global__ void k_eval_final(const Partial* __restrict__ partials, int n, Partial* __restrict__ out) {
    if (threadIdx.x != 0) return;
    Partial acc{0, 0, 0, 0, 0, 0, 0, 0};
    for (int b = 0; b < n; ++b) add_partial(acc, partials[b]);
    *out = acc;
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

}  // namespace hbp_b200
