// schedule.cu — the step after the plan: curriculum
// ordering, runtime assignment and the schedule CSV, on device plans.
//
// Reference: curriculum_order (src/schedule.cpp:10-63): iterations of groups
// below the cutoff are "short"; Rng(derive_seed(seed, "curriculum"))
// shuffles the short list, the first warmup_iterations of it become the
// warmup phase, and the SAME generator then shuffles the rest (remaining
// short ones followed by the long ones). Both shuffles are the exact
// parallel Fisher-Yates of shuffle.cu, the second starting at the draw the
// first stopped at. The plan is then a permutation of iterations: devices,
// packs and members are regathered level by level (scan of segment sizes,
// then one thread per segment). assign_runtime (schedule.cpp:65-77) and
// write_schedule_csv (schedule.cpp:79-89) read the groups' configs per
// iteration.
#include <algorithm>
#include <cstring>
#include <string>

#include "../../include/hbp_b200.h"
#include "engine.cuh"
#include "pipeline.cuh"
#include "rng.cuh"

using namespace hbp_b200;

namespace {

constexpr unsigned kSB = 256;
inline unsigned GS(u64 n) { return grid_for(n, kSB, 148u * 16u); }

template <typename F>
__global__ void k_each(u64 n, F f) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<u64>(gridDim.x) * blockDim.x)
        f(i);
}
template <typename F>
void each(Ctx& c, u64 n, F f, const char* name = "schedule") {
    if (n) LAUNCH_B(name, 0.0, k_each<F>, GS(n), kSB, 0, c.stream, n, f);
}

// exclusive prefix of sizes[k] (k < n) into off[0..n]
void offsets_of(Ctx& c, const int64_t* sizes, u64 n, int64_t* off) {
    const i64 nn = static_cast<i64>(n);
    scan_exclusive<u64>(
        nn + 1, [=] __device__(i64 i) { return i < nn ? static_cast<u64>(sizes[i]) : 0ull; },
        [=] __device__(i64 i, u64 v) { off[i] = static_cast<int64_t>(v); }, c.stream, c.scan, "scan.sched1");
}

}  // namespace

namespace hbp_b200 {

// New plan = the iterations of `in` in `order` (device array, n_iterations
// entries), phases `phase` (device, may be null).
void reorder_iterations(Ctx& c, const DevicePlan& in, const u32* order, const int8_t* phase, DevicePlan& out) {
    cudaStream_t s = c.stream;
    const u64 I = static_cast<u64>(in.n_iterations), D = static_cast<u64>(in.n_devices),
              P = static_cast<u64>(in.n_packs), M = static_cast<u64>(in.n_members);
    out.device_count = in.device_count;
    out.seed = in.seed;
    out.groups = in.groups;
    out.l_best = in.l_best;
    out.l_max = in.l_max;
    out.n_iterations = in.n_iterations;
    out.n_devices = in.n_devices;
    out.n_packs = in.n_packs;
    out.n_members = in.n_members;
    out.iter_group.alloc(I + 1, s);
    out.iter_dev_offsets.alloc(I + 1, s);
    out.dev_index.alloc(D + 1, s);
    out.dev_pack_offsets.alloc(D + 1, s);
    out.pack_capacity.alloc(P + 1, s);
    out.pack_total.alloc(P + 1, s);
    out.pack_attention.alloc(P + 1, s);
    out.pack_member_offsets.alloc(P + 1, s);
    out.member_index.alloc(M + 1, s);
    out.iter_phase.alloc(I + 1, s);
    const int32_t* ig = in.iter_group.p;
    const int64_t* ido = in.iter_dev_offsets.p;
    const int32_t* di = in.dev_index.p;
    const int64_t* dpo = in.dev_pack_offsets.p;
    const int64_t *pc = in.pack_capacity.p, *pt = in.pack_total.p, *pa = in.pack_attention.p,
                  *pmo = in.pack_member_offsets.p;
    const int32_t* mi = in.member_index.p;
    int32_t* oig = out.iter_group.p;
    int64_t* oido = out.iter_dev_offsets.p;
    int32_t* odi = out.dev_index.p;
    int64_t* odpo = out.dev_pack_offsets.p;
    int64_t *opc = out.pack_capacity.p, *opt = out.pack_total.p, *opa = out.pack_attention.p,
            *opmo = out.pack_member_offsets.p;
    int32_t* omi = out.member_index.p;
    int8_t* oph = out.iter_phase.p;
    // iterations
    DevBuf<int64_t> sz(std::max(std::max(I, D), P) + 1, s);
    int64_t* szp = sz.p;
    each(c, I, [=] __device__(u64 k) {
        const u32 o = order[k];
        oig[k] = ig[o];
        oph[k] = phase ? phase[k] : 0;
        szp[k] = ido[o + 1] - ido[o];
    });
    if (I) offsets_of(c, szp, I, oido);
    else CUDA_CHECK(cudaMemsetAsync(oido, 0, sizeof(int64_t), s));
    // devices (one thread per new iteration) -> old device of every new one
    DevBuf<int64_t> dmap(D + 1, s);
    int64_t* dm = dmap.p;
    each(c, I, [=] __device__(u64 k) {
        const u32 o = order[k];
        for (int64_t t = 0; t < ido[o + 1] - ido[o]; ++t) {
            const int64_t nd = oido[k] + t, od = ido[o] + t;
            dm[nd] = od;
            odi[nd] = di[od];
        }
    });
    each(c, D, [=] __device__(u64 g) { szp[g] = dpo[dm[g] + 1] - dpo[dm[g]]; });
    if (D) offsets_of(c, szp, D, odpo);
    else CUDA_CHECK(cudaMemsetAsync(odpo, 0, sizeof(int64_t), s));
    // packs (one thread per new device)
    DevBuf<int64_t> pmap(P + 1, s);
    int64_t* pm = pmap.p;
    each(c, D, [=] __device__(u64 g) {
        const int64_t od = dm[g];
        for (int64_t t = 0; t < dpo[od + 1] - dpo[od]; ++t) {
            const int64_t np = odpo[g] + t, op = dpo[od] + t;
            pm[np] = op;
            opc[np] = pc[op];
            opt[np] = pt[op];
            opa[np] = pa[op];
        }
    });
    each(c, P, [=] __device__(u64 q) { szp[q] = pmo[pm[q] + 1] - pmo[pm[q]]; });
    if (P) offsets_of(c, szp, P, opmo);
    else CUDA_CHECK(cudaMemsetAsync(opmo, 0, sizeof(int64_t), s));
    // members (one thread per new pack)
    each(c, P, [=] __device__(u64 q) {
        const int64_t op = pm[q];
        for (int64_t t = 0; t < pmo[op + 1] - pmo[op]; ++t) omi[opmo[q] + t] = mi[pmo[op] + t];
    });
    CUDA_CHECK(cudaStreamSynchronize(s));
}

void curriculum_device(Ctx& c, const DevicePlan& in, int32_t warmup, int32_t cutoff, DevicePlan& out) {
    if (warmup < 0) fail_validation("warmup_iterations must be >= 0");
    if (cutoff < 1 || cutoff > static_cast<int32_t>(in.groups.size()))
        fail_validation("short_group_cutoff must select at least one group and at most all of them");
    cudaStream_t s = c.stream;
    const u64 I = static_cast<u64>(in.n_iterations);
    // stable split: short iterations, then long ones
    DevBuf<u32> lists(I + 1, s), cnt(1, s);
    const int32_t* ig = in.iter_group.p;
    u32* lp = lists.p;
    u32* cp = cnt.p;
    u64 n_short = 0;
    if (I) {
        const i64 II = static_cast<i64>(I);
        scan_exclusive<u32>(
            II, [=] __device__(i64 i) { return ig[i] < cutoff ? 1u : 0u; },
            [=] __device__(i64 i, u32 v) {
                const bool sh = ig[i] < cutoff;
                if (sh) lp[v] = static_cast<u32>(i);
                if (i == II - 1) *cp = v + (sh ? 1u : 0u);
            },
            s, c.scan, "scan.sched2");
        n_short = read_scalar(c, cnt.p);
        const u64 ns = n_short;
        scan_exclusive<u32>(
            II, [=] __device__(i64 i) { return ig[i] < cutoff ? 0u : 1u; },
            [=] __device__(i64 i, u32 v) {
                if (!(ig[i] < cutoff)) lp[ns + v] = static_cast<u32>(i);
            },
            s, c.scan, "scan.sched3");
    }
    if (n_short < static_cast<u64>(warmup))
        fail_validation("curriculum needs " + std::to_string(warmup) + " short-group iterations but the plan has only " +
                        std::to_string(n_short));
    const uint64_t seed = derive_seed(in.seed, "curriculum");
    const u64 W = static_cast<u64>(warmup), R = I - W;
    DevBuf<u32> src(I + 1, s), order(I + 1, s), rest(R + 1, s);
    uint64_t used = 0;
    u32* sp = src.p;
    u32* op = order.p;
    u32* rp = rest.p;
    // shuffle(short_idx): order[0 .. n_short) = shuffled short list
    if (n_short > 0) {
        fy_source_positions(c, seed, static_cast<i64>(n_short), src.p, 0, &used);
        each(c, n_short, [=] __device__(u64 p) { op[p] = lp[sp[p]]; });
    }
    // rest = shuffled_short[W:] ++ long_idx, shuffled by the same generator
    each(c, R, [=] __device__(u64 p) { rp[p] = p < n_short - W ? op[W + p] : lp[n_short + (p - (n_short - W))]; });
    if (R > 0) {
        fy_source_positions(c, seed, static_cast<i64>(R), src.p, used, nullptr);
        each(c, R, [=] __device__(u64 p) { op[W + p] = rp[sp[p]]; });
    }
    DevBuf<int8_t> phase(I + 1, s);
    int8_t* ph = phase.p;
    each(c, I, [=] __device__(u64 k) { ph[k] = k < W ? 1 : 0; });
    reorder_iterations(c, in, order.p, phase.p, out);
}

}  // namespace hbp_b200

namespace {

struct CsvArgs {
    const int32_t* iter_group;
    const int8_t* phase;
    const hbp_group_config* groups;  // device copy
    int64_t n;
};

__host__ __device__ __forceinline__ u32 ndig(int64_t v) {
    u64 u = v < 0 ? 0ull - static_cast<u64>(v) : static_cast<u64>(v);
    u32 d = 1;
    u64 p = 10;
    while (d < 20 && u >= p) {
        ++d;
        p *= 10;
    }
    return d + (v < 0 ? 1 : 0);
}

__device__ __forceinline__ char* put_num(char* p, int64_t v) {
    u64 u = v < 0 ? 0ull - static_cast<u64>(v) : static_cast<u64>(v);
    if (v < 0) *p++ = '-';
    const u32 d = ndig(static_cast<int64_t>(u));
    for (u32 k = d; k-- > 0;) {
        p[k] = static_cast<char>('0' + u % 10);
        u /= 10;
    }
    return p + d;
}

// "i,group,sp,ckpt,phase\n" (schedule.cpp:82-88)
template <bool WRITE>
__device__ u64 csv_row(const CsvArgs& a, int64_t i, char* out) {
    const int32_t g = a.iter_group[i];
    const hbp_group_config& cfg = a.groups[g];
    const bool warm = a.phase && a.phase[i];
    const u64 n = ndig(i) + 1 + ndig(g) + 1 + ndig(cfg.sp) + 1 + ndig(cfg.ckpt) + 1 + 6 + 1;
    if (WRITE) {
        char* p = put_num(out, i);
        *p++ = ',';
        p = put_num(p, g);
        *p++ = ',';
        p = put_num(p, cfg.sp);
        *p++ = ',';
        p = put_num(p, cfg.ckpt);
        *p++ = ',';
        const char* ph = warm ? "warmup" : "hybrid";
        for (int k = 0; k < 6; ++k) *p++ = ph[k];
        *p = '\n';
    }
    return n;
}

__global__ void k_csv_len(CsvArgs a, u64* len) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < a.n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        len[i] = csv_row<false>(a, i, nullptr);
}
__global__ void k_csv_write(CsvArgs a, const u64* off, char* out) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < a.n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        csv_row<true>(a, i, out + off[i]);
}

template <typename F>
int sched_guarded(hbp_ctx* ctx, F&& fn) {
    if (ctx == nullptr) return HBP_ERR_VALIDATION;
    try {
        CtxScope scope(*ctx);
        fn();
        ctx->last_error.clear();
        return HBP_OK;
    } catch (const EngineError& e) {
        ctx->last_error = e.what();
        if (e.code == HBP_ERR_CUDA) cudaGetLastError();
        return e.code;
    } catch (const std::exception& e) {
        ctx->last_error = e.what();
        return HBP_ERR_CUDA;
    }
}

}  // namespace

// defined in capi.cu
hbp_plan* hbp_b200_new_plan(hbp_ctx* ctx);
void hbp_b200_delete_plan(hbp_plan* p);

extern "C" int hbp_curriculum_order(hbp_ctx* ctx, hbp_plan* plan, int32_t warmup_iterations,
                                    int32_t short_group_cutoff, hbp_plan** out) {
    return sched_guarded(ctx, [&] {
        *out = nullptr;
        if (plan == nullptr) fail_validation("null plan");
        if (!plan->dp.iter_group.p && plan->dp.n_iterations > 0)
            fail_validation("curriculum_order: the plan's device arrays are gone");
        hbp_plan* p = hbp_b200_new_plan(ctx);
        try {
            curriculum_device(*ctx, plan->dp, warmup_iterations, short_group_cutoff, p->dp);
        } catch (...) {
            hbp_b200_delete_plan(p);
            throw;
        }
        *out = p;
    });
}

extern "C" int hbp_assign_runtime(hbp_ctx* ctx, hbp_plan* plan, int32_t* sp, int32_t* ckpt, int64_t* switch_count) {
    return sched_guarded(ctx, [&] {
        if (plan == nullptr) fail_validation("null plan");
        const DevicePlan& dp = plan->dp;
        cudaStream_t s = ctx->stream;
        const u64 I = static_cast<u64>(dp.n_iterations);
        *switch_count = 0;
        if (I == 0) return;
        DevBuf<hbp_group_config> g(dp.groups.size(), s);
        CUDA_CHECK(cudaMemcpyAsync(g.p, dp.groups.data(), sizeof(hbp_group_config) * dp.groups.size(),
                                   cudaMemcpyHostToDevice, s));
        DevBuf<int32_t> dsp(I, s), dck(I, s);
        DevBuf<unsigned long long> sw(1, s);
        sw.zero();
        const int32_t* ig = dp.iter_group.p;
        const hbp_group_config* gp = g.p;
        int32_t* a = dsp.p;
        int32_t* b = dck.p;
        unsigned long long* swp = sw.p;
        // per-iteration RuntimeConfig, and changes between consecutive ones
        // (RuntimeConfig::operator== compares sp and ckpt)
        each(*ctx, I, [=] __device__(u64 i) {
            const hbp_group_config& c0 = gp[ig[i]];
            a[i] = c0.sp;
            b[i] = c0.ckpt;
            if (i > 0) {
                const hbp_group_config& cp = gp[ig[i - 1]];
                if (cp.sp != c0.sp || cp.ckpt != c0.ckpt) atomicAdd(swp, 1ull);
            }
        });
        CUDA_CHECK(cudaMemcpyAsync(sp, dsp.p, sizeof(int32_t) * I, cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaMemcpyAsync(ckpt, dck.p, sizeof(int32_t) * I, cudaMemcpyDeviceToHost, s));
        *switch_count = static_cast<int64_t>(read_scalar(*ctx, sw.p));
    });
}

extern "C" int hbp_schedule_csv(hbp_ctx* ctx, hbp_plan* plan, char* out, int64_t capacity, int64_t* out_len) {
    return sched_guarded(ctx, [&] {
        if (plan == nullptr) fail_validation("null plan");
        const DevicePlan& dp = plan->dp;
        cudaStream_t s = ctx->stream;
        static const char kHead[] = "iteration,group,sp,ckpt,phase\n";
        const u64 H = sizeof(kHead) - 1, I = static_cast<u64>(dp.n_iterations);
        u64 body = 0;
        DevBuf<hbp_group_config> g(dp.groups.size() + 1, s);
        if (!dp.groups.empty())
            CUDA_CHECK(cudaMemcpyAsync(g.p, dp.groups.data(), sizeof(hbp_group_config) * dp.groups.size(),
                                       cudaMemcpyHostToDevice, s));
        CsvArgs a{dp.iter_group.p, dp.iter_phase.p, g.p, static_cast<int64_t>(I)};
        DevBuf<u64> len(I + 1, s), off(I + 1, s);
        if (I) {
            LAUNCH(k_csv_len, GS(I), kSB, 0, s, a, len.p);
            const u64* lp = len.p;
            u64* opp = off.p;
            const i64 II = static_cast<i64>(I);
            scan_exclusive<u64>(
                II + 1, [=] __device__(i64 i) { return i < II ? lp[i] : 0ull; },
                [=] __device__(i64 i, u64 v) { opp[i] = v; }, s, ctx->scan);
            body = read_scalar(*ctx, off.p + I);
        }
        *out_len = static_cast<int64_t>(H + body);
        if (out == nullptr) return;
        if (capacity < static_cast<int64_t>(H + body))
            fail_validation("schedule_csv: output buffer of " + std::to_string(capacity) + " bytes, the schedule needs " +
                            std::to_string(H + body));
        std::memcpy(out, kHead, H);
        if (body) {
            DevBuf<char> text(body, s);
            LAUNCH(k_csv_write, GS(I), kSB, 0, s, a, off.p, text.p);
            CUDA_CHECK(cudaMemcpyAsync(out + H, text.p, body, cudaMemcpyDeviceToHost, s));
        }
        CUDA_CHECK(cudaStreamSynchronize(s));
    });
}
