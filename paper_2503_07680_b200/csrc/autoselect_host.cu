// autoselect_host.cu — C-ABI for the profilers and group auto-selection.
// The decisions run on the GPU (autoselect.cu); this file validates inputs
// exactly where the reference constructors do and turns the recorded
// failure events into the reference's exception messages, in the order the
// reference would concatenate them (costmodel.cpp:294-325,
// autoselect.cpp:76-168).
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hbp_b200.h"
#include "autoselect.cuh"
#include "costmodel.cuh"

namespace hbp_b200 {

std::string as_message(const AsErr& e) {
    const std::string L = std::to_string(e.length), S = std::to_string(e.sp), Ck = std::to_string(e.ckpt);
    switch (e.code) {
        case AS_V_SP: return "sp must be >= 1";
        case AS_V_CKPT: return "ckpt must lie in [0, layer_count]";
        case AS_V_GREEDY: return "greedy_profile_ckpt: ckpt_min must be < ckpt_max";
        case AS_I_SLOPE:
            return "GC does not reduce memory under this profile (slope " + std::to_string(e.slope) + " bytes/layer)";
        case AS_I_NOROW: return "no profile row for length " + L + ", sp " + S;
        case AS_I_OOMROW: return "profiled configuration is out of memory at length " + L + ", sp " + S;
        case AS_I_NOROW_CKPT: return "no profile row for length " + L + ", sp " + S + ", ckpt " + Ck;
        case AS_I_NOFIT: return "sp=" + S + " does not fit device memory even at ckpt " + Ck;
        default: return "unknown auto-selection failure";
    }
}

bool as_is_validation(int code) { return code == AS_V_SP || code == AS_V_CKPT || code == AS_V_GREEDY; }

namespace {

std::string as_message_mem(const AsErr& e, int64_t device_memory) {
    if (e.code != AS_I_MEM) return as_message(e);
    return "configuration sp=" + std::to_string(e.sp) + " ckpt=" + std::to_string(e.ckpt) + " at length " +
           std::to_string(e.length) + " requires " + std::to_string(e.used) + " bytes, " +
           std::to_string(device_memory) + " available";
}

[[noreturn]] void throw_as(const AsErr& e, int64_t device_memory) {
    const std::string m = as_message_mem(e, device_memory);
    if (as_is_validation(e.code)) fail_validation(m);
    fail_infeasible(m);
}

// "no feasible (sp, ckpt) for length L: sp=a: ...; sp=b: ..."
std::string best_failure(int64_t l, const std::vector<int32_t>& sps, const AsErr* fails, int64_t device_memory) {
    std::string f;
    for (size_t k = 0; k < sps.size(); ++k) {
        if (fails[k].code == AS_OK) continue;
        if (!f.empty()) f += "; ";
        f += "sp=" + std::to_string(sps[k]) + ": " + as_message_mem(fails[k], device_memory);
    }
    return "no feasible (sp, ckpt) for length " + std::to_string(l) + ": " + f;
}

int64_t devmem_of(const DevProfiler& p) {
    return p.kind == HBP_PROFILER_ANALYTIC ? p.profile.device_memory : p.device_memory;
}

}  // namespace

void upload_profiler(Ctx& c, const hbp_profiler* in, DeviceProfilerHolder& out) {
    if (in == nullptr) fail_validation("null profiler");
    DevProfiler p{};
    p.kind = in->kind;
    if (in->kind == HBP_PROFILER_ANALYTIC) {
        // AnalyticProfiler constructor (costmodel.cpp:110-121)
        const int pc = cm_profile_check(in->profile);
        if (pc) fail_validation(cm_profile_message(pc));
        p.profile = in->profile;
        p.ckpt_min = in->ckpt_min;
        p.ckpt_max = in->ckpt_max < 0 ? in->profile.layer_count : in->ckpt_max;
        if (p.ckpt_min < 0 || p.ckpt_min >= p.ckpt_max || p.ckpt_max > in->profile.layer_count)
            fail_validation("ckpt probe bounds must satisfy 0 <= ckpt_min < ckpt_max <= layer_count");
        p.device_memory = in->profile.device_memory;
    } else if (in->kind == HBP_PROFILER_TABLE) {
        // TableProfiler constructor (costmodel.cpp:144-156)
        for (int64_t i = 0; i < in->n_rows; ++i)
            for (int64_t j = 0; j < i; ++j)
                if (in->rows[i].length == in->rows[j].length && in->rows[i].sp == in->rows[j].sp)
                    fail_validation("duplicate profile row for length " + std::to_string(in->rows[i].length) +
                                    ", sp " + std::to_string(in->rows[i].sp));
        p.device_memory = in->device_memory;
        p.n_rows = in->n_rows;
        out.rows.alloc(static_cast<size_t>(in->n_rows) + 1, c.stream);
        if (in->n_rows)
            CUDA_CHECK(cudaMemcpyAsync(out.rows.p, in->rows, sizeof(hbp_profile_row) * in->n_rows,
                                       cudaMemcpyHostToDevice, c.stream));
        p.rows = out.rows.p;
    } else {
        fail_validation("unknown profiler kind");
    }
    out.host = p;
    out.dev.alloc(1, c.stream);
    CUDA_CHECK(cudaMemcpyAsync(out.dev.p, &out.host, sizeof(DevProfiler), cudaMemcpyHostToDevice, c.stream));
}

namespace {

AsQuery run_one(Ctx& c, DeviceProfilerHolder& h, AsQuery q, std::vector<AsErr>* fails = nullptr,
                const std::vector<int32_t>* sps = nullptr) {
    DevBuf<AsQuery> dq(1, c.stream);
    DevBuf<int32_t> dsp;
    DevBuf<AsErr> dfail;
    if (sps) {
        dsp.alloc(sps->size() + 1, c.stream);
        dfail.alloc(sps->size() + 1, c.stream);
        if (!sps->empty())
            CUDA_CHECK(cudaMemcpyAsync(dsp.p, sps->data(), sizeof(int32_t) * sps->size(), cudaMemcpyHostToDevice,
                                       c.stream));
        q.sps = dsp.p;
        q.n_sp = static_cast<int32_t>(sps->size());
        q.fails = dfail.p;
    }
    CUDA_CHECK(cudaMemcpyAsync(dq.p, &q, sizeof(q), cudaMemcpyHostToDevice, c.stream));
    run_queries(c, h.dev.p, dq.p, 1);
    AsQuery r = read_scalar(c, dq.p);
    if (fails && sps) *fails = read_vector(c, dfail.p, sps->size());
    return r;
}

}  // namespace

SelectResult select_groups_device(Ctx& c, const hbp_profiler* prof, const std::vector<int64_t>& lengths,
                                  const std::vector<int32_t>& sps) {
    // argument checks (autoselect.cpp:79-93), in the reference's order
    if (lengths.empty()) fail_validation("select_groups: no candidate lengths");
    for (size_t i = 1; i < lengths.size(); ++i)
        if (lengths[i] <= lengths[i - 1]) fail_validation("candidate lengths must be strictly ascending");
    for (const int32_t sp : sps)
        if (!(sp > 0 && (sp & (sp - 1)) == 0))
            fail_validation("sp candidates must be powers of two, got " + std::to_string(sp));
    DeviceProfilerHolder h;
    upload_profiler(c, prof, h);
    cudaStream_t s = c.stream;
    const size_t nl = lengths.size(), ns = sps.size();
    DevBuf<int64_t> dl(nl, s);
    DevBuf<int32_t> dsp(ns + 1, s);
    DevBuf<uint8_t> ok(nl, s);
    DevBuf<int32_t> bsp(nl, s), bck(nl, s);
    DevBuf<double> bsec(nl, s);
    DevBuf<AsErr> fails(nl * ns + 1, s);
    CUDA_CHECK(cudaMemcpyAsync(dl.p, lengths.data(), sizeof(int64_t) * nl, cudaMemcpyHostToDevice, s));
    if (ns) CUDA_CHECK(cudaMemcpyAsync(dsp.p, sps.data(), sizeof(int32_t) * ns, cudaMemcpyHostToDevice, s));
    AsProblem P{};
    P.profiler = h.dev.p;
    P.lengths = dl.p;
    P.n_lengths = static_cast<int32_t>(nl);
    P.sps = dsp.p;
    P.n_sp = static_cast<int32_t>(ns);
    P.length_ok = ok.p;
    P.best_sp = bsp.p;
    P.best_ckpt = bck.p;
    P.best_sec = bsec.p;
    P.fails = fails.p;
    DevBuf<AsProblem> dp(1, s);
    CUDA_CHECK(cudaMemcpyAsync(dp.p, &P, sizeof(P), cudaMemcpyHostToDevice, s));
    run_select_problems(c, dp.p, 1);
    const AsProblem R = read_scalar(c, dp.p);
    const int64_t devmem = devmem_of(h.host);
    if (R.status == AS_S_NONE || R.status == AS_S_LARGEST) {
        const auto okv = read_vector(c, ok.p, nl);
        const auto fv = read_vector(c, fails.p, nl * ns);
        std::string f;
        for (size_t i = 0; i < nl; ++i) {
            if (okv[i]) continue;
            if (!f.empty()) f += "; ";
            f += ns == 0 ? std::string("find_best_sp_ckpt: no sp candidates")
                         : best_failure(lengths[i], sps, fv.data() + i * ns, devmem);
        }
        if (R.status == AS_S_NONE) fail_infeasible("no candidate length is feasible: " + f);
        fail_infeasible("largest candidate length " + std::to_string(lengths.back()) + " is infeasible: " + f);
    }
    if (R.status == AS_S_STAGE2) throw_as(R.stage2, devmem);
    if (R.status == AS_S_MID)
        fail_infeasible("no feasible sp for mid-level group of length " + std::to_string(R.stage2.length));
    SelectResult out;
    out.groups.assign(R.out, R.out + R.n_out);
    out.l_best = R.l_best;
    out.l_max = R.l_max;
    // HierarchicalGroups::validate (autoselect.cpp:18-33)
    int64_t prev = 0;
    for (const auto& g : out.groups) {
        if (g.length <= prev) fail_validation("group lengths must be strictly increasing");
        if (g.sp < 1 || g.ckpt < 0) fail_validation("invalid group runtime config");
        prev = g.length;
    }
    return out;
}

}  // namespace hbp_b200

using namespace hbp_b200;

namespace {
template <typename F>
int as_guarded(hbp_ctx* ctx, F&& fn) {
    if (ctx == nullptr) return HBP_ERR_VALIDATION;
    try {
        CtxScope scope(*ctx);
        fn();
        ctx->last_error.clear();
        return HBP_OK;
    } catch (const EngineError& e) {
        ctx->last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        ctx->last_error = e.what();
        return HBP_ERR_CUDA;
    }
}

void query_or_throw(hbp_ctx* ctx, DeviceProfilerHolder& h, const AsQuery& r) {
    (void)ctx;
    if (r.err.code != AS_OK) throw_as(r.err, devmem_of(h.host));
}
}  // namespace

extern "C" {

int hbp_profiler_time(hbp_ctx* ctx, const hbp_profiler* profiler, int64_t length, int32_t sp, int32_t ckpt,
                      double* out) {
    return as_guarded(ctx, [&] {
        DeviceProfilerHolder h;
        upload_profiler(*ctx, profiler, h);
        AsQuery q{};
        q.op = AS_Q_TIME;
        q.length = length;
        q.sp = sp;
        q.ckpt = ckpt;
        const AsQuery r = run_one(*ctx, h, q);
        query_or_throw(ctx, h, r);
        *out = r.out_sec;
    });
}

int hbp_profiler_memory(hbp_ctx* ctx, const hbp_profiler* profiler, int64_t length, int32_t sp, int32_t ckpt,
                        int64_t* out) {
    return as_guarded(ctx, [&] {
        DeviceProfilerHolder h;
        upload_profiler(*ctx, profiler, h);
        AsQuery q{};
        q.op = AS_Q_MEMORY;
        q.length = length;
        q.sp = sp;
        q.ckpt = ckpt;
        const AsQuery r = run_one(*ctx, h, q);
        query_or_throw(ctx, h, r);
        *out = r.out_mem;
    });
}

int hbp_profiler_derive_ckpt(hbp_ctx* ctx, const hbp_profiler* profiler, int64_t length, int32_t sp, int32_t* out) {
    return as_guarded(ctx, [&] {
        DeviceProfilerHolder h;
        upload_profiler(*ctx, profiler, h);
        AsQuery q{};
        q.op = AS_Q_DERIVE;
        q.length = length;
        q.sp = sp;
        const AsQuery r = run_one(*ctx, h, q);
        query_or_throw(ctx, h, r);
        *out = r.out_ckpt;
    });
}

int hbp_greedy_profile_ckpt(hbp_ctx* ctx, const hbp_profiler* profiler, int64_t length, int32_t sp, int32_t ckpt_min,
                            int32_t ckpt_max, int32_t* out) {
    return as_guarded(ctx, [&] {
        DeviceProfilerHolder h;
        upload_profiler(*ctx, profiler, h);
        AsQuery q{};
        q.op = AS_Q_GREEDY;
        q.length = length;
        q.sp = sp;
        q.ckpt_min = ckpt_min;
        q.ckpt_max = ckpt_max;
        const AsQuery r = run_one(*ctx, h, q);
        query_or_throw(ctx, h, r);
        *out = r.out_ckpt;
    });
}

int hbp_find_best_sp_ckpt(hbp_ctx* ctx, const hbp_profiler* profiler, int64_t length, const int32_t* sp_candidates,
                          int32_t n_sp, int32_t* out_sp, int32_t* out_ckpt, double* out_seconds) {
    return as_guarded(ctx, [&] {
        if (n_sp <= 0) fail_validation("find_best_sp_ckpt: no sp candidates");
        DeviceProfilerHolder h;
        upload_profiler(*ctx, profiler, h);
        const std::vector<int32_t> sps(sp_candidates, sp_candidates + n_sp);
        AsQuery q{};
        q.op = AS_Q_BEST;
        q.length = length;
        std::vector<AsErr> fails;
        const AsQuery r = run_one(*ctx, h, q, &fails, &sps);
        if (!r.ok) fail_infeasible(best_failure(length, sps, fails.data(), devmem_of(h.host)));
        *out_sp = r.out_sp;
        *out_ckpt = r.out_ckpt;
        *out_seconds = r.out_sec;
    });
}

int hbp_select_groups(hbp_ctx* ctx, const int64_t* candidate_lengths, int32_t n_lengths, const hbp_profiler* profiler,
                      const int32_t* sp_candidates, int32_t n_sp, hbp_group_config* out_groups, int32_t* out_count,
                      int64_t* out_l_best, int64_t* out_l_max) {
    return as_guarded(ctx, [&] {
        const std::vector<int64_t> ls(candidate_lengths, candidate_lengths + (n_lengths > 0 ? n_lengths : 0));
        const std::vector<int32_t> sps(sp_candidates, sp_candidates + (n_sp > 0 ? n_sp : 0));
        const SelectResult r = select_groups_device(*ctx, profiler, ls, sps);
        for (size_t i = 0; i < r.groups.size(); ++i) out_groups[i] = r.groups[i];
        *out_count = static_cast<int32_t>(r.groups.size());
        *out_l_best = r.l_best;
        *out_l_max = r.l_max;
    });
}

}  // extern "C"
