// autoselect.cu — profilers, Algorithm 3/4 and Algorithm 1 on the GPU.
//
// Reference: AnalyticProfiler / TableProfiler (src/costmodel.cpp:110-265),
// greedy_profile_ckpt (Alg. 4, :271-292), find_best_sp_ckpt (Alg. 3,
// :294-325), select_groups + nearest_feasible_sp (Alg. 1,
// src/autoselect.cpp:35-168). One thread evaluates one select_groups
// problem, so a sweep over many candidate sets runs one launch. Failures are
// recorded as (code, numbers) events; the host turns them into the
// reference's exact exception text (autoselect_host.cpp) -- no decision is
// taken on the host.
#include <cmath>
#include <string>

#include "autoselect.cuh"
#include "costmodel.cuh"

namespace hbp_b200 {

namespace {

struct Ctxt {
    const DevProfiler* p;
};

__device__ const hbp_profile_row* table_find(const DevProfiler& p, int64_t l, int32_t sp) {
    for (int64_t i = 0; i < p.n_rows; ++i)
        if (p.rows[i].length == l && p.rows[i].sp == sp) return &p.rows[i];
    return nullptr;
}

__device__ AsErr mk(int code, int64_t l = 0, int32_t sp = 0, int32_t ckpt = 0, int64_t used = 0, double slope = 0.0) {
    AsErr e;
    e.code = code;
    e.length = l;
    e.sp = sp;
    e.ckpt = ckpt;
    e.used = used;
    e.slope = slope;
    return e;
}

// memory_used checks (costmodel.cpp:37-42)
__device__ AsErr mem_used(const hbp_hardware_profile& pr, int64_t l, int32_t sp, int32_t ckpt, int64_t& out) {
    if (sp < 1) return mk(AS_V_SP);
    if (ckpt < 0 || ckpt > pr.layer_count) return mk(AS_V_CKPT);
    out = cm_memory_used(l, sp, ckpt, pr);
    return mk(AS_OK);
}

__device__ AsErr p_memory(const DevProfiler& p, int64_t l, int32_t sp, int32_t ckpt, int64_t& out) {
    if (p.kind == HBP_PROFILER_ANALYTIC) {  // costmodel.cpp:131-134
        int64_t used = 0;
        AsErr e = mem_used(p.profile, l, sp, ckpt, used);
        if (e.code) return e;
        out = p.profile.device_memory - used;
        return e;
    }
    const hbp_profile_row* r = table_find(p, l, sp);  // costmodel.cpp:242-251
    if (!r) return mk(AS_I_NOROW, l, sp);
    out = r->oom ? -1 : p.device_memory - r->memory_bytes;
    return mk(AS_OK);
}

__device__ AsErr p_time(const DevProfiler& p, int64_t l, int32_t sp, int32_t ckpt, double& out) {
    if (p.kind == HBP_PROFILER_ANALYTIC) {  // one full pack of length l, costmodel.cpp:123-129
        if (l == 0) {
            out = 0.0;
            return mk(AS_OK);
        }
        int64_t used = 0;
        AsErr e = mem_used(p.profile, l, sp, ckpt, used);
        if (e.code) return e;
        if (used > p.profile.device_memory) return mk(AS_I_MEM, l, sp, ckpt, used);
        out = cm_iter_time(l, l * l, sp, ckpt, p.profile);
        return e;
    }
    const hbp_profile_row* r = table_find(p, l, sp);  // costmodel.cpp:223-240
    if (!r) return mk(AS_I_NOROW, l, sp);
    if (r->oom) return mk(AS_I_OOMROW, l, sp);
    if (r->ckpt != ckpt) return mk(AS_I_NOROW_CKPT, l, sp, ckpt);
    out = r->seconds;
    return mk(AS_OK);
}

__device__ AsErr greedy_ckpt(const DevProfiler& p, int64_t l, int32_t sp, int32_t cmin, int32_t cmax, int32_t& out) {
    if (cmin >= cmax) return mk(AS_V_GREEDY);
    int64_t a = 0, b = 0;
    AsErr e = p_memory(p, l, sp, cmin, a);
    if (e.code) return e;
    e = p_memory(p, l, sp, cmax, b);
    if (e.code) return e;
    const double m1r = static_cast<double>(a), m2r = static_cast<double>(b);
    const double m_ave = __ddiv_rn(__dsub_rn(m2r, m1r), static_cast<double>(cmax - cmin));
    if (m_ave <= 0.0) return mk(AS_I_SLOPE, l, sp, 0, 0, m_ave);
    const double c_o = __dsub_rn(static_cast<double>(cmax), __ddiv_rn(m2r, m_ave));
    int32_t rounded = static_cast<int32_t>(ceil(c_o));
    rounded = rounded < 0 ? 0 : (rounded > cmax ? cmax : rounded);
    out = rounded;
    return mk(AS_OK);
}

__device__ AsErr p_ckpt(const DevProfiler& p, int64_t l, int32_t sp, int32_t& out) {
    if (p.kind == HBP_PROFILER_ANALYTIC) return greedy_ckpt(p, l, sp, p.ckpt_min, p.ckpt_max, out);
    const hbp_profile_row* r = table_find(p, l, sp);  // costmodel.cpp:253-265
    if (!r) return mk(AS_I_NOROW, l, sp);
    if (r->oom) return mk(AS_I_OOMROW, l, sp);
    out = r->ckpt;
    return mk(AS_OK);
}

// Alg. 3 for one length; failures per sp go to fails[0..n_sp)
__device__ bool best_sp_ckpt(const DevProfiler& p, int64_t l, const int32_t* sps, int32_t nsp, int32_t& osp,
                             int32_t& ockpt, double& osec, AsErr* fails) {
    bool have = false;
    for (int32_t k = 0; k < nsp; ++k) {
        const int32_t sp = sps[k];
        fails[k] = mk(AS_OK);
        int32_t ckpt = 0;
        AsErr e = p_ckpt(p, l, sp, ckpt);
        int64_t mem = 0;
        if (!e.code) e = p_memory(p, l, sp, ckpt, mem);
        if (!e.code && mem < 0) e = mk(AS_I_NOFIT, l, sp, ckpt);
        double sec = 0.0;
        if (!e.code) e = p_time(p, l, sp, ckpt, sec);
        if (e.code) {
            fails[k] = e;
            continue;
        }
        if (!have || sec < osec) {
            have = true;
            osp = sp;
            ockpt = ckpt;
            osec = sec;
        }
    }
    return have;
}

__device__ bool is_pow2(int32_t v) { return v > 0 && (v & (v - 1)) == 0; }

__global__ void k_select(AsProblem* probs, int n_problems) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_problems) return;
    AsProblem& P = probs[i];
    const DevProfiler& p = *P.profiler;
    P.status = AS_OK;
    // Stage 1 (autoselect.cpp:102-124)
    int np = 0;
    int best = -1;
    for (int32_t li = 0; li < P.n_lengths; ++li) {
        int32_t sp = 0, ck = 0;
        double sec = 0.0;
        const bool ok = P.n_sp > 0 &&
                        best_sp_ckpt(p, P.lengths[li], P.sps, P.n_sp, sp, ck, sec, P.fails + static_cast<int64_t>(li) * P.n_sp);
        P.length_ok[li] = ok ? 1 : 0;
        if (!ok) continue;
        P.best_sp[li] = sp;
        P.best_ckpt[li] = ck;
        P.best_sec[li] = sec;
        ++np;
        if (best < 0 || sec < P.best_sec[best]) best = li;
    }
    if (np == 0) {
        P.status = AS_S_NONE;
        return;
    }
    const int last = P.n_lengths - 1;
    if (!P.length_ok[last]) {
        P.status = AS_S_LARGEST;
        return;
    }
    const int64_t l_best = P.lengths[best], l_max = P.lengths[last];
    const int32_t s_best = P.best_sp[best], c_best = P.best_ckpt[best];
    const int32_t s_max = P.best_sp[last], c_max = P.best_ckpt[last];
    // Stage 2 (autoselect.cpp:128-149)
    const int64_t l1 = l_best / s_best;
    const int64_t l2 = l_max / s_max;
    hbp_group_config raw[4];
    int nraw = 0;
    int32_t c1 = 0;
    AsErr e = p_ckpt(p, l1, 1, c1);
    if (e.code) {
        P.status = AS_S_STAGE2;
        P.stage2 = e;
        return;
    }
    raw[nraw++] = hbp_group_config{l1, 1, c1};
    raw[nraw++] = hbp_group_config{l_best, s_best, c_best};
    if (l2 > l_best) {
        // nearest_feasible_sp (autoselect.cpp:41-72)
        const double target = static_cast<double>(l2) / static_cast<double>(l1);
        int32_t bsp = -1, bck = 0;
        double bgap = 0.0;
        for (int32_t k = 0; k < P.n_sp; ++k) {
            const int32_t sp = P.sps[k];
            if (!is_pow2(sp)) continue;
            int32_t ck = 0;
            if (p_ckpt(p, l2, sp, ck).code) continue;
            int64_t mem = 0;
            if (p_memory(p, l2, sp, ck, mem).code) continue;
            if (mem < 0) continue;
            const double gap = fabs(log2(static_cast<double>(sp)) - log2(target));
            if (bsp < 0 || gap < bgap || (gap == bgap && sp < bsp)) {
                bsp = sp;
                bgap = gap;
                bck = ck;
            }
        }
        if (bsp < 0) {
            P.status = AS_S_MID;
            P.stage2 = mk(0, l2);
            return;
        }
        raw[nraw++] = hbp_group_config{l2, bsp, bck};
    }
    raw[nraw++] = hbp_group_config{l_max, s_max, c_max};
    // dedup by length keeping the lower sp, ascending (std::map)
    hbp_group_config ded[4];
    int nd = 0;
    for (int k = 0; k < nraw; ++k) {
        int f = -1;
        for (int q = 0; q < nd; ++q)
            if (ded[q].length == raw[k].length) f = q;
        if (f < 0) ded[nd++] = raw[k];
        else if (raw[k].sp < ded[f].sp) ded[f] = raw[k];
    }
    for (int x = 1; x < nd; ++x)
        for (int y = x; y > 0 && ded[y].length < ded[y - 1].length; --y) {
            const hbp_group_config tmp = ded[y];
            ded[y] = ded[y - 1];
            ded[y - 1] = tmp;
        }
    for (int k = 0; k < nd; ++k) P.out[k] = ded[k];
    P.n_out = nd;
    P.l_best = l_best;
    P.l_max = l_max;
}

// Single profiler queries: one thread per query.
__global__ void k_queries(const DevProfiler* p, AsQuery* qs, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    AsQuery& q = qs[i];
    switch (q.op) {
        case AS_Q_GREEDY:
            q.err = greedy_ckpt(*p, q.length, q.sp, q.ckpt_min, q.ckpt_max, q.out_ckpt);
            break;
        case AS_Q_DERIVE:
            q.err = p_ckpt(*p, q.length, q.sp, q.out_ckpt);
            break;
        case AS_Q_MEMORY:
            q.err = p_memory(*p, q.length, q.sp, q.ckpt, q.out_mem);
            break;
        case AS_Q_TIME:
            q.err = p_time(*p, q.length, q.sp, q.ckpt, q.out_sec);
            break;
        case AS_Q_BEST:
            q.ok = best_sp_ckpt(*p, q.length, q.sps, q.n_sp, q.out_sp, q.out_ckpt, q.out_sec, q.fails) ? 1 : 0;
            break;
        default:
            break;
    }
}

}  // namespace

void run_select_problems(Ctx& c, AsProblem* d_probs, int n) {
    if (n <= 0) return;
    LAUNCH(k_select, (n + 127) / 128, 128, 0, c.stream, d_probs, n);
}

void run_queries(Ctx& c, const DevProfiler* d_prof, AsQuery* d_q, int n) {
    if (n <= 0) return;
    LAUNCH(k_queries, (n + 127) / 128, 128, 0, c.stream, d_prof, d_q, n);
}

}  // namespace hbp_b200
