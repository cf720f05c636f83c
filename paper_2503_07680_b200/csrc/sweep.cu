// sweep.cu — the auto-selection candidate sweep.
//
// For every candidate HierarchicalGroups c: simulate(build_plan(samples,
// groups_c, options), profile).total_seconds, +inf when the reference would
// raise InfeasibleError (sim.cpp:34-39), argmin with the lowest index on
// ties. A plan depends only on the group lengths (packing never reads sp or
// ckpt; sp > 1 only flags comm tokens, which simulate derives from the group
// config), so candidates are grouped by length set: one GPU build_plan per
// distinct set, then one simulate per candidate over the plan in HBM with
// the candidate's (sp, ckpt) per group.
#include <cmath>
#include <limits>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/hbp_b200.h"
#include "costmodel.cuh"
#include "metrics.cuh"
#include "pipeline.cuh"

using namespace hbp_b200;

namespace {
template <typename F>
int sw_guarded(hbp_ctx* ctx, F&& fn) {
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
}  // namespace

extern "C" int hbp_sweep(hbp_ctx* ctx, const hbp_samples* samples, const hbp_group_config* cand_groups,
                         const int64_t* cand_offsets, const int64_t* cand_l_best, int64_t n_candidates,
                         const hbp_plan_options* options, const hbp_hardware_profile* profile, double* out_seconds,
                         int64_t* out_best) {
    return sw_guarded(ctx, [&] {
        *out_best = -1;
        if (n_candidates <= 0) return;
        DeviceCorpus corpus;
        ingest(*ctx, samples, corpus);
        validate_corpus(*ctx, samples, corpus, (samples && samples->source) ? samples->source : "");
        const int pc = cm_profile_check(*profile);
        std::vector<double> secs(static_cast<size_t>(n_candidates), std::numeric_limits<double>::infinity());
        // Candidates in index order, so the first non-infeasible error is the
        // one the reference would raise; the plan of the current length set
        // is kept in HBM and reused by every candidate that shares it.
        std::vector<int64_t> cur_set;
        std::unique_ptr<DevicePlan> plan_p(new DevicePlan());
        bool have_plan = false;
        for (int64_t c = 0; c < n_candidates; ++c) {
            std::vector<hbp_group_config> g(cand_groups + cand_offsets[c], cand_groups + cand_offsets[c + 1]);
            std::vector<int64_t> ls;
            for (const auto& x : g) ls.push_back(x.length);
            if (!have_plan || ls != cur_set) {
                PlanArgs a;
                a.groups = g;
                a.l_best = cand_l_best[c];
                a.l_max = g.empty() ? 0 : g.back().length;
                a.strategy = options->strategy;
                a.device_count = options->device_count;
                a.balance_batching = options->balance_batching != 0;
                a.greedy_fill = options->greedy_fill != 0;
                a.seed = options->seed;
                plan_p.reset(new DevicePlan());
                have_plan = false;
                build_plan_device(*ctx, corpus, a, *plan_p);  // validates groups, l_max, device count
                have_plan = true;
                cur_set = ls;
            } else {
                validate_groups(g, g.back().length);
            }
            if (pc) fail_validation(cm_profile_message(pc));  // simulate -> profile.validate()
            const DevicePlan& plan = *plan_p;
            const PlanArrays pa{plan.iter_group.p,    plan.iter_dev_offsets.p, plan.dev_pack_offsets.p,
                                plan.pack_capacity.p, plan.pack_total.p,       plan.pack_attention.p,
                                plan.n_iterations,    plan.n_devices};
            EvalOut eo;
            try {
                eval_plan(*ctx, pa, options->device_count, g, profile, eo, nullptr, nullptr, nullptr, nullptr, nullptr,
                          nullptr);
                secs[static_cast<size_t>(c)] = eo.total_seconds;
            } catch (const EngineError& e) {
                if (e.code != HBP_ERR_INFEASIBLE) throw;
            }
        }
        int64_t best = -1;
        for (int64_t c = 0; c < n_candidates; ++c) {
            out_seconds[c] = secs[static_cast<size_t>(c)];
            if (std::isfinite(secs[static_cast<size_t>(c)]) && (best < 0 || secs[static_cast<size_t>(c)] < secs[static_cast<size_t>(best)]))
                best = c;
        }
        *out_best = best;
    });
}
