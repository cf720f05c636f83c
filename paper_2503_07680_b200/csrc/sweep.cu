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
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <thread>
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

namespace {

// One block = a maximal run of consecutive candidates with the same length
// set: processed exactly as the sequential sweep would (plan built at the
// block's first candidate with its groups, group validation for the rest),
// so every candidate gets the same seconds or the same error.
struct SweepBlock {
    int64_t begin, end;
};

struct SweepErr {
    int code = HBP_OK;
    std::string msg;
};

void sweep_block(hbp_ctx& c, const DeviceCorpus& corpus, const SweepBlock& b, const hbp_group_config* cand_groups,
                 const int64_t* cand_offsets, const int64_t* cand_l_best, const hbp_plan_options* options,
                 const hbp_hardware_profile* profile, int pc, std::vector<double>& secs, std::vector<SweepErr>& errs) {
    CtxScope scope(c);
    std::unique_ptr<DevicePlan> plan;
    for (int64_t k = b.begin; k < b.end; ++k) {
        std::vector<hbp_group_config> g(cand_groups + cand_offsets[k], cand_groups + cand_offsets[k + 1]);
        try {
            if (k == b.begin) {
                PlanArgs a;
                a.groups = g;
                a.l_best = cand_l_best[k];
                a.l_max = g.empty() ? 0 : g.back().length;
                a.strategy = options->strategy;
                a.device_count = options->device_count;
                a.balance_batching = options->balance_batching != 0;
                a.greedy_fill = options->greedy_fill != 0;
                a.seed = options->seed;
                plan.reset(new DevicePlan());
                // build_plan_device only reads the corpus (ingest is the only writer)
                build_plan_device(c, const_cast<DeviceCorpus&>(corpus), a, *plan);  // validates groups, l_max, devices
            } else {
                validate_groups(g, g.back().length);
            }
            if (pc) fail_validation(cm_profile_message(pc));  // simulate -> profile.validate()
            const PlanArrays pa{plan->iter_group.p,    plan->iter_dev_offsets.p, plan->dev_pack_offsets.p,
                                plan->pack_capacity.p, plan->pack_total.p,       plan->pack_attention.p,
                                plan->n_iterations,    plan->n_devices};
            EvalOut eo;
            try {
                eval_plan(c, pa, options->device_count, g, profile, eo, nullptr, nullptr, nullptr, nullptr, nullptr,
                          nullptr);
                secs[static_cast<size_t>(k)] = eo.total_seconds;
            } catch (const EngineError& e) {
                if (e.code != HBP_ERR_INFEASIBLE) throw;
            }
        } catch (const EngineError& e) {
            errs[static_cast<size_t>(k)] = {e.code, e.what()};
            return;  // the sequential sweep stops here
        } catch (const std::exception& e) {
            errs[static_cast<size_t>(k)] = {HBP_ERR_CUDA, e.what()};
            return;
        }
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
        std::vector<SweepErr> errs(static_cast<size_t>(n_candidates));
        std::vector<SweepBlock> blocks;
        auto lengths_of = [&](int64_t k) {
            std::vector<int64_t> ls;
            for (int64_t q = cand_offsets[k]; q < cand_offsets[k + 1]; ++q) ls.push_back(cand_groups[q].length);
            return ls;
        };
        for (int64_t k = 0; k < n_candidates; ++k) {
            if (k == 0 || lengths_of(k) != lengths_of(k - 1)) blocks.push_back({k, k + 1});
            else blocks.back().end = k + 1;
        }
        // Plans at sweep sizes are launch- and latency-bound, so blocks run
        // concurrently: each worker thread owns a context (its own stream)
        // on the same GPU and takes blocks in order; the corpus in HBM is
        // shared read-only.
        const char* ew = std::getenv("HBP_SWEEP_STREAMS");
        int W = ew ? std::atoi(ew) : 8;
        W = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(W, static_cast<int64_t>(blocks.size()))));
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));  // corpus ready for the workers' streams
        std::vector<hbp_ctx*> workers(static_cast<size_t>(W), nullptr);
        for (int w = 0; w < W; ++w)
            if (hbp_ctx_create(ctx->device, &workers[static_cast<size_t>(w)]) != HBP_OK)
                throw EngineError(HBP_ERR_CUDA, "sweep: cannot create a worker stream");
        std::atomic<size_t> next{0};
        auto work = [&](hbp_ctx* wc) {
            for (size_t bi; (bi = next.fetch_add(1)) < blocks.size();)
                sweep_block(*wc, corpus, blocks[bi], cand_groups, cand_offsets, cand_l_best, options, profile, pc,
                            secs, errs);
            cudaStreamSynchronize(wc->stream);
        };
        std::vector<std::thread> threads;
        for (int w = 1; w < W; ++w) threads.emplace_back(work, workers[static_cast<size_t>(w)]);
        work(workers[0]);
        for (auto& t : threads) t.join();
        for (auto* wc : workers) {
            ctx->launches += wc->launches;
            hbp_ctx_destroy(wc);
        }
        // the error the sequential sweep would raise: the first in index order
        for (int64_t k = 0; k < n_candidates; ++k)
            if (errs[static_cast<size_t>(k)].code != HBP_OK)
                throw EngineError(errs[static_cast<size_t>(k)].code, errs[static_cast<size_t>(k)].msg);
        int64_t best = -1;
        for (int64_t c = 0; c < n_candidates; ++c) {
            out_seconds[c] = secs[static_cast<size_t>(c)];
            if (std::isfinite(secs[static_cast<size_t>(c)]) && (best < 0 || secs[static_cast<size_t>(c)] < secs[static_cast<size_t>(best)]))
                best = c;
        }
        *out_best = best;
    });
}
