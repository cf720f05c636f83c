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
#include "sweep.cuh"
#include "../../include/hbp_b200_testing.h"

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

// One block = a maximal run of consecutive evaluated candidates with the
// same length set: processed exactly as the sequential sweep would (plan
// built at the block's first candidate with its groups, group validation for
// the rest), so every candidate gets the same seconds or the same error.
// Positions index `idx` (the global candidate indices evaluated here).
struct SweepBlock {
    int64_t begin, end;
};

void sweep_block(hbp_ctx& c, const DeviceCorpus& corpus, const SweepBlock& b, const int64_t* idx,
                 const hbp_group_config* cand_groups, const int64_t* cand_offsets, const int64_t* cand_l_best,
                 const hbp_plan_options* options, const hbp_hardware_profile* profile, int pc,
                 std::vector<double>& secs, std::vector<SweepErr>& errs) {
    CtxScope scope(c);
    std::unique_ptr<DevicePlan> plan;
    for (int64_t q = b.begin; q < b.end; ++q) {
        const int64_t k = idx[q];
        std::vector<hbp_group_config> g(cand_groups + cand_offsets[k], cand_groups + cand_offsets[k + 1]);
        try {
            if (q == b.begin) {
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

std::vector<int64_t> lengths_of(const hbp_group_config* cand_groups, const int64_t* cand_offsets, int64_t k) {
    std::vector<int64_t> ls;
    for (int64_t q = cand_offsets[k]; q < cand_offsets[k + 1]; ++q) ls.push_back(cand_groups[q].length);
    return ls;
}

}  // namespace

namespace hbp_b200 {

void sweep_ingest(hbp_ctx& c, const hbp_samples* samples, DeviceCorpus& corpus) {
    ingest(c, samples, corpus);
    validate_corpus(c, samples, corpus, (samples && samples->source) ? samples->source : "");
}

void sweep_evaluate(hbp_ctx& c, const DeviceCorpus& corpus, const hbp_group_config* cand_groups,
                    const int64_t* cand_offsets, const int64_t* cand_l_best, const std::vector<int64_t>& idx,
                    const hbp_plan_options* options, const hbp_hardware_profile* profile, std::vector<double>& secs,
                    std::vector<SweepErr>& errs) {
    if (idx.empty()) return;
    const int pc = cm_profile_check(*profile);
    std::vector<SweepBlock> blocks;
    for (size_t q = 0; q < idx.size(); ++q) {
        if (q == 0 || idx[q] != idx[q - 1] + 1 ||
            lengths_of(cand_groups, cand_offsets, idx[q]) != lengths_of(cand_groups, cand_offsets, idx[q - 1]))
            blocks.push_back({static_cast<int64_t>(q), static_cast<int64_t>(q) + 1});
        else
            blocks.back().end = static_cast<int64_t>(q) + 1;
    }
    // Plans at sweep sizes are launch- and latency-bound, so blocks run
    // concurrently: each worker thread owns a context (its own stream)
    // on the same GPU and takes blocks in order; the corpus in HBM is
    // shared read-only.
    const char* ew = std::getenv("HBP_SWEEP_STREAMS");
    int W = ew ? std::atoi(ew) : 16;
    // every worker holds one plan build in flight: ~300 B per sample at its
    // peak (pools, shuffle and next-fit scratch, the pack table sized by n;
    // measured 25 GB per worker at 100M), so at C5 sizes the free HBM, not
    // the streams, bounds the concurrency
    {
        size_t free_b = 0, total_b = 0;
        CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
        const double per_worker = 300.0 * static_cast<double>(std::max<int64_t>(corpus.n, 1)) + (256.0 * (1 << 20));
        const int by_mem = static_cast<int>(0.75 * static_cast<double>(free_b) / per_worker);
        W = std::max(1, std::min(W, by_mem));
    }
    W = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(W, static_cast<int64_t>(blocks.size()))));
    CUDA_CHECK(cudaStreamSynchronize(c.stream));  // corpus ready for the workers' streams
    // worker contexts live as long as the calling context: their streams,
    // memory pools and block caches stay warm from one sweep to the next
    while (static_cast<int>(c.workers.size()) < W) {
        hbp_ctx* wc = nullptr;
        if (hbp_ctx_create(c.device, &wc) != HBP_OK) throw EngineError(HBP_ERR_CUDA, "sweep: cannot create a worker stream");
        static const char* eb = std::getenv("HBP_SWEEP_BLOCKING");
        wc->blocking_sync = eb != nullptr && std::atoi(eb) != 0;
        c.workers.push_back(wc);
    }
    std::vector<hbp_ctx*> workers(c.workers.begin(), c.workers.begin() + W);
    for (auto* wc : workers) wc->launches = 0;
    std::atomic<size_t> next{0};
    auto work = [&](hbp_ctx* wc) {
        for (size_t bi; (bi = next.fetch_add(1)) < blocks.size();)
            sweep_block(*wc, corpus, blocks[bi], idx.data(), cand_groups, cand_offsets, cand_l_best, options,
                        profile, pc, secs, errs);
        cudaStreamSynchronize(wc->stream);
    };
    std::vector<std::thread> threads;
    for (int w = 1; w < W; ++w) threads.emplace_back(work, workers[static_cast<size_t>(w)]);
    work(workers[0]);
    for (auto& t : threads) t.join();
    for (auto* wc : workers) c.launches += wc->launches;
}

std::vector<int64_t> sweep_shard(const hbp_group_config* cand_groups, const int64_t* cand_offsets,
                                 int64_t n_candidates, int rank, int world) {
    // whole length sets, dealt round-robin in decreasing estimated cost (more
    // groups and smaller groups pack more packs): every plan is built once
    std::map<std::vector<int64_t>, std::vector<int64_t>> sets;
    for (int64_t k = 0; k < n_candidates; ++k) sets[lengths_of(cand_groups, cand_offsets, k)].push_back(k);
    std::vector<const std::pair<const std::vector<int64_t>, std::vector<int64_t>>*> order;
    for (const auto& kv : sets) order.push_back(&kv);
    std::stable_sort(order.begin(), order.end(), [](auto* a, auto* b) {
        if (a->first.size() != b->first.size()) return a->first.size() > b->first.size();
        return a->first < b->first;  // (first length, then the whole set) ascending
    });
    std::vector<int64_t> mine;
    for (size_t k = 0; k < order.size(); ++k)
        if (static_cast<int>(k % static_cast<size_t>(world)) == rank)
            mine.insert(mine.end(), order[k]->second.begin(), order[k]->second.end());
    std::sort(mine.begin(), mine.end());
    return mine;
}

}  // namespace hbp_b200

extern "C" int hbp_sweep(hbp_ctx* ctx, const hbp_samples* samples, const hbp_group_config* cand_groups,
                         const int64_t* cand_offsets, const int64_t* cand_l_best, int64_t n_candidates,
                         const hbp_plan_options* options, const hbp_hardware_profile* profile, double* out_seconds,
                         int64_t* out_best) {
    return sw_guarded(ctx, [&] {
        *out_best = -1;
        if (n_candidates <= 0) return;
        DeviceCorpus corpus;
        sweep_ingest(*ctx, samples, corpus);
        std::vector<double> secs(static_cast<size_t>(n_candidates), std::numeric_limits<double>::infinity());
        std::vector<SweepErr> errs(static_cast<size_t>(n_candidates));
        std::vector<int64_t> all(static_cast<size_t>(n_candidates));
        for (int64_t k = 0; k < n_candidates; ++k) all[static_cast<size_t>(k)] = k;
        sweep_evaluate(*ctx, corpus, cand_groups, cand_offsets, cand_l_best, all, options, profile, secs, errs);
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

extern "C" int hbp_test_sweep_shard(const hbp_group_config* cand_groups, const int64_t* cand_offsets,
                                    int64_t n_candidates, int32_t rank, int32_t world, int64_t* out_idx,
                                    int64_t* out_n) {
    if (world < 1 || rank < 0 || rank >= world || n_candidates < 0) return HBP_ERR_VALIDATION;
    const auto v = sweep_shard(cand_groups, cand_offsets, n_candidates, rank, world);
    for (size_t i = 0; i < v.size(); ++i) out_idx[i] = v[i];
    *out_n = static_cast<int64_t>(v.size());
    return HBP_OK;
}
