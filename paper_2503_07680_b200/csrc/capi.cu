// capi.cpp — the extern "C" boundary (include/hbp_b200.h). Every entry point
// converts exceptions into the reference's status codes and keeps the exact
// message on the context; the work itself is queued on the context stream.
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/hbp_b200.h"
#include "../../include/hbp_b200_testing.h"
#include "costmodel.cuh"
#include "engine.cuh"
#include "metrics.cuh"
#include "pipeline.cuh"
#include "radix.cuh"

namespace hbp_b200 {
thread_local int64_t* g_launch_counter = nullptr;
thread_local KernelProfiler* g_prof = nullptr;
thread_local BlockCache* g_cache = nullptr;
}

struct StageSummary {
    std::string name;
    double ms = 0, bytes = 0;
    int64_t launches = 0;
};
static thread_local std::vector<StageSummary> t_stage_summary;

using namespace hbp_b200;

namespace {

template <typename F>
int guarded(hbp_ctx* ctx, F&& fn) {
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
    } catch (const std::bad_alloc&) {
        ctx->last_error = "host out of memory";
        return HBP_ERR_CUDA;
    } catch (const std::exception& e) {
        ctx->last_error = e.what();
        return HBP_ERR_CUDA;
    }
}

}  // namespace


static hbp_plan* new_plan(hbp_ctx* ctx) {
    auto* p = new hbp_plan();
    p->owner = ctx;
    ctx->plans.insert(p);
    return p;
}

static void delete_plan(hbp_plan* p);
hbp_plan* hbp_b200_new_plan(hbp_ctx* ctx) { return new_plan(ctx); }
void hbp_b200_delete_plan(hbp_plan* p) { delete_plan(p); }

static void delete_plan(hbp_plan* p) {
    if (p->owner) {
        p->owner->plans.erase(p);
        p->owner->host_pool.release(p->dp.host);  // keep the pinned block for the next plan
        p->dp.host = HostBlock{};
    }
    delete p;
}

extern "C" {

void hbp_hardware_profile_defaults(hbp_hardware_profile* p) {
    p->per_token_linear_cost = 2.5e-4;
    p->per_token2_attention_cost = 1.5e-9;
    p->sp_comm_cost = 1.6e-5;
    p->gc_recompute_factor = 1.0 / 3.0;
    p->fixed_iteration_cost = 0.0;
    p->layer_count = 32;
    p->base_memory = 24LL << 30;
    p->per_token_activation_memory = 300000.0;
    p->gc_memory_saving_per_layer = 300000.0 * 0.75 * 4096.0;
    p->reference_length = 4096;
    p->device_memory = 80LL << 30;
}

int hbp_ctx_create(int device, hbp_ctx** out) {
    if (out == nullptr) return HBP_ERR_VALIDATION;
    *out = nullptr;
    // contexts, their side streams and the sweep's workers are independent
    // streams: give them their own hardware queues (read when the process's
    // CUDA context is created; no effect if that already happened)
    setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0);
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return HBP_ERR_CUDA;
    }
    if (device < 0 || device >= count) return HBP_ERR_VALIDATION;
    auto* c = new hbp_ctx();
    c->device = device;
    // the main stream at the highest priority: the side stream's kernels
    // (engine.cuh side_fork) only take what the main stream leaves idle
    int prio_lo = 0, prio_hi = 0;
    if (cudaSetDevice(device) != cudaSuccess || cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_hi) != cudaSuccess) {
        cudaGetLastError();
        delete c;
        return HBP_ERR_CUDA;
    }
    // a private stream-ordered pool per context (BlockCache::pool): freed
    // scratch stays in it between calls, and reuse never makes one
    // context's stream wait for another's (nor the side stream for the main
    // one: internal dependencies off, a block is reused once its free ran)
    {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        cudaMemPool_t pool = nullptr;
        if (cudaMemPoolCreate(&pool, &props) == cudaSuccess) {
            uint64_t threshold = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
            int no = 0;
            cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no);
            c->blocks.pool = pool;
        } else {
            cudaGetLastError();
        }
    }
    *out = c;
    return HBP_OK;
}

void hbp_ctx_destroy(hbp_ctx* ctx) {
    if (ctx == nullptr) return;
    for (hbp_ctx* w : ctx->workers) hbp_ctx_destroy(w);
    ctx->workers.clear();
    cudaSetDevice(ctx->device);
    if (ctx->stream) {
        cudaStreamSynchronize(ctx->stream);
        for (hbp_plan* p : ctx->plans) {  // outliving plans keep their host view only
            p->dp.release_device();
            p->owner = nullptr;
        }
        ctx->plans.clear();
        ctx->scan.status.release();
        ctx->scan.counter.release();
        if (ctx->side) {
            cudaStreamSynchronize(ctx->side);
            ctx->side_scan.status.release();
            ctx->side_scan.counter.release();
            cudaStreamSynchronize(ctx->side);
            cudaStreamDestroy(ctx->side);
            cudaEventDestroy(ctx->ev_fork);
            cudaEventDestroy(ctx->ev_join);
        }
        ctx->blocks.stream = ctx->stream;
        ctx->blocks.clear();  // after every buffer that returns blocks to it
        cudaStreamSynchronize(ctx->stream);
        cudaStreamDestroy(ctx->stream);
        if (ctx->blocks.pool) cudaMemPoolDestroy(ctx->blocks.pool);
        if (ctx->ev_sync) cudaEventDestroy(ctx->ev_sync);
    }
    delete ctx;
}

const char* hbp_last_error(const hbp_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

int hbp_ctx_synchronize(hbp_ctx* ctx) {
    return guarded(ctx, [&] { CUDA_CHECK(cudaStreamSynchronize(ctx->stream)); });
}

void* hbp_ctx_stream(hbp_ctx* ctx) { return ctx ? reinterpret_cast<void*>(ctx->stream) : nullptr; }

int64_t hbp_ctx_launch_count(const hbp_ctx* ctx) { return ctx ? ctx->launches : 0; }

int hbp_ctx_set_profiling(hbp_ctx* ctx, int32_t on) {
    return guarded(ctx, [&] {
        if (on) {
            // drop stale records
            for (auto& r : ctx->prof.recs) {
                ctx->prof.spare.push_back(r.a);
                ctx->prof.spare.push_back(r.b);
            }
            ctx->prof.recs.clear();
        }
        ctx->prof.on = on != 0;
    });
}

int hbp_ctx_stage_stats(hbp_ctx* ctx, int32_t index, char* name, int32_t name_len, double* ms, int64_t* launches,
                        double* bytes) {
    return guarded(ctx, [&] {
        if (!ctx->prof.recs.empty()) {
            CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
            std::map<std::string, StageSummary> agg;
            for (auto& r : ctx->prof.recs) {
                float t = 0;
                CUDA_CHECK(cudaEventElapsedTime(&t, r.a, r.b));
                auto& s = agg[r.name];
                s.name = r.name;
                s.ms += t;
                s.bytes += r.bytes;
                s.launches += 1;
                ctx->prof.spare.push_back(r.a);
                ctx->prof.spare.push_back(r.b);
            }
            ctx->prof.recs.clear();
            t_stage_summary.clear();
            for (auto& kv : agg) t_stage_summary.push_back(kv.second);
        }
        if (index < 0 || static_cast<size_t>(index) >= t_stage_summary.size()) fail_validation("no such stage");
        const auto& s = t_stage_summary[static_cast<size_t>(index)];
        if (name && name_len > 0) {
            std::strncpy(name, s.name.c_str(), static_cast<size_t>(name_len) - 1);
            name[name_len - 1] = '\0';
        }
        *ms = s.ms;
        *launches = s.launches;
        *bytes = s.bytes;
    });
}

// ---- hot path -----------------------------------------------------------------

static std::vector<hbp_group_config> groups_of(const hbp_groups* g) {
    if (g == nullptr || g->count < 0 || (g->count > 0 && g->groups == nullptr))
        throw EngineError(HBP_ERR_VALIDATION, "no packing groups");
    return std::vector<hbp_group_config>(g->groups, g->groups + g->count);
}

static std::string source_of(const hbp_samples* s) { return (s && s->source) ? s->source : ""; }

int hbp_load_lengths(hbp_ctx* ctx, const char* text, int64_t bytes, int32_t format, const char* source,
                     int64_t* out_ids, int64_t* out_lengths, int64_t capacity, int32_t out_memory,
                     int64_t* out_count) {
    return guarded(ctx, [&] {
        if (bytes < 0 || (bytes > 0 && text == nullptr)) fail_validation("corpus text is null");
        DevBuf<int64_t> lens, ids;
        const i64 n =
            parse_corpus_text(*ctx, text, static_cast<u64>(bytes), format, source ? source : "", lens, ids);
        if (n > capacity)
            fail_validation("output capacity " + std::to_string(capacity) + " < " + std::to_string(n) + " samples");
        if (out_memory == HBP_MEM_DEVICE) {
            CUDA_CHECK(cudaMemcpyAsync(out_lengths, lens.p, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, ctx->stream));
            if (out_ids)
                CUDA_CHECK(cudaMemcpyAsync(out_ids, ids.p, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, ctx->stream));
            CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        } else {
            staged_copy(*ctx, out_lengths, lens.p, sizeof(int64_t) * static_cast<size_t>(n), false);
            if (out_ids) staged_copy(*ctx, out_ids, ids.p, sizeof(int64_t) * static_cast<size_t>(n), false);
        }
        *out_count = n;
    });
}

int hbp_validate(hbp_ctx* ctx, const hbp_samples* samples) {
    return guarded(ctx, [&] {
        DeviceCorpus corpus;
        ingest(*ctx, samples, corpus);
        validate_corpus(*ctx, samples, corpus, source_of(samples));
    });
}

int hbp_group_data(hbp_ctx* ctx, const hbp_samples* samples, const hbp_groups* groups, int64_t* group_offsets,
                   int32_t* member_index) {
    return guarded(ctx, [&] {
        const auto g = groups_of(groups);
        validate_groups(g, groups->l_max);
        DeviceCorpus corpus;
        ingest(*ctx, samples, corpus);
        std::vector<int64_t> off;
        std::vector<int32_t> mem;
        group_data_device(*ctx, corpus, g, groups->l_max, off, mem);
        std::memcpy(group_offsets, off.data(), sizeof(int64_t) * off.size());
        if (!mem.empty()) std::memcpy(member_index, mem.data(), sizeof(int32_t) * mem.size());
    });
}

int hbp_pack(hbp_ctx* ctx, const hbp_samples* samples, int64_t capacity, const hbp_strategy* strategy, uint64_t seed,
             hbp_plan** out) {
    return guarded(ctx, [&] {
        *out = nullptr;
        validate_strategy(*strategy);
        if (capacity < 1) fail_validation("pack capacity must be >= 1");
        DeviceCorpus corpus;
        ingest(*ctx, samples, corpus);
        auto* p = new_plan(ctx);
        try {
            pack_device(*ctx, corpus, capacity, *strategy, seed, p->dp);
            p->dp.seed = seed;
        } catch (...) {
            delete_plan(p);
            throw;
        }
        *out = p;
    });
}

int hbp_build_batching_plan(hbp_ctx* ctx, const hbp_samples* samples, hbp_group_config group,
                            int32_t device_count, int32_t mode, uint64_t seed, hbp_plan** out) {
    return guarded(ctx, [&] {
        *out = nullptr;
        if (mode != HBP_BATCHING_SORTED && mode != HBP_BATCHING_RANDOM) fail_validation("unknown batching mode");
        DeviceCorpus corpus;
        ingest(*ctx, samples, corpus);
        validate_corpus(*ctx, samples, corpus, source_of(samples));  // balance.cpp:263
        auto* p = new_plan(ctx);
        try {
            batching_plan_device(*ctx, corpus, group, device_count, mode == HBP_BATCHING_SORTED, seed, p->dp);
        } catch (...) {
            delete_plan(p);
            throw;
        }
        *out = p;
    });
}

int hbp_plan_from_json(hbp_ctx* ctx, const char* text, int64_t bytes, hbp_plan** out, int64_t* out_n_members) {
    return guarded(ctx, [&] {
        *out = nullptr;
        if (bytes < 0 || (bytes > 0 && text == nullptr)) fail_validation("manifest text is null");
        auto* p = new_plan(ctx);
        try {
            plan_from_json_device(*ctx, text, static_cast<u64>(bytes), p->dp, p->read_ids, p->read_lens);
        } catch (...) {
            delete_plan(p);
            throw;
        }
        *out_n_members = p->dp.n_members;
        *out = p;
    });
}

int hbp_plan_upload(hbp_ctx* ctx, const hbp_plan_view* v, hbp_plan** out) {
    return guarded(ctx, [&] {
        *out = nullptr;
        if (v == nullptr) fail_validation("null plan view");
        auto* p = new_plan(ctx);
        try {
            DevicePlan& d = p->dp;
            cudaStream_t s = ctx->stream;
            d.device_count = v->device_count;
            d.seed = v->seed;
            d.groups.assign(v->groups.groups, v->groups.groups + v->groups.count);
            d.l_best = v->groups.l_best;
            d.l_max = v->groups.l_max;
            d.n_iterations = v->n_iterations;
            d.n_devices = v->n_devices;
            d.n_packs = v->n_packs;
            d.n_members = v->n_members;
            auto up = [&](auto& buf, const auto* src, int64_t n) {
                buf.alloc(static_cast<size_t>(n) + 1, s);
                if (n > 0 && src)
                    CUDA_CHECK(cudaMemcpyAsync(buf.p, src, sizeof(*src) * static_cast<size_t>(n), cudaMemcpyHostToDevice, s));
            };
            up(d.iter_group, v->iter_group, d.n_iterations);
            up(d.iter_dev_offsets, v->iter_dev_offsets, d.n_iterations + 1);
            up(d.dev_index, v->dev_index, d.n_devices);
            up(d.dev_pack_offsets, v->dev_pack_offsets, d.n_devices + 1);
            up(d.pack_capacity, v->pack_capacity, d.n_packs);
            up(d.pack_total, v->pack_total, d.n_packs);
            up(d.pack_attention, v->pack_attention, d.n_packs);
            up(d.pack_member_offsets, v->pack_member_offsets, d.n_packs + 1);
            up(d.member_index, v->member_index, d.n_members);
            if (v->iter_phase) up(d.iter_phase, v->iter_phase, d.n_iterations);
            CUDA_CHECK(cudaStreamSynchronize(s));
        } catch (...) {
            delete_plan(p);
            throw;
        }
        *out = p;
    });
}

int hbp_plan_members(hbp_ctx* ctx, hbp_plan* plan, int64_t* ids, int64_t* lengths) {
    return guarded(ctx, [&] {
        if (plan == nullptr) fail_validation("null plan");
        if (!plan->read_ids.p) fail_validation("plan_members: the plan was not read from a manifest");
        const size_t m = static_cast<size_t>(plan->dp.n_members);
        staged_copy(*ctx, ids, plan->read_ids.p, sizeof(int64_t) * m, false);
        staged_copy(*ctx, lengths, plan->read_lens.p, sizeof(int64_t) * m, false);
    });
}

int hbp_padded_batching(hbp_ctx* ctx, const hbp_samples* samples, int64_t token_budget, int32_t mode,
                        uint64_t seed, int32_t* order, int64_t* batch_offsets, int64_t* batch_max,
                        int64_t* n_batches) {
    return guarded(ctx, [&] {
        if (mode != HBP_BATCHING_SORTED && mode != HBP_BATCHING_RANDOM) fail_validation("unknown batching mode");
        DeviceCorpus corpus;
        ingest(*ctx, samples, corpus);
        PaddedBatches pb;
        padded_batches_device(*ctx, corpus, token_budget, mode == HBP_BATCHING_SORTED, seed, pb);
        const u64 n = pb.n, B = pb.n_batches;
        *n_batches = static_cast<int64_t>(B);
        if (n == 0) {
            batch_offsets[0] = 0;
            return;
        }
        cudaStream_t s = ctx->stream;
        const u64* ord = pb.order.p;
        const u32* bs = pb.bstart.p;
        const u32* bm = pb.bmax.p;
        DevBuf<int32_t> dord(n, s);
        DevBuf<int64_t> doff(B + 1, s), dmax(B + 1, s);
        int32_t* po = dord.p;
        int64_t* pf = doff.p;
        int64_t* pm = dmax.p;
        for_each_index(*ctx, n, [=] __device__(u64 i) { po[i] = static_cast<int32_t>(static_cast<u32>(ord[i])); });
        for_each_index(*ctx, B + 1, [=] __device__(u64 b) {
            pf[b] = b < B ? static_cast<int64_t>(bs[b]) : static_cast<int64_t>(n);
            if (b < B) pm[b] = bm[b];
        });
        CUDA_CHECK(cudaMemcpyAsync(order, dord.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaMemcpyAsync(batch_offsets, doff.p, sizeof(int64_t) * (B + 1), cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaMemcpyAsync(batch_max, dmax.p, sizeof(int64_t) * B, cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int hbp_build_plan(hbp_ctx* ctx, const hbp_samples* samples, const hbp_groups* groups,
                   const hbp_plan_options* options, hbp_plan** out) {
    return guarded(ctx, [&] {
        *out = nullptr;
        trace_begin(*ctx);
        DeviceCorpus corpus;
        ingest(*ctx, samples, corpus);
        validate_corpus(*ctx, samples, corpus, source_of(samples));  // balance.cpp:209
        trace_mark(*ctx, "ingest+validate");
        PlanArgs a;
        a.groups = groups_of(groups);
        a.l_best = groups->l_best;
        a.l_max = groups->l_max;
        a.strategy = options->strategy;
        a.device_count = options->device_count;
        a.balance_batching = options->balance_batching != 0;
        a.greedy_fill = options->greedy_fill != 0;
        a.seed = options->seed;
        auto* p = new_plan(ctx);
        try {
            build_plan_device(*ctx, corpus, a, p->dp);
            trace_dump(*ctx, "build_plan");
        } catch (...) {
            delete_plan(p);
            throw;
        }
        *out = p;
    });
}

int hbp_greedy_fill(hbp_ctx* ctx, const hbp_packs_in* packs, int32_t n_pools, const int64_t* pool_offsets,
                    const int64_t* pool_ids, const int64_t* pool_lengths, int64_t* out_added_offsets,
                    int64_t* out_added, uint8_t* out_pool_keep) {
    return guarded(ctx, [&] {
        std::vector<int64_t> off, added;
        std::vector<uint8_t> keep;
        greedy_fill_device(*ctx, packs->n_packs, packs->pack_capacity, packs->pack_offsets, packs->lengths, n_pools,
                           pool_offsets, pool_ids, pool_lengths, off, added, keep);
        std::memcpy(out_added_offsets, off.data(), sizeof(int64_t) * off.size());
        if (!added.empty()) std::memcpy(out_added, added.data(), sizeof(int64_t) * added.size());
        if (!keep.empty()) std::memcpy(out_pool_keep, keep.data(), keep.size());
    });
}

int hbp_balance_batching(hbp_ctx* ctx, const hbp_packs_in* packs, int64_t capacity, int32_t device_count,
                         int32_t group_index, int32_t random_batching, uint64_t seed, hbp_plan** out) {
    return guarded(ctx, [&] {
        *out = nullptr;
        if (device_count < 1) fail_validation("device count must be >= 1");
        auto* p = new_plan(ctx);
        try {
            batching_device(*ctx, capacity, packs->n_packs, packs->pack_capacity, packs->pack_offsets, packs->ids,
                            packs->lengths, device_count, group_index, random_batching != 0, seed, p->dp);
            p->dp.groups.assign(static_cast<size_t>(group_index) + 1, hbp_group_config{capacity, 1, 0});
            p->dp.l_max = capacity;
        } catch (...) {
            delete_plan(p);
            throw;
        }
        *out = p;
    });
}

int hbp_plan_view_get(hbp_ctx* ctx, hbp_plan* plan, hbp_plan_view* out) {
    return guarded(ctx, [&] {
        if (plan == nullptr) fail_validation("null plan");
        DevicePlan& d = plan->dp;
        plan_to_host(*ctx, d);
        hbp_plan_view& v = plan->view;
        v.device_count = d.device_count;
        v.seed = d.seed;
        v.groups.groups = d.groups.data();
        v.groups.count = static_cast<int32_t>(d.groups.size());
        v.groups.l_best = d.l_best;
        v.groups.l_max = d.l_max;
        v.n_iterations = d.n_iterations;
        v.n_devices = d.n_devices;
        v.n_packs = d.n_packs;
        v.n_members = d.n_members;
        v.iter_group = d.h_iter_group;
        v.iter_dev_offsets = d.h_iter_dev_offsets;
        v.dev_index = d.h_dev_index;
        v.dev_pack_offsets = d.h_dev_pack_offsets;
        v.pack_capacity = d.h_pack_capacity;
        v.pack_total = d.h_pack_total;
        v.pack_attention = d.h_pack_attention;
        v.pack_member_offsets = d.h_pack_member_offsets;
        v.member_index = d.h_member_index;
        v.iter_phase = d.h_iter_phase;
        *out = v;
    });
}

void hbp_plan_free(hbp_plan* plan) {
    if (plan) delete_plan(plan);
}

namespace {

// Uploads the pack-level arrays of a host view.
struct UploadedPlan {
    DevBuf<int32_t> ig;
    DevBuf<int64_t> ido, dpo, cap, tot, att;
    PlanArrays arrays{};
    std::vector<hbp_group_config> groups;
};

void upload_view(hbp_ctx* ctx, const hbp_plan_view* v, UploadedPlan& u) {
    cudaStream_t s = ctx->stream;
    const size_t I = static_cast<size_t>(v->n_iterations), D = static_cast<size_t>(v->n_devices),
                 P = static_cast<size_t>(v->n_packs);
    auto up = [&](auto& buf, const auto* src, size_t n) {
        buf.alloc(n + 1, s);
        if (n) CUDA_CHECK(cudaMemcpyAsync(buf.p, src, sizeof(src[0]) * n, cudaMemcpyHostToDevice, s));
    };
    up(u.ig, v->iter_group, I);
    up(u.ido, v->iter_dev_offsets, I + 1);
    up(u.dpo, v->dev_pack_offsets, D + 1);
    up(u.cap, v->pack_capacity, P);
    up(u.tot, v->pack_total, P);
    up(u.att, v->pack_attention, P);
    u.arrays = PlanArrays{u.ig.p, u.ido.p, u.dpo.p, u.cap.p, u.tot.p, u.att.p, static_cast<i64>(I), static_cast<i64>(D)};
    u.groups = groups_of(&v->groups);
    // group indices must address the plan's groups (Plan::group_of uses .at())
    for (size_t i = 0; i < I; ++i)
        if (v->iter_group[i] < 0 || static_cast<size_t>(v->iter_group[i]) >= u.groups.size())
            throw EngineError(HBP_ERR_VALIDATION, "iteration group index out of range");
}

PlanArrays arrays_of(const DevicePlan& d) {
    return PlanArrays{d.iter_group.p, d.iter_dev_offsets.p, d.dev_pack_offsets.p, d.pack_capacity.p, d.pack_total.p,
                      d.pack_attention.p, d.n_iterations, d.n_devices};
}

void run_eval(hbp_ctx* ctx, const PlanArrays& pa, int32_t device_count, const std::vector<hbp_group_config>& groups,
              const hbp_hardware_profile* profile, EvalOut& eo, double* h_dbr, double* h_abr, double* h_secs,
              double* h_dcomp, double* h_dcomm, double* h_didle) {
    cudaStream_t s = ctx->stream;
    const size_t I = static_cast<size_t>(pa.I), D = static_cast<size_t>(pa.D);
    DevBuf<double> dbr, abr, secs, dc, dm, di;
    if (h_dbr) dbr.alloc(I + 1, s);
    if (h_abr) abr.alloc(I + 1, s);
    if (h_secs) secs.alloc(I + 1, s);
    if (h_dcomp) dc.alloc(D + 1, s);
    if (h_dcomm) dm.alloc(D + 1, s);
    if (h_didle) di.alloc(D + 1, s);
    eval_plan(*ctx, pa, device_count, groups, profile, eo, dbr.p, abr.p, secs.p, dc.p, dm.p, di.p);
    auto down = [&](double* h, DevBuf<double>& d, size_t n) {
        if (h && n) CUDA_CHECK(cudaMemcpyAsync(h, d.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    };
    down(h_dbr, dbr, I);
    down(h_abr, abr, I);
    down(h_secs, secs, I);
    down(h_dcomp, dc, D);
    down(h_dcomm, dm, D);
    down(h_didle, di, D);
    CUDA_CHECK(cudaStreamSynchronize(s));
}

}  // namespace

int hbp_report(hbp_ctx* ctx, const hbp_plan_view* plan, hbp_metrics* out, double* per_iteration_dbr,
               double* per_iteration_abr) {
    return guarded(ctx, [&] {
        if (plan->n_iterations == 0) fail_validation("metrics report: empty plan");
        UploadedPlan u;
        upload_view(ctx, plan, u);
        EvalOut eo;
        run_eval(ctx, u.arrays, plan->device_count, u.groups, nullptr, eo, per_iteration_dbr, per_iteration_abr,
                 nullptr, nullptr, nullptr, nullptr);
        *out = eo.m;
    });
}

namespace {
// Σ tokens, Σ comm tokens and the widest iteration of a run of device
// batches: integer sums, so the ratios the reference forms from its
// sequential double sums (metrics.cpp:71-105) come out identical
__global__ void k_run_totals(const int64_t* __restrict__ tokens, const int64_t* __restrict__ comm,
                             const int64_t* __restrict__ iter_off, u64 n_iter, u64 n_dev,
                             unsigned long long* __restrict__ out) {
    unsigned long long t = 0, cm = 0, w = 0;
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n_dev || i < n_iter;
         i += static_cast<u64>(gridDim.x) * blockDim.x) {
        if (i < n_dev) {
            t += static_cast<unsigned long long>(tokens[i]);
            cm += static_cast<unsigned long long>(comm[i]);
        }
        if (i < n_iter) w = max(w, static_cast<unsigned long long>(iter_off[i + 1] - iter_off[i]));
    }
    t = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(t & 0xffffffffu)) +
        (static_cast<unsigned long long>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(t >> 32))) << 32);
    cm = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(cm & 0xffffffffu)) +
         (static_cast<unsigned long long>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(cm >> 32))) << 32);
    w = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(min(w, 0xffffffffull)));
    if ((threadIdx.x & 31u) == 0) {
        atomicAdd(&out[0], t);
        atomicAdd(&out[1], cm);
        atomicMax(&out[2], w);
    }
}
}  // namespace

int hbp_run_totals(hbp_ctx* ctx, const int64_t* tokens, const int64_t* comm_tokens, const int64_t* iter_dev_offsets,
                   int64_t n_iterations, int64_t* out) {
    return guarded(ctx, [&] {
        const u64 I = static_cast<u64>(std::max<int64_t>(n_iterations, 0));
        const u64 D = I ? static_cast<u64>(iter_dev_offsets[I]) : 0;
        cudaStream_t s = ctx->stream;
        DevBuf<int64_t> dt(D + 1, s), dc(D + 1, s), doff(I + 1, s);
        DevBuf<unsigned long long> o(3, s);
        o.zero();
        if (D) {
            CUDA_CHECK(cudaMemcpyAsync(dt.p, tokens, sizeof(int64_t) * D, cudaMemcpyHostToDevice, s));
            CUDA_CHECK(cudaMemcpyAsync(dc.p, comm_tokens, sizeof(int64_t) * D, cudaMemcpyHostToDevice, s));
        }
        if (I) CUDA_CHECK(cudaMemcpyAsync(doff.p, iter_dev_offsets, sizeof(int64_t) * (I + 1), cudaMemcpyHostToDevice, s));
        if (I || D)
            LAUNCH_B("metrics.run_totals", 16.0 * D + 8.0 * I, k_run_totals, grid_for(std::max(I, D), 256, 148u * 4u), 256,
                     0, s, dt.p, dc.p, doff.p, I, D, o.p);
        const auto h = read_vector(*ctx, o.p, 3);
        for (int k = 0; k < 3; ++k) out[k] = static_cast<int64_t>(h[k]);
    });
}

int hbp_report_plan(hbp_ctx* ctx, hbp_plan* plan, hbp_metrics* out, double* per_iteration_dbr,
                    double* per_iteration_abr) {
    return guarded(ctx, [&] {
        EvalOut eo;
        run_eval(ctx, arrays_of(plan->dp), plan->dp.device_count, plan->dp.groups, nullptr, eo, per_iteration_dbr,
                 per_iteration_abr, nullptr, nullptr, nullptr, nullptr);
        *out = eo.m;
    });
}

int hbp_simulate(hbp_ctx* ctx, const hbp_plan_view* plan, const hbp_hardware_profile* profile, hbp_sim_totals* out,
                 double* iteration_seconds, double* device_compute, double* device_comm, double* device_idle) {
    return guarded(ctx, [&] {
        const int pc = cm_profile_check(*profile);
        if (pc) fail_validation(cm_profile_message(pc));
        if (plan->n_iterations == 0) fail_validation("simulate: empty plan");
        UploadedPlan u;
        upload_view(ctx, plan, u);
        EvalOut eo;
        run_eval(ctx, u.arrays, plan->device_count, u.groups, profile, eo, nullptr, nullptr, iteration_seconds,
                 device_compute, device_comm, device_idle);
        out->metrics = eo.m;
        out->total_seconds = eo.total_seconds;
        out->gpu_days = eo.total_seconds * static_cast<double>(plan->device_count) / 86400.0;
        out->switch_count = eo.switch_count;
        out->device_count = plan->device_count;
    });
}

int hbp_simulate_plan(hbp_ctx* ctx, hbp_plan* plan, const hbp_hardware_profile* profile, hbp_sim_totals* out,
                      double* iteration_seconds) {
    return guarded(ctx, [&] {
        const int pc = cm_profile_check(*profile);
        if (pc) fail_validation(cm_profile_message(pc));
        if (plan->dp.n_iterations == 0) fail_validation("simulate: empty plan");
        EvalOut eo;
        run_eval(ctx, arrays_of(plan->dp), plan->dp.device_count, plan->dp.groups, profile, eo, nullptr, nullptr,
                 iteration_seconds, nullptr, nullptr, nullptr);
        out->metrics = eo.m;
        out->total_seconds = eo.total_seconds;
        out->gpu_days = eo.total_seconds * static_cast<double>(plan->dp.device_count) / 86400.0;
        out->switch_count = eo.switch_count;
        out->device_count = plan->dp.device_count;
    });
}

int hbp_eval_columns(hbp_ctx* ctx, hbp_plan* plan, int32_t phase, int32_t col0, int32_t col1,
                     const hbp_hardware_profile* profile, const hbp_eval_columns_bufs* bufs) {
    return guarded(ctx, [&] {
        if (plan == nullptr || bufs == nullptr) fail_validation("null plan or buffers");
        if (phase != 0 && phase != 1) fail_validation("eval_columns: phase must be 0 or 1");
        if (col0 < 0 || col1 < col0) fail_validation("eval_columns: bad column range");
        eval_columns(*ctx, arrays_of(plan->dp), plan->dp.groups, profile, phase, col0, col1, *bufs);
    });
}

int hbp_eval_columns_finish(hbp_ctx* ctx, hbp_plan* plan, const hbp_hardware_profile* profile,
                            const hbp_eval_columns_bufs* bufs, hbp_metrics* out, hbp_sim_totals* sim) {
    return guarded(ctx, [&] {
        if (plan == nullptr || bufs == nullptr) fail_validation("null plan or buffers");
        EvalOut eo;
        eval_columns_finish(*ctx, arrays_of(plan->dp), plan->dp.device_count, plan->dp.groups, profile, *bufs, eo);
        if (out) *out = eo.m;
        if (sim) {
            sim->metrics = eo.m;
            sim->total_seconds = eo.total_seconds;
            sim->gpu_days = eo.total_seconds * static_cast<double>(plan->dp.device_count) / 86400.0;
            sim->switch_count = eo.switch_count;
            sim->device_count = plan->dp.device_count;
        }
    });
}

int hbp_memory_used(hbp_ctx* ctx, int64_t length, int32_t sp, int32_t ckpt, const hbp_hardware_profile* profile,
                    int64_t* out) {
    return guarded(ctx, [&] {
        if (sp < 1) fail_validation("sp must be >= 1");
        if (ckpt < 0 || ckpt > profile->layer_count) fail_validation("ckpt must lie in [0, layer_count]");
        *out = cm_memory_used(length, sp, ckpt, *profile);
    });
}

// ---- testing hooks ----------------------------------------------------------

int hbp_test_set_force_reject(hbp_ctx* ctx, uint64_t step) {
    if (ctx == nullptr) return HBP_ERR_VALIDATION;
    ctx->test_force_reject = step;
    return HBP_OK;
}

int hbp_test_shuffle_positions(hbp_ctx* ctx, uint64_t seed, int64_t m, uint32_t* out_src) {
    return guarded(ctx, [&] {
        if (m <= 0) return;
        DevBuf<u32> src(static_cast<size_t>(m), ctx->stream);
        fy_source_positions(*ctx, seed, m, src.p);
        CUDA_CHECK(cudaMemcpyAsync(out_src, src.p, sizeof(u32) * m, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int hbp_test_scan_u32(hbp_ctx* ctx, const uint32_t* in, int64_t n, uint64_t* out) {
    return guarded(ctx, [&] {
        if (n <= 0) return;
        DevBuf<u32> din(static_cast<size_t>(n), ctx->stream);
        DevBuf<u64> dout(static_cast<size_t>(n), ctx->stream);
        CUDA_CHECK(cudaMemcpyAsync(din.p, in, sizeof(u32) * n, cudaMemcpyHostToDevice, ctx->stream));
        const u32* ip = din.p;
        u64* op = dout.p;
        scan_exclusive<u64>(
            n, [=] __device__(i64 i) { return static_cast<u64>(ip[i]); },
            [=] __device__(i64 i, u64 v) { op[i] = v; }, ctx->stream, ctx->scan);
        CUDA_CHECK(cudaMemcpyAsync(out, dout.p, sizeof(u64) * n, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int hbp_test_radix_sort(hbp_ctx* ctx, uint32_t* keys, uint32_t* values, int64_t n, int32_t bits,
                        int32_t descending) {
    return guarded(ctx, [&] {
        if (n <= 0) return;
        DevBuf<u32> k(static_cast<size_t>(n), ctx->stream), v(static_cast<size_t>(n), ctx->stream);
        CUDA_CHECK(cudaMemcpyAsync(k.p, keys, sizeof(u32) * n, cudaMemcpyHostToDevice, ctx->stream));
        CUDA_CHECK(cudaMemcpyAsync(v.p, values, sizeof(u32) * n, cudaMemcpyHostToDevice, ctx->stream));
        radix_sort_pairs(*ctx, k.p, v.p, n, bits, descending != 0);
        CUDA_CHECK(cudaMemcpyAsync(keys, k.p, sizeof(u32) * n, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_CHECK(cudaMemcpyAsync(values, v.p, sizeof(u32) * n, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

}  // extern "C"
