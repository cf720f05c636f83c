// comm.cu — the multi-GPU entry points over NCCL.
//
// The reference is single-process; its "devices" are vector entries
// (proj/include/hbp/balance.hpp:18-22). Two parts of the path shard across
// the GPUs of one box with one exchange each, and both exchanges are NCCL
// collectives issued here, in C++, on the context's stream:
//
//  * hbp_sweep_sharded — the auto-selection sweep (BASELINE C3 / C5): whole
//    length sets dealt to ranks, every rank evaluates its share with the
//    single-GPU sweep, then ncclAllReduce(MIN) of the per-candidate seconds
//    (+inf where not owned), ncclAllGather of each rank's first error
//    (global index, code, message) and of each rank's (best seconds, best
//    index) -- the NCCL argmin, lowest index on ties.
//  * hbp_eval_sharded — report + simulate of one plan by data-parallel
//    column (BASELINE C4's 8-rank DP): phase-0 vectors all-reduced MAX /
//    SUM / MIN, phase-1 integer gaps all-reduced SUM, then every rank
//    finishes identically (bit-identical to the single-GPU result).
//
// NCCL is resolved at run time (dlopen "libnccl.so.2": the copy already in
// the process -- e.g. torch's -- or the system's), so the engine library has
// no link-time dependency on it and a process without NCCL only fails when
// it asks for a communicator.
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hbp_b200.h"
#include "costmodel.cuh"
#include "engine.cuh"
#include "metrics.cuh"
#include "pipeline.cuh"
#include "sweep.cuh"

using namespace hbp_b200;

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h == nullptr) {
            const char* e = dlerror();
            api.why = std::string("NCCL unavailable: ") + (e ? e : "libnccl.so.2 not found");
            return;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
        api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
        api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
        api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce && api.all_gather &&
                 api.group_start && api.group_end && api.error_string;
        if (!api.ok) api.why = "NCCL unavailable: libnccl.so.2 lacks a required symbol";
    });
    return api;
}

const NcclApi& need_nccl() {
    const NcclApi& a = nccl();
    if (!a.ok) throw EngineError(HBP_ERR_CUDA, a.why);
    return a;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw EngineError(HBP_ERR_CUDA, std::string("NCCL ") + what + ": " + nccl().error_string(r));
}

template <typename F>
int cm_guarded(hbp_ctx* ctx, F&& fn) {
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

// One rank's first sweep error, exchanged by all-gather (fixed size).
struct ErrRecord {
    int64_t index;  // global candidate index, INT64_MAX when none
    int32_t code;
    int32_t len;
    char msg[496];
};
static_assert(sizeof(ErrRecord) == 512, "ErrRecord is exchanged as 512 bytes");

struct BestRecord {
    double seconds;
    int64_t index;
};

}  // namespace

struct hbp_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1, device = 0;
};

extern "C" {

int hbp_comm_unique_id(hbp_ctx* ctx, unsigned char* out_id) {
    return cm_guarded(ctx, [&] {
        static_assert(sizeof(ncclUniqueId) == HBP_COMM_ID_BYTES, "ncclUniqueId size");
        ncclUniqueId id;
        nccl_check(need_nccl().get_unique_id(&id), "ncclGetUniqueId");
        std::memcpy(out_id, &id, sizeof(id));
    });
}

int hbp_comm_create(hbp_ctx* ctx, const unsigned char* id, int32_t rank, int32_t world, hbp_comm** out) {
    return cm_guarded(ctx, [&] {
        if (out == nullptr || id == nullptr) fail_validation("comm: null id or output");
        *out = nullptr;
        if (world < 1 || rank < 0 || rank >= world) fail_validation("comm: rank must lie in [0, world)");
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        auto* c = new hbp_comm();
        c->rank = rank;
        c->world = world;
        c->device = ctx->device;
        const ncclResult_t r = need_nccl().comm_init_rank(&c->comm, world, uid, rank);
        if (r != ncclSuccess) {
            delete c;
            nccl_check(r, "ncclCommInitRank");
        }
        *out = c;
    });
}

void hbp_comm_destroy(hbp_comm* comm) {
    if (comm == nullptr) return;
    if (comm->comm) {
        cudaSetDevice(comm->device);
        nccl().comm_destroy(comm->comm);
    }
    delete comm;
}

int hbp_sweep_sharded(hbp_ctx* ctx, hbp_comm* comm, const hbp_samples* samples, const hbp_group_config* cand_groups,
                      const int64_t* cand_offsets, const int64_t* cand_l_best, int64_t n_candidates,
                      const hbp_plan_options* options, const hbp_hardware_profile* profile, double* out_seconds,
                      int64_t* out_best, int64_t* out_local) {
    return cm_guarded(ctx, [&] {
        if (comm == nullptr) fail_validation("sweep_sharded: null communicator");
        const NcclApi& api = need_nccl();
        *out_best = -1;
        if (out_local) *out_local = 0;
        if (n_candidates <= 0) return;
        cudaStream_t s = ctx->stream;
        // the corpus is replicated: every rank validates it and fails the same
        // way before any collective
        DeviceCorpus corpus;
        sweep_ingest(*ctx, samples, corpus);
        const auto mine = sweep_shard(cand_groups, cand_offsets, n_candidates, comm->rank, comm->world);
        if (out_local) *out_local = static_cast<int64_t>(mine.size());
        const double inf = std::numeric_limits<double>::infinity();
        std::vector<double> secs(static_cast<size_t>(n_candidates), inf);
        std::vector<SweepErr> errs(static_cast<size_t>(n_candidates));
        sweep_evaluate(*ctx, corpus, cand_groups, cand_offsets, cand_l_best, mine, options, profile, secs, errs);

        // this rank's first error and best feasible candidate
        ErrRecord er{};
        er.index = std::numeric_limits<int64_t>::max();
        BestRecord br{inf, -1};
        for (int64_t k : mine) {
            const auto& e = errs[static_cast<size_t>(k)];
            if (e.code != HBP_OK && k < er.index) {
                er.index = k;
                er.code = e.code;
                er.len = static_cast<int32_t>(std::min<size_t>(e.msg.size(), sizeof(er.msg)));
                std::memcpy(er.msg, e.msg.data(), static_cast<size_t>(er.len));
            }
            const double t = secs[static_cast<size_t>(k)];
            if (std::isfinite(t) && (br.index < 0 || t < br.seconds)) br = {t, k};
        }
        const size_t W = static_cast<size_t>(comm->world);
        DevBuf<double> d_secs(static_cast<size_t>(n_candidates), s);
        DevBuf<char> d_err(sizeof(ErrRecord) * (W + 1), s), d_best(sizeof(BestRecord) * (W + 1), s);
        CUDA_CHECK(cudaMemcpyAsync(d_secs.p, secs.data(), sizeof(double) * secs.size(), cudaMemcpyHostToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(d_err.p, &er, sizeof(er), cudaMemcpyHostToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(d_best.p, &br, sizeof(br), cudaMemcpyHostToDevice, s));
        nccl_check(api.group_start(), "ncclGroupStart");
        nccl_check(api.all_reduce(d_secs.p, d_secs.p, secs.size(), ncclFloat64, ncclMin, comm->comm, s),
                   "ncclAllReduce");
        nccl_check(api.all_gather(d_err.p, d_err.p + sizeof(ErrRecord), sizeof(ErrRecord), ncclUint8, comm->comm, s),
                   "ncclAllGather");
        nccl_check(api.all_gather(d_best.p, d_best.p + sizeof(BestRecord), sizeof(BestRecord), ncclUint8,
                                  comm->comm, s),
                   "ncclAllGather");
        nccl_check(api.group_end(), "ncclGroupEnd");
        std::vector<ErrRecord> all_err(W);
        std::vector<BestRecord> all_best(W);
        CUDA_CHECK(cudaMemcpyAsync(all_err.data(), d_err.p + sizeof(ErrRecord), sizeof(ErrRecord) * W,
                                   cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaMemcpyAsync(all_best.data(), d_best.p + sizeof(BestRecord), sizeof(BestRecord) * W,
                                   cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaMemcpyAsync(out_seconds, d_secs.p, sizeof(double) * secs.size(), cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        // the error the sequential sweep would raise: the first in index order
        const ErrRecord* first = nullptr;
        for (const auto& e : all_err)
            if (e.index != std::numeric_limits<int64_t>::max() && (first == nullptr || e.index < first->index))
                first = &e;
        if (first) throw EngineError(first->code, std::string(first->msg, static_cast<size_t>(first->len)));
        // NCCL argmin: min seconds, lowest index on ties, infeasible loses
        BestRecord best{inf, -1};
        for (const auto& b : all_best)
            if (b.index >= 0 && (best.index < 0 || b.seconds < best.seconds ||
                                 (b.seconds == best.seconds && b.index < best.index)))
                best = b;
        *out_best = best.index;
    });
}

int hbp_eval_sharded(hbp_ctx* ctx, hbp_comm* comm, hbp_plan* plan, const hbp_hardware_profile* profile,
                     hbp_metrics* out, hbp_sim_totals* sim) {
    return cm_guarded(ctx, [&] {
        if (comm == nullptr || plan == nullptr) fail_validation("eval_sharded: null communicator or plan");
        const NcclApi& api = need_nccl();
        cudaStream_t s = ctx->stream;
        const DevicePlan& dp = plan->dp;
        const PlanArrays pa{dp.iter_group.p,    dp.iter_dev_offsets.p, dp.dev_pack_offsets.p,
                            dp.pack_capacity.p, dp.pack_total.p,       dp.pack_attention.p,
                            dp.n_iterations,    dp.n_devices};
        const size_t n = static_cast<size_t>(std::max<int64_t>(dp.n_iterations, 1));
        // rank r owns DP columns [r N / W, (r + 1) N / W) of every iteration
        const int32_t N = dp.device_count;
        const int32_t c0 = static_cast<int32_t>(static_cast<int64_t>(comm->rank) * N / comm->world);
        const int32_t c1 = static_cast<int32_t>(static_cast<int64_t>(comm->rank + 1) * N / comm->world);
        // 7 int64 vectors + busy (f64) + sim_err, zeroed on the context stream
        DevBuf<int64_t> iv(7 * n + 1, s);
        DevBuf<double> busy(n, s);
        CUDA_CHECK(cudaMemsetAsync(iv.p, 0, sizeof(int64_t) * (7 * n + 1), s));
        CUDA_CHECK(cudaMemsetAsync(busy.p, 0, sizeof(double) * n, s));
        hbp_eval_columns_bufs b{};
        b.tmax = iv.p;
        b.amax = iv.p + n;
        b.tokens = iv.p + 2 * n;
        b.pad_gap = iv.p + 3 * n;
        b.pad_cap = iv.p + 4 * n;
        b.tgap = iv.p + 5 * n;
        b.agap = iv.p + 6 * n;
        b.sim_err = iv.p + 7 * n;
        b.busy = busy.p;
        eval_columns(*ctx, pa, dp.groups, profile, 0, c0, c1, b);
        nccl_check(api.group_start(), "ncclGroupStart");
        nccl_check(api.all_reduce(b.tmax, b.tmax, 2 * n, ncclInt64, ncclMax, comm->comm, s), "ncclAllReduce");
        nccl_check(api.all_reduce(b.tokens, b.tokens, 3 * n, ncclInt64, ncclSum, comm->comm, s), "ncclAllReduce");
        if (profile) {
            nccl_check(api.all_reduce(b.busy, b.busy, n, ncclFloat64, ncclMax, comm->comm, s), "ncclAllReduce");
            nccl_check(api.all_reduce(b.sim_err, b.sim_err, 1, ncclInt64, ncclMin, comm->comm, s), "ncclAllReduce");
        }
        nccl_check(api.group_end(), "ncclGroupEnd");
        eval_columns(*ctx, pa, dp.groups, profile, 1, c0, c1, b);  // same stream: after the exchange
        nccl_check(api.all_reduce(b.tgap, b.tgap, 2 * n, ncclInt64, ncclSum, comm->comm, s), "ncclAllReduce");
        EvalOut eo;
        eval_columns_finish(*ctx, pa, N, dp.groups, profile, b, eo);
        if (out) *out = eo.m;
        if (sim && profile) {
            sim->metrics = eo.m;
            sim->total_seconds = eo.total_seconds;
            sim->gpu_days = eo.total_seconds * static_cast<double>(N) / 86400.0;
            sim->switch_count = eo.switch_count;
            sim->device_count = N;
        }
    });
}

}  // extern "C"
