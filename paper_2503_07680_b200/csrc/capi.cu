// capi.cpp — the extern "C" boundary (include/hbp_b200.h). Every entry point
// converts exceptions into the reference's status codes and keeps the exact
// message on the context; the work itself is queued on the context stream.
#include <cstring>
#include <string>

#include "../../include/hbp_b200.h"
#include "../../include/hbp_b200_testing.h"
#include "engine.cuh"
#include "radix.cuh"

namespace hbp_b200 {
thread_local int64_t* g_launch_counter = nullptr;
}

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
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return HBP_ERR_CUDA;
    }
    if (device < 0 || device >= count) return HBP_ERR_VALIDATION;
    auto* c = new hbp_ctx();
    c->device = device;
    if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        delete c;
        return HBP_ERR_CUDA;
    }
    // keep freed scratch in the stream-ordered pool between calls
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t threshold = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
    }
    *out = c;
    return HBP_OK;
}

void hbp_ctx_destroy(hbp_ctx* ctx) {
    if (ctx == nullptr) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) {
        cudaStreamSynchronize(ctx->stream);
        ctx->scan.status.release();
        ctx->scan.counter.release();
        cudaStreamSynchronize(ctx->stream);
        cudaStreamDestroy(ctx->stream);
    }
    delete ctx;
}

const char* hbp_last_error(const hbp_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

int hbp_ctx_synchronize(hbp_ctx* ctx) {
    return guarded(ctx, [&] { CUDA_CHECK(cudaStreamSynchronize(ctx->stream)); });
}

void* hbp_ctx_stream(hbp_ctx* ctx) { return ctx ? reinterpret_cast<void*>(ctx->stream) : nullptr; }

int64_t hbp_ctx_launch_count(const hbp_ctx* ctx) { return ctx ? ctx->launches : 0; }

// ---- testing hooks ----------------------------------------------------------

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
