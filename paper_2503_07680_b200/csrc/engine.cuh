// engine.cuh — the per-context state and the stage entry points of the
// B200 batch-construction engine. One context = one CUDA stream; all
// scratch is stream-ordered (cudaMallocAsync) so stages queue back to back
// and the host only synchronises where a data-dependent size is needed.
#pragma once

#include <string>
#include <vector>

#include "common.cuh"
#include "scan.cuh"

#include <chrono>
#include <cstring>
#include <cstdlib>
#include <map>
#include <set>

struct hbp_plan;

struct hbp_ctx {
    // plans created on this context; their device arrays are freed (stream
    // ordered) before the stream goes away, their host views stay readable
    std::set<hbp_plan*> plans;
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string last_error;
    int64_t launches = 0;
    int64_t syncs = 0;  // host round trips (read_scalar / read_vector)
    hbp_b200::BlockCache blocks;  // declared before every cached buffer it outlives
    hbp_b200::ScanScratch scan;
    // a second stream for stages independent of the one in flight (e.g. the
    // greedy-fill pool sort while the larger group packs); its scans use
    // their own status ring. Created on first use.
    cudaStream_t side = nullptr;
    hbp_b200::ScanScratch side_scan;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool side_off = false;  // HBP_NO_SIDE: forks run inline on the main stream
    std::vector<hbp_ctx*> workers;  // the sweep's worker contexts (kept warm; destroyed with this one)
    // host round trips wait on a blocking-sync event instead of spinning
    // (the sweep's many worker threads would otherwise spin on the host cores
    // they need for launching)
    bool blocking_sync = false;
    cudaEvent_t ev_sync = nullptr;
    hbp_b200::Pinned pinned;
    hbp_b200::PinnedPool host_pool;  // plan host views
    // stage trace (HBP_TRACE=1): wall time between marks, stream synchronised
    bool trace = std::getenv("HBP_TRACE") != nullptr;
    std::map<std::string, double> trace_ms;
    std::chrono::steady_clock::time_point trace_last{};
    hbp_b200::KernelProfiler prof;
    // tests only (hbp_test_set_force_reject): the Fisher-Yates step whose
    // first draw is treated as rejected; 0 = none
    uint64_t test_force_reject = 0;
};

namespace hbp_b200 {

using Ctx = hbp_ctx;

inline void trace_begin(Ctx& c) {
    if (!c.trace) return;
    cudaStreamSynchronize(c.stream);
    c.trace_last = std::chrono::steady_clock::now();
}
inline void trace_mark(Ctx& c, const char* stage) {
    if (!c.trace) return;
    cudaStreamSynchronize(c.stream);
    const auto now = std::chrono::steady_clock::now();
    c.trace_ms[stage] += std::chrono::duration<double, std::milli>(now - c.trace_last).count();
    c.trace_last = now;
}
inline void trace_dump(Ctx& c, const char* title) {
    if (!c.trace) return;
    double tot = 0;
    for (auto& kv : c.trace_ms) tot += kv.second;
    std::fprintf(stderr, "[hbp trace] %s: %.3f ms\n", title, tot);
    for (auto& kv : c.trace_ms) std::fprintf(stderr, "[hbp trace]   %-28s %9.3f ms\n", kv.first.c_str(), kv.second);
    c.trace_ms.clear();
}

// Makes `ctx` the current launch-count sink and device for this thread.
struct CtxScope {
    int64_t* prev;
    KernelProfiler* prev_prof;
    BlockCache* prev_cache;
    explicit CtxScope(Ctx& c) : prev(g_launch_counter), prev_prof(g_prof), prev_cache(g_cache) {
        g_launch_counter = &c.launches;
        g_prof = &c.prof;
        c.blocks.stream = c.stream;
        g_cache = &c.blocks;
        CUDA_CHECK(cudaSetDevice(c.device));
    }
    ~CtxScope() {
        g_launch_counter = prev;
        g_prof = prev_prof;
        g_cache = prev_cache;
    }
};

// Fork / join of the context's side stream: work enqueued inside a
// SideScope runs on the side stream after everything enqueued on the main
// stream before fork(); join() makes the main stream wait for it. Buffers
// that cross the two are allocated on the main stream before the fork and
// released after the join; buffers allocated inside a SideScope are the side
// stream's own (stream-ordered there, outside the main stream's cache).
inline void side_fork(Ctx& c) {
    static const bool no_side = std::getenv("HBP_NO_SIDE") != nullptr;  // A/B: everything on one stream
    if (no_side) {
        c.side_off = true;
        return;
    }
    if (!c.side) {
        int lo = 0, hi = 0;  // lowest priority (the main stream has the highest)
        CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CUDA_CHECK(cudaStreamCreateWithPriority(&c.side, cudaStreamNonBlocking, lo));
        CUDA_CHECK(cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming));
        CUDA_CHECK(cudaEventCreateWithFlags(&c.ev_join, cudaEventDisableTiming));
    }
    CUDA_CHECK(cudaEventRecord(c.ev_fork, c.stream));
    CUDA_CHECK(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
}
inline void side_join(Ctx& c) {
    if (c.side_off) return;
    CUDA_CHECK(cudaEventRecord(c.ev_join, c.side));
    CUDA_CHECK(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
}
// Joins a fork when it goes out of scope (also on an exception), so that
// buffers declared before it are released only after the side stream is done.
struct SideJoin {
    Ctx& c;
    bool armed = false;
    explicit SideJoin(Ctx& cc) : c(cc) {}
    void join() {
        if (armed) side_join(c);
        armed = false;
    }
    ~SideJoin() {
        if (armed && !c.side_off) {
            cudaEventRecord(c.ev_join, c.side);
            cudaStreamWaitEvent(c.stream, c.ev_join, 0);
        }
    }
};
struct SideScope {
    Ctx& c;
    explicit SideScope(Ctx& cc) : c(cc) {
        if (c.side_off) return;
        std::swap(c.stream, c.side);
        std::swap(c.scan, c.side_scan);
    }
    ~SideScope() {
        if (c.side_off) return;
        std::swap(c.stream, c.side);
        std::swap(c.scan, c.side_scan);
    }
};

// Waits for the context's stream (spinning, or on a blocking-sync event).
inline void ctx_sync(Ctx& c) {
    if (!c.blocking_sync) {
        CUDA_CHECK(cudaStreamSynchronize(c.stream));
        return;
    }
    if (!c.ev_sync) CUDA_CHECK(cudaEventCreateWithFlags(&c.ev_sync, cudaEventBlockingSync | cudaEventDisableTiming));
    CUDA_CHECK(cudaEventRecord(c.ev_sync, c.stream));
    CUDA_CHECK(cudaEventSynchronize(c.ev_sync));
}

// Copies a few device scalars to host (one sync).
template <typename T>
T read_scalar(Ctx& c, const T* dptr) {
    c.pinned.ensure(sizeof(T));
    ++c.syncs;
    CUDA_CHECK(cudaMemcpyAsync(c.pinned.p, dptr, sizeof(T), cudaMemcpyDeviceToHost, c.stream));
    ctx_sync(c);
    return *reinterpret_cast<T*>(c.pinned.p);
}

// Host <-> device copies of pageable host memory through two pinned blocks
// of the context's pool: chunk k + 1 crosses PCIe while chunk k is copied on
// the host. Synchronous on return.
inline void staged_copy(Ctx& c, void* dst, const void* src, size_t n, bool to_device) {
    if (n == 0) return;
    constexpr size_t kChunk = size_t(32) << 20;
    if (n <= kChunk / 8) {  // small: one pageable copy
        CUDA_CHECK(cudaMemcpyAsync(dst, src, n, to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, c.stream));
        CUDA_CHECK(cudaStreamSynchronize(c.stream));
        return;
    }
    HostBlock stage[2] = {c.host_pool.acquire(std::min(kChunk, n)), c.host_pool.acquire(std::min(kChunk, n))};
    cudaEvent_t done[2];
    CUDA_CHECK(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
    CUDA_CHECK(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
    const size_t chunks = (n + kChunk - 1) / kChunk;
    auto* d = static_cast<char*>(dst);
    const auto* h = static_cast<const char*>(src);
    auto len = [&](size_t k) { return std::min(kChunk, n - k * kChunk); };
    if (to_device) {
        for (size_t k = 0; k < chunks; ++k) {
            if (k >= 2) CUDA_CHECK(cudaEventSynchronize(done[k & 1]));  // block k - 2 has crossed
            std::memcpy(stage[k & 1].p, h + k * kChunk, len(k));
            CUDA_CHECK(cudaMemcpyAsync(d + k * kChunk, stage[k & 1].p, len(k), cudaMemcpyHostToDevice, c.stream));
            CUDA_CHECK(cudaEventRecord(done[k & 1], c.stream));
        }
        CUDA_CHECK(cudaStreamSynchronize(c.stream));
    } else {
        auto issue = [&](size_t k) {
            CUDA_CHECK(cudaMemcpyAsync(stage[k & 1].p, d + k * kChunk, len(k), cudaMemcpyDeviceToHost, c.stream));
            CUDA_CHECK(cudaEventRecord(done[k & 1], c.stream));
        };
        auto* out = static_cast<char*>(dst);
        const auto* dev = static_cast<const char*>(src);
        d = const_cast<char*>(dev);
        issue(0);
        for (size_t k = 0; k < chunks; ++k) {
            if (k + 1 < chunks) issue(k + 1);
            CUDA_CHECK(cudaEventSynchronize(done[k & 1]));
            std::memcpy(out + k * kChunk, stage[k & 1].p, len(k));
        }
    }
    CUDA_CHECK(cudaEventDestroy(done[0]));
    CUDA_CHECK(cudaEventDestroy(done[1]));
    c.host_pool.release(stage[0]);
    c.host_pool.release(stage[1]);
}

template <typename T>
std::vector<T> read_vector(Ctx& c, const T* dptr, size_t n) {
    // through the context's pinned staging buffer: a copy into pageable
    // memory serialises with other streams' work on the device
    std::vector<T> out(n);
    ++c.syncs;
    if (n) {
        c.pinned.ensure(sizeof(T) * n);
        CUDA_CHECK(cudaMemcpyAsync(c.pinned.p, dptr, sizeof(T) * n, cudaMemcpyDeviceToHost, c.stream));
        ctx_sync(c);
        std::memcpy(out.data(), c.pinned.p, sizeof(T) * n);
    }
    return out;
}

// Generic element-wise launch: f(i) for i in [0, n).
template <typename F>
__global__ void k_for_each(u64 n, F f) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<u64>(gridDim.x) * blockDim.x)
        f(i);
}
template <typename F>
void for_each_index(Ctx& c, u64 n, F f) {
    if (n == 0) return;
    LAUNCH(k_for_each<F>, grid_for(n, 256, 148u * 16u), 256, 0, c.stream, n, f);
}

// ---- stage: exact Fisher-Yates (shuffle.cu) --------------------------------
// src[p] = the input position whose element Rng(seed).shuffle() leaves at
// output position p, for a vector of m elements (reference rng.hpp:61-68).
// draw_base: draws of the same Rng already consumed (a second shuffle with
// one generator, schedule.cpp:39-48); draws_used: draws this one consumed.
void fy_source_positions(Ctx& c, uint64_t seed, i64 m, u32* src, uint64_t draw_base = 0,
                         uint64_t* draws_used = nullptr);
// out[p] = in[src[p]] for 8-byte elements.
void gather_u64(Ctx& c, const u64* in, const u32* src, u64* out, i64 m);
// out = in permuted by the exact Fisher-Yates of `seed` (fy_source_positions
// + gather in one pass: out[p] = in[src(p)])
void fy_shuffle_u64(Ctx& c, uint64_t seed, i64 m, const u64* in, u64* out);
void gather_u32(Ctx& c, const u32* in, const u32* src, u32* out, i64 m);

}  // namespace hbp_b200
