// common.cuh — shared plumbing for the HBP B200 engine: error handling, the
// per-context stream and scratch allocator, launch accounting, and small
// device helpers. Everything here is host/device infrastructure; the
// algorithms live in the stage files (shuffle.cu, nextfit.cu, firstfit.cu,
// batching.cu, metrics.cu, costmodel.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <map>
#include <mutex>
#include <set>
#include <stdexcept>
#include <utility>
#include <string>
#include <vector>

#include "../../include/hbp_b200.h"

namespace hbp_b200 {

using u8 = uint8_t;
using u32 = uint32_t;
using u64 = uint64_t;
using i64 = int64_t;

constexpr int kSMs = 148;          // B200: 2 dies x 74 SMs
constexpr u32 kNone = 0xffffffffu; // "no element" sentinel for u32 links

// Engine errors carry the reference's status code and exact message.
struct EngineError : std::runtime_error {
    int code;
    EngineError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail_validation(const std::string& m) { throw EngineError(HBP_ERR_VALIDATION, m); }
[[noreturn]] inline void fail_infeasible(const std::string& m) { throw EngineError(HBP_ERR_INFEASIBLE, m); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        throw EngineError(HBP_ERR_CUDA, std::string("CUDA error in ") + what + " (" + file + ":" +
                                            std::to_string(line) + "): " + cudaGetErrorString(e));
    }
}
#define CUDA_CHECK(x) ::hbp_b200::cuda_check((x), #x, __FILE__, __LINE__)

// Function attributes and occupancy are per (kernel, device) and do not
// change: set / query them once per process instead of on every launch
// (these driver calls take a context-wide lock that the sweep's worker
// threads would queue on).
inline void set_max_dynamic_smem_once(const void* func, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    if (done.count({func, dev})) return;
    CUDA_CHECK(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done.insert({func, dev});
}

// Per-context cache of device blocks. Every stage allocates its scratch
// per call; on one stream a block freed by an earlier stage can be handed
// to a later one right away (stream order), so after warm-up a call makes
// no allocator API calls at all -- at sweep sizes (100K samples per plan)
// those calls, not the kernels, were the cost. Sizes are rounded to a
// quarter power of two (<= 25% slack); beyond kLimit cached bytes, blocks
// go back to the stream-ordered pool.
struct BlockCache {
    cudaStream_t stream = nullptr;
    // the owning context's own stream-ordered pool (null: the device's
    // default pool). A private pool never hands a context a block another
    // context freed, so contexts building plans at once never wait on each
    // other's streams through the allocator.
    cudaMemPool_t pool = nullptr;
    std::map<size_t, std::vector<void*>> free_blocks;
    size_t cached = 0;
    static constexpr size_t kLimit = size_t(16) << 30;
    static size_t round(size_t bytes) {
        size_t c = bytes < 512 ? 512 : bytes;
        size_t p = 1;
        while ((p << 1) <= c) p <<= 1;
        const size_t step = p / 4 < 512 ? 512 : p / 4;
        return (c + step - 1) / step * step;
    }
    void* get(size_t rounded) {
        auto it = free_blocks.find(rounded);
        if (it != free_blocks.end() && !it->second.empty()) {
            void* q = it->second.back();
            it->second.pop_back();
            cached -= rounded;
            return q;
        }
        void* q = nullptr;
        if (pool) CUDA_CHECK(cudaMallocFromPoolAsync(&q, rounded, pool, stream));
        else CUDA_CHECK(cudaMallocAsync(&q, rounded, stream));
        return q;
    }
    void put(void* q, size_t rounded) {
        if (cached + rounded > kLimit) {
            cudaFreeAsync(q, stream);
            return;
        }
        free_blocks[rounded].push_back(q);
        cached += rounded;
    }
    void clear() {
        for (auto& kv : free_blocks)
            for (void* q : kv.second) cudaFreeAsync(q, stream);
        free_blocks.clear();
        cached = 0;
    }
};
// The cache of the context this thread is running (set by CtxScope).
extern thread_local BlockCache* g_cache;

// Stream-ordered device buffer owned by a context (block cache over the
// cudaMallocAsync pool).
template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    BlockCache* cache = nullptr;  // where the block goes back
    size_t bytes = 0;             // rounded block size (cached blocks)
    DevBuf() = default;
    DevBuf(size_t count, cudaStream_t stream) { alloc(count, stream); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s), cache(o.cache), bytes(o.bytes) {
        o.p = nullptr;
        o.n = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p; n = o.n; s = o.s; cache = o.cache; bytes = o.bytes;
            o.p = nullptr; o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count, cudaStream_t stream) {
        release();
        s = stream;
        n = count;
        if (!count) return;
        if (g_cache && g_cache->stream == stream) {
            cache = g_cache;
            bytes = BlockCache::round(sizeof(T) * count);
            p = static_cast<T*>(cache->get(bytes));
        } else {
            cache = nullptr;
            if (g_cache && g_cache->pool)
                CUDA_CHECK(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p), sizeof(T) * count, g_cache->pool,
                                                   stream));
            else
                CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * count, stream));
        }
    }
    void release() {
        if (p) {
            if (cache) cache->put(p, bytes);
            else cudaFreeAsync(p, s);
        }
        p = nullptr;
        n = 0;
    }
    T* get() const { return p; }
    void zero() const {
        if (n) CUDA_CHECK(cudaMemsetAsync(p, 0, sizeof(T) * n, s));
    }
};

// Pinned host staging buffer for small readbacks.
struct Pinned {
    void* p = nullptr;
    size_t bytes = 0;
    void ensure(size_t b) {
        if (b <= bytes) return;
        if (p) cudaFreeHost(p);
        CUDA_CHECK(cudaMallocHost(&p, b));
        bytes = b;
    }
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
};

// Pinned host blocks recycled across calls (plan host views): pinning
// memory costs far more than copying into it.
struct HostBlock {
    void* p = nullptr;
    size_t bytes = 0;
};

struct PinnedPool {
    std::vector<HostBlock> free_blocks;
    static constexpr size_t kKeep = 4;
    HostBlock acquire(size_t bytes) {
        size_t best = free_blocks.size();
        for (size_t i = 0; i < free_blocks.size(); ++i)
            if (free_blocks[i].bytes >= bytes && (best == free_blocks.size() || free_blocks[i].bytes < free_blocks[best].bytes))
                best = i;
        if (best < free_blocks.size()) {
            HostBlock b = free_blocks[best];
            free_blocks.erase(free_blocks.begin() + static_cast<std::ptrdiff_t>(best));
            return b;
        }
        HostBlock b;
        b.bytes = bytes + bytes / 4 + 4096;
        CUDA_CHECK(cudaMallocHost(&b.p, b.bytes));
        return b;
    }
    void release(HostBlock b) {
        if (!b.p) return;
        free_blocks.push_back(b);
        if (free_blocks.size() > kKeep) {  // drop the smallest
            size_t s = 0;
            for (size_t i = 1; i < free_blocks.size(); ++i)
                if (free_blocks[i].bytes < free_blocks[s].bytes) s = i;
            cudaFreeHost(free_blocks[s].p);
            free_blocks.erase(free_blocks.begin() + static_cast<std::ptrdiff_t>(s));
        }
    }
    ~PinnedPool() {
        for (auto& b : free_blocks) cudaFreeHost(b.p);
    }
};

// ---------------------------------------------------------------------------
// kernel launch accounting (bench.py reports gpu_launches)
// ---------------------------------------------------------------------------
extern thread_local int64_t* g_launch_counter;
inline void count_launch() {
    if (g_launch_counter) ++*g_launch_counter;
}

inline unsigned grid_for(size_t n, unsigned block, unsigned cap = 148u * 16u) {
    size_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return static_cast<unsigned>(g);
}

#define LAUNCH(kernel, grid, block, smem, stream, ...) LAUNCH_B(#kernel, 0.0, kernel, grid, block, smem, stream, __VA_ARGS__)

// Per-kernel-family device time (CUDA events on the launching stream) and
// algorithmic bytes, collected only while profiling is switched on
// (hbp_ctx_set_profiling). Feeds bench.py's roofline.
struct KernelProfiler {
    bool on = false;
    struct Rec {
        const char* name;
        cudaEvent_t a, b;
        double bytes;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> spare;
    cudaEvent_t event() {
        if (!spare.empty()) {
            cudaEvent_t e = spare.back();
            spare.pop_back();
            return e;
        }
        cudaEvent_t e;
        CUDA_CHECK(cudaEventCreate(&e));
        return e;
    }
    ~KernelProfiler() {
        for (auto& r : recs) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        for (auto e : spare) cudaEventDestroy(e);
    }
};
extern thread_local KernelProfiler* g_prof;

#define LAUNCH_B(name, bytes, kernel, grid, block, smem, stream, ...)                       \
    do {                                                                                    \
        ::hbp_b200::KernelProfiler* _p = ::hbp_b200::g_prof;                                \
        const bool _on = _p && _p->on;                                                      \
        cudaEvent_t _e0 = nullptr;                                                          \
        if (_on) {                                                                          \
            _e0 = _p->event();                                                              \
            CUDA_CHECK(cudaEventRecord(_e0, (stream)));                                     \
        }                                                                                   \
        kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                        \
        ::hbp_b200::count_launch();                                                         \
        CUDA_CHECK(cudaGetLastError());                                                     \
        if (_on) {                                                                          \
            cudaEvent_t _e1 = _p->event();                                                  \
            CUDA_CHECK(cudaEventRecord(_e1, (stream)));                                     \
            _p->recs.push_back({(name), _e0, _e1, static_cast<double>(bytes)});             \
        }                                                                                   \
    } while (0)

// Cooperative launch (all CTAs co-resident, or cudaErrorCooperativeLaunchTooLarge).
#define LAUNCH_COOP(name, bytes, kernel, grid, block, smem, stream, args)                   \
    do {                                                                                    \
        ::hbp_b200::KernelProfiler* _p = ::hbp_b200::g_prof;                                \
        const bool _on = _p && _p->on;                                                      \
        cudaEvent_t _e0 = nullptr;                                                          \
        if (_on) {                                                                          \
            _e0 = _p->event();                                                              \
            CUDA_CHECK(cudaEventRecord(_e0, (stream)));                                     \
        }                                                                                   \
        CUDA_CHECK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kernel), (grid), \
                                               (block), (args), (smem), (stream)));         \
        ::hbp_b200::count_launch();                                                         \
        if (_on) {                                                                          \
            cudaEvent_t _e1 = _p->event();                                                  \
            CUDA_CHECK(cudaEventRecord(_e1, (stream)));                                     \
            _p->recs.push_back({(name), _e0, _e1, static_cast<double>(bytes)});             \
        }                                                                                   \
    } while (0)

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned warp_id() { return threadIdx.x >> 5; }

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane_id() >= static_cast<unsigned>(o)) v += t;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        T t = __shfl_xor_sync(0xffffffffu, v, o);
        v = t > v ? t : v;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        T t = __shfl_xor_sync(0xffffffffu, v, o);
        v = t < v ? t : v;
    }
    return v;
}

// Block-wide exclusive scan (blockDim.x multiple of 32, <= 1024). `total`
// receives the block sum. Uses 33 words of the provided shared scratch.
template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* smem, T& total) {
    const unsigned lane = lane_id(), wid = warp_id(), nw = blockDim.x >> 5;
    T inc = warp_inclusive_scan(v);
    if (lane == 31) smem[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        T w = lane < nw ? smem[lane] : T(0);
        T wi = warp_inclusive_scan(w);
        if (lane < nw) smem[lane] = wi - w;
        if (lane == nw - 1) smem[32] = wi;
    }
    __syncthreads();
    T out = smem[wid] + inc - v;
    total = smem[32];
    __syncthreads();
    return out;
}

}  // namespace hbp_b200
