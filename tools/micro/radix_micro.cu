// Micro-benchmark of the stable LSD radix sort (radix.cu): 10M / 100M
// (u32 key, u32 value) pairs, 24-bit keys (three 8-bit passes).
//   nvcc -O3 -std=c++17 --extended-lambda -gencode arch=compute_100a,code=sm_100a \
//        -I include -o tools/micro/radix_micro tools/micro/radix_micro.cu
#include "../../paper_2503_07680_b200/csrc/radix.cu"

#include <cstdlib>
#include <vector>

namespace hbp_b200 {
thread_local int64_t* g_launch_counter = nullptr;
thread_local KernelProfiler* g_prof = nullptr;
thread_local BlockCache* g_cache = nullptr;
}  // namespace hbp_b200

using namespace hbp_b200;

int main(int argc, char** argv) {
    const i64 n = argc > 1 ? std::atoll(argv[1]) : 10000000;
    const int bits = argc > 2 ? std::atoi(argv[2]) : 24;
    hbp_ctx c;
    cudaStreamCreate(&c.stream);
    std::vector<u32> hk(n), hv(n);
    uint64_t x = 88172645463325252ull;
    for (i64 i = 0; i < n; ++i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        hk[i] = static_cast<u32>(x) & ((bits >= 32) ? 0xffffffffu : ((1u << bits) - 1));
        hv[i] = static_cast<u32>(i);
    }
    u32 *k0, *v0, *k, *v, *tk, *tv;
    cudaMalloc(&k0, n * 4); cudaMalloc(&v0, n * 4); cudaMalloc(&k, n * 4); cudaMalloc(&v, n * 4);
    cudaMalloc(&tk, n * 4); cudaMalloc(&tv, n * 4);
    cudaMemcpy(k0, hk.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(v0, hv.data(), n * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e9;
    for (int r = 0; r < 6; ++r) {
        cudaMemcpyAsync(k, k0, n * 4, cudaMemcpyDeviceToDevice, c.stream);
        cudaMemcpyAsync(v, v0, n * 4, cudaMemcpyDeviceToDevice, c.stream);
        cudaEventRecord(a, c.stream);
        radix_sort_pairs(c, k, v, n, bits, false, tk, tv);
        cudaEventRecord(b, c.stream);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r > 0 && ms < best) best = ms;
    }
    std::vector<u32> ok(n), ov(n);
    cudaMemcpy(ok.data(), k, n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(ov.data(), v, n * 4, cudaMemcpyDeviceToHost);
    bool sorted = true;
    for (i64 i = 1; i < n && sorted; ++i)
        sorted = ok[i - 1] < ok[i] || (ok[i - 1] == ok[i] && ov[i - 1] < ov[i]);
    const int passes = (bits + 7) / 8;
    std::printf("n=%lld bits=%d: %.1f us, %.1f us/pass, %.0f GB/s per pass (16 B/elem), stable-sorted %s\n",
                (long long)n, bits, best * 1e3, best * 1e3 / passes, 16.0 * n * passes / best / 1e6,
                sorted ? "yes" : "NO");
    return 0;
}
