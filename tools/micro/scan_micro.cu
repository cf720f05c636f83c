// Micro-benchmark of the decoupled look-back scan (scan.cuh): GB/s of a
// plain exclusive scan over u64 / u32 arrays, against a device copy.
//   nvcc -O3 -std=c++17 --extended-lambda -gencode arch=compute_100a,code=sm_100a \
//        -I include -o tools/micro/scan_micro tools/micro/scan_micro.cu
#include "../../paper_2503_07680_b200/csrc/scan.cuh"

#include <cstdlib>

namespace hbp_b200 {
thread_local int64_t* g_launch_counter = nullptr;
thread_local KernelProfiler* g_prof = nullptr;
thread_local BlockCache* g_cache = nullptr;
}  // namespace hbp_b200

using namespace hbp_b200;

template <typename T, int ITEMS, int BLOCK = 256>
float time_scan(i64 n, const T* in, T* out, ScanScratch& sc, cudaStream_t s, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&] {
        scan_exclusive<T, ITEMS, BLOCK>(
            n, [=] __device__(i64 i) { return in[i]; }, [=] __device__(i64 i, T v) { out[i] = v; }, s, sc);
    };
    run();
    cudaEventRecord(a, s);
    for (int r = 0; r < reps; ++r) run();
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main(int argc, char** argv) {
    const i64 n = argc > 1 ? std::atoll(argv[1]) : 10000000;
    cudaStream_t s;
    cudaStreamCreate(&s);
    u64 *in, *out;
    cudaMalloc(&in, n * 8);
    cudaMalloc(&out, n * 8);
    cudaMemset(in, 1, n * 8);
    ScanScratch sc;
    const int reps = 20;
    {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaMemcpyAsync(out, in, n * 8, cudaMemcpyDeviceToDevice, s);
        cudaEventRecord(a, s);
        for (int r = 0; r < reps; ++r) cudaMemcpyAsync(out, in, n * 8, cudaMemcpyDeviceToDevice, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= reps;
        std::printf("n=%lld memcpy u64: %.1f us, %.0f GB/s\n", (long long)n, ms * 1e3, 16.0 * n / ms / 1e6);
    }
    float ms;
    ms = time_scan<u64, 4>(n, in, out, sc, s, reps);
    std::printf("scan u64 ITEMS 4 : %.1f us, %.0f GB/s\n", ms * 1e3, 16.0 * n / ms / 1e6);
    ms = time_scan<u64, 8>(n, in, out, sc, s, reps);
    std::printf("scan u64 ITEMS 8 : %.1f us, %.0f GB/s\n", ms * 1e3, 16.0 * n / ms / 1e6);
    ms = time_scan<u64, 16>(n, in, out, sc, s, reps);
    std::printf("scan u64 ITEMS 16: %.1f us, %.0f GB/s\n", ms * 1e3, 16.0 * n / ms / 1e6);
    ms = time_scan<u64, 16, 512>(n, in, out, sc, s, reps);
    std::printf("scan u64 ITEMS 16 x 512: %.1f us, %.0f GB/s\n", ms * 1e3, 16.0 * n / ms / 1e6);
    ms = time_scan<u64, 32, 256>(n, in, out, sc, s, reps);
    std::printf("scan u64 ITEMS 32 x 256: %.1f us, %.0f GB/s\n", ms * 1e3, 16.0 * n / ms / 1e6);
    ms = time_scan<u32, 8>(n, reinterpret_cast<u32*>(in), reinterpret_cast<u32*>(out), sc, s, reps);
    std::printf("scan u32 ITEMS 8 : %.1f us, %.0f GB/s\n", ms * 1e3, 8.0 * n / ms / 1e6);
    ms = time_scan<u32, 16>(n, reinterpret_cast<u32*>(in), reinterpret_cast<u32*>(out), sc, s, reps);
    std::printf("scan u32 ITEMS 16: %.1f us, %.0f GB/s\n", ms * 1e3, 8.0 * n / ms / 1e6);
    ms = time_scan<u32, 32>(n, reinterpret_cast<u32*>(in), reinterpret_cast<u32*>(out), sc, s, reps);
    std::printf("scan u32 ITEMS 32: %.1f us, %.0f GB/s\n", ms * 1e3, 8.0 * n / ms / 1e6);
    ms = time_scan<u32, 32, 512>(n, reinterpret_cast<u32*>(in), reinterpret_cast<u32*>(out), sc, s, reps);
    std::printf("scan u32 ITEMS 32 x 512: %.1f us, %.0f GB/s\n", ms * 1e3, 8.0 * n / ms / 1e6);
    std::printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
