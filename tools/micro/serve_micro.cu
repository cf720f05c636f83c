// Micro-benchmark of the first-fit chain's per-block serve (one warp, no
// hand-off): cycles per served run for bins/runs shaped like the C2 FFD and
// greedy-fill launches.
//   nvcc -O3 -std=c++17 --extended-lambda -gencode arch=compute_100a,code=sm_100a \
//        -I include -o tools/micro/serve_micro tools/micro/serve_micro.cu
#include "../../paper_2503_07680_b200/csrc/chain.cu"

#include <random>

namespace hbp_b200 {
thread_local int64_t* g_launch_counter = nullptr;
thread_local KernelProfiler* g_prof = nullptr;
thread_local BlockCache* g_cache = nullptr;

template <int M>
__global__ void k_serve_micro(ChainArgs a, const u32* R0, const u32* s_in, const u32* c_in, int iters,
                              unsigned long long* out) {
    const u32 lane = threadIdx.x & 31u;
    u32 R[M], N[M];
    unsigned long long tot = 0, runs = 0;
    for (int it = 0; it < iters; ++it) {
        u32 lmax = 0;
#pragma unroll
        for (int i = 0; i < M; ++i) {
            R[i] = R0[(it % 64) * 32 * M + lane * M + i];
            N[i] = 0;
            lmax = max(lmax, R[i]);
        }
        u32 wmax = __reduce_max_sync(0xffffffffu, lmax);
        const u32 s = s_in[(it % 64) * 32 + lane];
        u32 c = c_in[(it % 64) * 32 + lane];
        const unsigned act = __ballot_sync(0xffffffffu, c > 0 && s <= wmax);
        __syncwarp();
        const long long t0 = clock64();
        serve<M, false>(a, act, s, 1000000u, c, R, N, wmax, 0, lane);
        __syncwarp();
        const long long t1 = clock64();
        tot += t1 - t0;
        runs += __popc(act);
        if (c == 12345u) out[2] = wmax;  // keep results alive
    }
    if (lane == 0) {
        out[0] = tot;
        out[1] = runs;
    }
}

}  // namespace hbp_b200

using namespace hbp_b200;

int main(int argc, char** argv) {
    const int only = argc > 1 ? std::atoi(argv[1]) : -1;
    int idx = -1;
    constexpr int M = 8;
    struct Shape { const char* name; u32 cap, rlo, rhi, slo, shi, clo, chi; };
    const Shape shapes[] = {
        {"g1-ffd-like (cap 128K, s 16K-64K, c 1-8)", 131072, 0, 65536, 16384, 65536, 1, 8},
        {"g0-ffd-like (cap 16K, s 2K-6K, c 20-80)", 16384, 0, 12000, 2000, 6000, 20, 80},
        {"fill-like (cap 16K, s 100-2K, c 100-1000)", 16384, 0, 4000, 100, 2000, 100, 1000},
        {"one lane per run (R 6-12K, s 5-6K, c 1-4)", 16384, 6000, 12000, 5000, 6000, 1, 4},
        {"two lanes per run (R 6-12K, s 5-6K, c 9-14)", 16384, 6000, 12000, 5000, 6000, 9, 14},
        {"frontier (empty bins, s 5-6K, c 40-60)", 16384, 16384, 16384, 5000, 6000, 40, 60},
    };
    std::mt19937 rng(1);
    for (const auto& sh : shapes) {
        if (++idx, only >= 0 && idx != only) continue;
        std::vector<u32> R(64 * 32 * M), S(64 * 32), Cc(64 * 32);
        for (auto& x : R) x = sh.rlo + rng() % (sh.rhi - sh.rlo + 1);
        for (int blk = 0; blk < 64; ++blk) {
            std::vector<u32> v(32);
            for (auto& x : v) x = sh.slo + rng() % (sh.shi - sh.slo + 1);
            std::sort(v.begin(), v.end(), std::greater<u32>());
            for (int l = 0; l < 32; ++l) {
                S[blk * 32 + l] = v[l];
                Cc[blk * 32 + l] = sh.clo + rng() % (sh.chi - sh.clo + 1);
            }
        }
        u32 *dR, *dS, *dC;
        unsigned long long* dout;
        cudaMalloc(&dR, R.size() * 4);
        cudaMalloc(&dS, S.size() * 4);
        cudaMalloc(&dC, Cc.size() * 4);
        cudaMalloc(&dout, 24);
        cudaMemcpy(dR, R.data(), R.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dS, S.data(), S.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dC, Cc.data(), Cc.size() * 4, cudaMemcpyHostToDevice);
        for (u32 wave : {33u}) {
            ChainArgs a{};
            k_serve_micro<M><<<1, 32>>>(a, dR, dS, dC, 2000, dout);
            unsigned long long h[3];
            cudaMemcpy(h, dout, 24, cudaMemcpyDeviceToHost);
            std::printf("%-45s %s: %.0f cycles per block, %.1f cycles per active run (%.1f active/block)\n", sh.name,
                        wave == 33 ? "per-run " : "wavefront", double(h[0]) / 2000, double(h[0]) / double(h[1]),
                        double(h[1]) / 2000);
        }
        cudaFree(dR);
        cudaFree(dS);
        cudaFree(dC);
        cudaFree(dout);
    }
    std::printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
