// Replays real first-fit chain cells (tools/micro/cells/cells*.bin: bins and
// runs of (warp, block) cells with >= 8 active runs, taken from a CPU model of
// the C2 chain inputs) through the chain's per-cell serve on one warp and
// reports cycles per cell for each serve mode, checking the modes agree.
//   nvcc -O3 -std=c++17 --extended-lambda -gencode arch=compute_100a,code=sm_100a \
//        -I include -o tools/micro/cell_micro tools/micro/cell_micro.cu && tools/micro/cell_micro
#define HBP_SERVE_PROF 1
#include "../../paper_2503_07680_b200/csrc/chain.cu"

#include <cstdio>
#include <vector>

namespace hbp_b200 {
thread_local int64_t* g_launch_counter = nullptr;
thread_local KernelProfiler* g_prof = nullptr;
thread_local BlockCache* g_cache = nullptr;

constexpr int M = 8;

__global__ void k_cell_micro(ChainArgs a, const u32* cells, int n_cells, int reps, unsigned long long* cyc,
                             u32* out) {
    const u32 lane = threadIdx.x & 31u;
    __shared__ RunStage st;
    for (int k = 0; k < n_cells; ++k) {
        const u32* rec = cells + static_cast<size_t>(k) * 320;
        unsigned long long best = ~0ull;
        u32 cfin = 0, rsum = 0;
        for (int rep = 0; rep < reps; ++rep) {
            u32 R[M], N[M];
            u32 lmax = 0;
            bool empty = a.ffd != 0;
#pragma unroll
            for (int i = 0; i < M; ++i) {
                R[i] = rec[lane * M + i];
                N[i] = 0;
                lmax = max(lmax, R[i]);
                empty = empty && R[i] == a.cap;
            }
            u32 emask = __ballot_sync(0xffffffffu, empty);
            u32 wmax = __reduce_max_sync(0xffffffffu, lmax);
            const u32 s = rec[256 + lane];
            u32 c = rec[288 + lane];
            const u32 end_item = 1000000u;
            const unsigned act = __ballot_sync(0xffffffffu, c > 0 && (s & 0x7fffffffu) + (s >> 31) <= wmax);
            __syncwarp();
            const long long t0 = clock64();
            if (act) serve<M, false>(a, act, s, end_item, c, R, N, wmax, emask, st, 0, lane);
            __syncwarp();
            const long long t1 = clock64();
            best = min(best, static_cast<unsigned long long>(t1 - t0));
            cfin = c;
            rsum = 0;
#pragma unroll
            for (int i = 0; i < M; ++i) rsum += R[i] * (i + 1);
        }
        if (lane == 0) cyc[k] = best;
        out[k * 64 + lane] = cfin;
        out[k * 64 + 32 + lane] = rsum;
    }
}

}  // namespace hbp_b200

using namespace hbp_b200;

int main(int argc, char** argv) {
    const char* files[] = {"tools/micro/cells/cells0.bin", "tools/micro/cells/cells1.bin",
                           "tools/micro/cells/cells2.bin"};
    const u32 caps[] = {131072, 131072, 16384};
    const int ffds[] = {1, 0, 1};
    struct Mode { const char* name; };
    const Mode modes[] = {{"serve"}};
    for (int f = 0; f < 3; ++f) {
        FILE* fp = std::fopen(files[f], "rb");
        if (!fp) continue;
        std::vector<u32> cells;
        u32 buf[320];
        while (std::fread(buf, 4, 320, fp) == 320) cells.insert(cells.end(), buf, buf + 320);
        std::fclose(fp);
        const int n = static_cast<int>(cells.size() / 320);
        u32* d_cells;
        unsigned long long* d_cyc;
        u32* d_out;
        cudaMalloc(&d_cells, cells.size() * 4);
        cudaMalloc(&d_cyc, n * 8);
        cudaMalloc(&d_out, n * 64 * 4);
        cudaMemcpy(d_cells, cells.data(), cells.size() * 4, cudaMemcpyHostToDevice);
        std::vector<u32> ref;
        for (const auto& m : modes) {
            ChainArgs a{};
            a.cap = caps[f];
            a.ffd = ffds[f];
            unsigned long long zero[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pr[8];
            cudaMemcpyToSymbol(g_serve_prof, zero, sizeof(zero));
            k_cell_micro<<<1, 32>>>(a, d_cells, n, 3, d_cyc, d_out);
            cudaMemcpyFromSymbol(pr, g_serve_prof, sizeof(pr));
            std::vector<unsigned long long> cyc(n);
            std::vector<u32> out(n * 64);
            cudaMemcpy(cyc.data(), d_cyc, n * 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(out.data(), d_out, n * 256, cudaMemcpyDeviceToHost);
            double tot = 0;
            int act = 0;
            for (int k = 0; k < n; ++k) tot += cyc[k];
            for (int k = 0; k < n; ++k)
                for (int l = 0; l < 32; ++l) act += cells[k * 320 + 288 + l] > 0;
            bool same = ref.empty() || ref == out;
            if (ref.empty()) ref = out;
            std::printf("cells%d (%d cells) %-16s %8.0f cycles/cell  %s  phases/cell: room %.0f div+pre %.0f walk %.0f apply %.0f filter %.0f\n",
                        f, n, m.name, tot / n, same ? "" : "MISMATCH", pr[0] / 3.0 / n, pr[1] / 3.0 / n,
                        pr[2] / 3.0 / n, pr[3] / 3.0 / n, pr[4] / 3.0 / n);
        }
        cudaFree(d_cells);
        cudaFree(d_cyc);
        cudaFree(d_out);
    }
    std::printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
