// Experiment: row-major bins for the first-fit chain's serve (lane l, row i
// holds bin 32 i + l) against the lane-major serve (lane l holds bins
// M l .. M l + M - 1), on the real cells of tools/micro/cells/. Non-frontier
// serve only (FFD's empty bins served as ordinary bins in both).
#include "../../paper_2503_07680_b200/csrc/chain.cu"

#include <cstdio>
#include <vector>

namespace hbp_b200 {
thread_local int64_t* g_launch_counter = nullptr;
thread_local KernelProfiler* g_prof = nullptr;
thread_local BlockCache* g_cache = nullptr;

constexpr int M = 8;

// runs in `act` (lane = run, in order) against row-major bins R[i] (bin 32 i + lane)
__device__ __forceinline__ void serve_rows(unsigned act, u32 s, u32& c, u32 (&R)[M], u32 (&N)[M], u32 lane) {
    const u32 s_eff = (s & 0x7fffffffu) + (s >> 31);
    const u32 inv_own = (s & 0x7fffffffu) ? 0xffffffffu / (s & 0x7fffffffu) : 0u;
    u32 lmax = 0;
#pragma unroll
    for (int i = 0; i < M; ++i) lmax = max(lmax, R[i]);
    while (act) {
        const int r = __ffs(act) - 1;
        act &= act - 1;
        const u32 Sraw = __shfl_sync(0xffffffffu, s, r);
        const u32 S = Sraw & 0x7fffffffu, strict = Sraw >> 31;
        const u32 inv = __shfl_sync(0xffffffffu, inv_own, r);
        u32 left = __shfl_sync(0xffffffffu, c, r);
        bool took = false;
#pragma unroll
        for (int i = 0; i < M; ++i) {
            if (left == 0) break;
            unsigned room = __ballot_sync(0xffffffffu, R[i] >= S + strict);
            if (!room) continue;
            took = true;
            const u32 Re = R[i] > strict ? R[i] - strict : 0u;
            u32 q = __umulhi(Re, inv);
            q += (Re - q * S >= S) ? 1u : 0u;
            // lanes of this row in order: walk the first lanes, scan if many
            int walked = 0;
            while (room && left && walked < 3) {
                const int f = __ffs(room) - 1;
                room &= room - 1;
                const u32 qf = __shfl_sync(0xffffffffu, q, f);
                const u32 t = min(qf, left);
                if (static_cast<int>(lane) == f) {
                    R[i] -= t * S;
                    N[i] += t;
                }
                left -= t;
                ++walked;
            }
            if (room && left) {
                const u32 v = (room >> lane) & 1u ? min(q, left) : 0u;
                u32 incl = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= static_cast<u32>(o)) incl = min(incl + t, left);
                }
                const u32 excl = incl - v;  // saturated prefix before this lane
                const u32 t = excl < left ? min(v, left - excl) : 0u;
                R[i] -= t * S;
                N[i] += t;
                left -= __shfl_sync(0xffffffffu, incl, 31);
            }
        }
        if (static_cast<int>(lane) == r) c = left;
        if (took && act) {
            lmax = 0;
#pragma unroll
            for (int i = 0; i < M; ++i) lmax = max(lmax, R[i]);
            act &= __ballot_sync(0xffffffffu, s_eff <= __reduce_max_sync(0xffffffffu, lmax));
        }
    }
}

__global__ void k_rows(ChainArgs a, const u32* cells, int n_cells, int reps, int rows, unsigned long long* cyc,
                       u32* out) {
    const u32 lane = threadIdx.x & 31u;
    __shared__ RunStage st;
    for (int k = 0; k < n_cells; ++k) {
        const u32* rec = cells + static_cast<size_t>(k) * 320;
        unsigned long long best = ~0ull;
        for (int rep = 0; rep < reps; ++rep) {
            u32 R[M], N[M];
            u32 lmax = 0;
#pragma unroll
            for (int i = 0; i < M; ++i) {
                R[i] = rows ? rec[i * 32 + lane] : rec[lane * M + i];
                N[i] = 0;
                lmax = max(lmax, R[i]);
            }
            u32 emask = 0;
            u32 wmax = __reduce_max_sync(0xffffffffu, lmax);
            const u32 s = rec[256 + lane];
            u32 c = rec[288 + lane];
            const unsigned act = __ballot_sync(0xffffffffu, c > 0 && (s & 0x7fffffffu) + (s >> 31) <= wmax);
            __syncwarp();
            const long long t0 = clock64();
            if (act) {
                if (rows) serve_rows(act, s, c, R, N, lane);
                else serve<M, false>(a, act, s, 1000000u, c, R, N, wmax, emask, st, 0, lane);
            }
            __syncwarp();
            const long long t1 = clock64();
            best = min(best, static_cast<unsigned long long>(t1 - t0));
            // canonical output: c per run, residuals in bin order
            out[k * 288 + lane] = c;
#pragma unroll
            for (int i = 0; i < M; ++i) out[k * 288 + 32 + (rows ? i * 32 + lane : lane * M + i)] = R[i];
        }
        if (lane == 0) cyc[k] = best;
    }
}

}  // namespace hbp_b200

using namespace hbp_b200;

int main() {
    const char* files[] = {"tools/micro/cells/cells0.bin", "tools/micro/cells/cells1.bin",
                           "tools/micro/cells/cells2.bin"};
    const u32 caps[] = {131072, 131072, 16384};
    for (int f = 0; f < 3; ++f) {
        FILE* fp = std::fopen(files[f], "rb");
        if (!fp) continue;
        std::vector<u32> cells;
        u32 buf[320];
        while (std::fread(buf, 4, 320, fp) == 320) cells.insert(cells.end(), buf, buf + 320);
        std::fclose(fp);
        const int n = static_cast<int>(cells.size() / 320);
        u32 *d_cells, *d_out;
        unsigned long long* d_cyc;
        cudaMalloc(&d_cells, cells.size() * 4);
        cudaMalloc(&d_cyc, n * 8);
        cudaMalloc(&d_out, n * 288 * 4);
        cudaMemcpy(d_cells, cells.data(), cells.size() * 4, cudaMemcpyHostToDevice);
        std::vector<u32> ref;
        for (int rows = 0; rows < 2; ++rows) {
            ChainArgs a{};
            a.cap = caps[f];
            a.ffd = 0;
            k_rows<<<1, 32>>>(a, d_cells, n, 3, rows, d_cyc, d_out);
            std::vector<unsigned long long> cyc(n);
            std::vector<u32> out(n * 288);
            cudaMemcpy(cyc.data(), d_cyc, n * 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(out.data(), d_out, n * 288 * 4, cudaMemcpyDeviceToHost);
            double tot = 0;
            for (int k = 0; k < n; ++k) tot += cyc[k];
            // the two layouts place items in different bins (bin order differs), so compare the
            // per-run leftovers and the multiset of residuals only when they must agree: leftovers
            const bool same_c = ref.empty() || [&] {
                for (int k = 0; k < n; ++k)
                    for (int l = 0; l < 32; ++l)
                        if (ref[k * 288 + l] != out[k * 288 + l]) return false;
                return true;
            }();
            if (ref.empty()) ref = out;
            std::printf("cells%d (%d cells) %-10s %8.0f cycles/cell %s\n", f, n, rows ? "row-major" : "lane-major",
                        tot / n, same_c ? "" : "(leftovers differ: bin order differs)");
        }
    }
    std::printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
