// radix.cu — stable LSD radix sort of (u32 key, u32 value) pairs.
//
// Used for every ordering on the path that the reference defines by a
// comparison sort with a total order: sort_decreasing (packing.cpp:55-60,
// length desc / id asc over an id-ordered input), the stable attention sort
// of balance_batching (balance.cpp:185-189) and the per-length FIFO order of
// greedy_fill (balance.cpp:52-60). Each 8-bit pass: (1) per-tile digit
// histograms staged in shared memory, written digit-major; (2) one
// decoupled look-back scan gives every (digit, tile) its global offset;
// (3) the tile is re-read and each element gets its stable rank inside the
// tile from warp match masks plus per-warp digit counters, then is written
// to offset + rank. Descending order sorts ~key.
#include "engine.cuh"
#include "radix.cuh"

namespace hbp_b200 {

namespace {

constexpr int RB = 256;      // threads per block
constexpr int RITEMS = 16;   // elements per thread per tile
constexpr int RTILE = RB * RITEMS;
constexpr int RW = RB / 32;  // warps per block

__device__ __forceinline__ u32 digit_of(u32 k, int shift, bool desc) {
    const u32 kk = desc ? ~k : k;
    return (kk >> shift) & 0xffu;
}

__global__ void __launch_bounds__(RB) k_radix_hist(const u32* __restrict__ keys, u64 n, int shift, bool desc,
                                                   u32* __restrict__ hist, u32 ntiles) {
    __shared__ u32 h[RW][256];
    for (int i = threadIdx.x; i < RW * 256; i += RB) (&h[0][0])[i] = 0;
    __syncthreads();
    const u64 base = static_cast<u64>(blockIdx.x) * RTILE;
    const unsigned w = warp_id();
#pragma unroll 4
    for (int k = 0; k < RITEMS; ++k) {
        const u64 i = base + static_cast<u64>(k) * RB + threadIdx.x;
        if (i < n) atomicAdd(&h[w][digit_of(keys[i], shift, desc)], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += RB) {
        u32 s = 0;
#pragma unroll
        for (int q = 0; q < RW; ++q) s += h[q][d];
        hist[static_cast<u64>(d) * ntiles + blockIdx.x] = s;
    }
}

__global__ void __launch_bounds__(RB) k_radix_scatter(const u32* __restrict__ keys_in,
                                                      const u32* __restrict__ vals_in, u32* __restrict__ keys_out,
                                                      u32* __restrict__ vals_out, u64 n, int shift, bool desc,
                                                      const u32* __restrict__ offs, u32 ntiles) {
    __shared__ u32 s_base[256];      // running count per digit within this tile
    __shared__ u32 s_wc[RW][256];    // per-warp digit counts of the current sub-round
    const unsigned lane = lane_id(), w = warp_id();
    for (int d = threadIdx.x; d < 256; d += RB) s_base[d] = offs[static_cast<u64>(d) * ntiles + blockIdx.x];
    const u64 base = static_cast<u64>(blockIdx.x) * RTILE;
    const unsigned lt = (1u << lane) - 1u;
    for (int k = 0; k < RITEMS; ++k) {
        for (int i = threadIdx.x; i < RW * 256; i += RB) (&s_wc[0][0])[i] = 0;
        __syncthreads();
        const u64 i = base + static_cast<u64>(k) * RB + threadIdx.x;
        const bool valid = i < n;
        u32 key = 0, val = 0, d = 0xffffffffu;
        if (valid) {
            key = keys_in[i];
            val = vals_in[i];
            d = digit_of(key, shift, desc);
        }
        const unsigned active = __ballot_sync(0xffffffffu, valid);
        unsigned peers = __match_any_sync(0xffffffffu, d);
        peers &= active;
        const u32 rank_in_warp = __popc(peers & lt);
        if (valid && rank_in_warp == 0) s_wc[w][d] = __popc(peers);
        __syncthreads();
        // exclusive prefix over warps for each digit, then advance s_base
        for (int dd = threadIdx.x; dd < 256; dd += RB) {
            u32 run = s_base[dd];
#pragma unroll
            for (int q = 0; q < RW; ++q) {
                const u32 c = s_wc[q][dd];
                s_wc[q][dd] = run;
                run += c;
            }
            s_base[dd] = run;
        }
        __syncthreads();
        if (valid) {
            const u32 pos = s_wc[w][d] + rank_in_warp;
            keys_out[pos] = key;
            vals_out[pos] = val;
        }
        __syncthreads();
    }
}

}  // namespace

void radix_sort_pairs(Ctx& c, u32* keys, u32* vals, i64 n_signed, int bits, bool descending, u32* tmp_keys,
                      u32* tmp_vals) {
    if (n_signed <= 1) return;
    const u64 n = static_cast<u64>(n_signed);
    cudaStream_t s = c.stream;
    const u32 ntiles = static_cast<u32>((n + RTILE - 1) / RTILE);
    DevBuf<u32> hist(static_cast<size_t>(ntiles) * 256, s);
    DevBuf<u32> offs(static_cast<size_t>(ntiles) * 256, s);
    DevBuf<u32> tk, tv;
    if (!tmp_keys) {
        tk.alloc(n, s);
        tmp_keys = tk.p;
    }
    if (!tmp_vals) {
        tv.alloc(n, s);
        tmp_vals = tv.p;
    }
    const int passes = (bits + 7) / 8;
    u32 *ki = keys, *vi = vals, *ko = tmp_keys, *vo = tmp_vals;
    for (int p = 0; p < passes; ++p) {
        const int shift = 8 * p;
        LAUNCH_B("radix.hist", 4.0 * n, k_radix_hist, ntiles, RB, 0, s, ki, n, shift, descending, hist.p, ntiles);
        const u32* hp = hist.p;
        u32* op = offs.p;
        scan_exclusive<u32>(
            static_cast<i64>(ntiles) * 256, [=] __device__(i64 i) { return hp[i]; },
            [=] __device__(i64 i, u32 v) { op[i] = v; }, s, c.scan);
        LAUNCH_B("radix.scatter", 16.0 * n, k_radix_scatter, ntiles, RB, 0, s, ki, vi, ko, vo, n, shift, descending,
                 offs.p, ntiles);
        std::swap(ki, ko);
        std::swap(vi, vo);
    }
    if (ki != keys) {
        CUDA_CHECK(cudaMemcpyAsync(keys, ki, sizeof(u32) * n, cudaMemcpyDeviceToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(vals, vi, sizeof(u32) * n, cudaMemcpyDeviceToDevice, s));
    }
}

}  // namespace hbp_b200
