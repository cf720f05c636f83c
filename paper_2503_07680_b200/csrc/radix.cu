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

#ifndef HBP_RADIX_ITEMS
#define HBP_RADIX_ITEMS 8
#endif
#ifndef HBP_RADIX_MINB
#define HBP_RADIX_MINB 4
#endif
constexpr int RB = 256;                   // threads per block
constexpr int RITEMS = HBP_RADIX_ITEMS;   // elements per thread per tile
constexpr int RTILE = RB * RITEMS;
constexpr int RW = RB / 32;  // warps per block

__device__ __forceinline__ u32 digit_of(u32 k, int shift, bool desc) {
    const u32 kk = desc ? ~k : k;
    return (kk >> shift) & 0xffu;
}

// Lanes of the warp holding the same 8-bit digit (among `valid` lanes):
// eight ballots, cheaper than match.any on B200.
__device__ __forceinline__ unsigned digit_peers(u32 d, bool valid) {
    unsigned peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const bool bit = (d >> b) & 1u;
        const unsigned m = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? m : ~m;
    }
    return peers;
}

__global__ void __launch_bounds__(RB) k_radix_hist(const u32* __restrict__ keys, u64 n, int shift, bool desc,
                                                   u32* __restrict__ hist, u32 ntiles) {
    __shared__ u32 h[RW][256];
    for (int i = threadIdx.x; i < RW * 256; i += RB) (&h[0][0])[i] = 0;
    __syncthreads();
    const u64 base = static_cast<u64>(blockIdx.x) * RTILE;
    const unsigned w = warp_id(), lane = lane_id();
#pragma unroll 4
    for (int k = 0; k < RITEMS; ++k) {
        const u64 i = base + static_cast<u64>(k) * RB + threadIdx.x;
        const bool valid = i < n;
        const u32 d = valid ? digit_of(keys[i], shift, desc) : 0u;
        const unsigned peers = digit_peers(d, valid);
        if (valid && (peers & ((1u << lane) - 1u)) == 0) h[w][d] += __popc(peers);  // one leader per digit
        __syncwarp();  // the next item's leader of the same digit may be another lane
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += RB) {
        u32 s = 0;
#pragma unroll
        for (int q = 0; q < RW; ++q) s += h[q][d];
        hist[static_cast<u64>(d) * ntiles + blockIdx.x] = s;
    }
}

// Scatter of one pass. Ranks the tile in shared memory (warp match masks
// give each element its rank among equal digits of its warp; per-warp digit
// counts, a prefix over warps and one block scan over digits give the
// tile-local digit starts), places keys and values there in digit order, then
// writes them out striped: consecutive threads write consecutive positions of
// a digit's run, so global writes are coalesced. Three block barriers per
// tile. Warp w owns the contiguous chunk [w * 512, (w + 1) * 512) of the tile,
// which keeps the ranking stable.
__global__ void __launch_bounds__(RB, HBP_RADIX_MINB) k_radix_scatter(const u32* __restrict__ keys_in,
                                                      const u32* __restrict__ vals_in, u32* __restrict__ keys_out,
                                                      u32* __restrict__ vals_out, u64 n, int shift, bool desc,
                                                      const u32* __restrict__ offs, u32 ntiles) {
    __shared__ u32 s_k[RTILE];
    __shared__ u32 s_v[RTILE];
    __shared__ unsigned short s_wc[RW][256];  // per-warp digit counts, then offsets within the digit
    __shared__ u32 s_dstart[256];
    __shared__ u32 s_goff[256];
    __shared__ u32 s_red[33];
    const unsigned lane = lane_id(), w = warp_id();
    const u64 base = static_cast<u64>(blockIdx.x) * RTILE;
    const u32 len = static_cast<u32>(base + RTILE < n ? RTILE : n - base);
    for (int d = lane; d < 256; d += 32) s_wc[w][d] = 0;
    __syncwarp();
    constexpr int PER_WARP = RTILE / RW;  // 512
    u32 key[RITEMS], val[RITEMS], dg[RITEMS], rk[RITEMS];
#pragma unroll
    for (int k = 0; k < RITEMS; ++k) {
        const u32 li = w * PER_WARP + k * 32 + lane;
        const bool valid = li < len;
        key[k] = valid ? keys_in[base + li] : 0u;
        val[k] = valid ? vals_in[base + li] : 0u;
        dg[k] = valid ? digit_of(key[k], shift, desc) : 256u;
    }
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int k = 0; k < RITEMS; ++k) {
        const u32 d = dg[k];
        const unsigned peers = digit_peers(d, d < 256u);
        const u32 old = d < 256u ? s_wc[w][d] : 0u;
        rk[k] = old + __popc(peers & lt);
        __syncwarp();
        if (d < 256u && (peers & lt) == 0) s_wc[w][d] = static_cast<unsigned short>(old + __popc(peers));
        __syncwarp();
    }
    __syncthreads();
    {
        const u32 d = threadIdx.x;  // RB == 256 digits
        u32 run = 0;
#pragma unroll
        for (int q = 0; q < RW; ++q) {
            const u32 c = s_wc[q][d];
            s_wc[q][d] = static_cast<unsigned short>(run);
            run += c;
        }
        u32 tot;
        const u32 ex = block_exclusive_scan<u32>(run, s_red, tot);
        s_dstart[d] = ex;
        s_goff[d] = offs[static_cast<u64>(d) * ntiles + blockIdx.x];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < RITEMS; ++k) {
        const u32 d = dg[k];
        if (d < 256u) {
            const u32 p = s_dstart[d] + s_wc[w][d] + rk[k];
            s_k[p] = key[k];
            s_v[p] = val[k];
        }
    }
    __syncthreads();
    for (u32 p = threadIdx.x; p < len; p += RB) {
        const u32 kk = s_k[p];
        const u32 d = digit_of(kk, shift, desc);
        const u32 g = s_goff[d] + (p - s_dstart[d]);
        keys_out[g] = kk;
        vals_out[g] = s_v[p];
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
            [=] __device__(i64 i, u32 v) { op[i] = v; }, s, c.scan, "scan.radix1");
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
