// radix.cu — stable LSD radix sort of (u32 key, u32 value) pairs.
//
// Used for every ordering on the path that the reference defines by a
// comparison sort with a total order: sort_decreasing (packing.cpp:55-60,
// length desc / id asc over an id-ordered input), the stable attention sort
// of balance_batching (balance.cpp:185-189) and the per-length FIFO order of
// greedy_fill (balance.cpp:52-60). Onesweep: one read of the keys builds
// the digit histograms of every 8-bit pass; each pass is then one kernel
// (tiles staged by bulk asynchronous copies, stable warp-match ranks, look-back
// across tiles, coalesced digit-ordered writes). Descending order sorts ~key.
#include "engine.cuh"
#include "radix.cuh"

#include <mutex>
#include <set>

namespace hbp_b200 {

namespace {

// ---------------------------------------------------------------------------
// Onesweep (one histogram pass for every digit, then one kernel per digit
// pass with decoupled look-back across tiles; no per-pass histogram or scan
// launches). Tiles of 4096 pairs are staged in shared memory by one bulk
// asynchronous copy (cp.async.bulk, completion on an mbarrier), ranked
// stably with warp match masks in warp-striped order, counted per digit,
// offset across tiles by look-back on (flag << 62 | count) status words, and
// written out in digit order so global stores are coalesced.
// ---------------------------------------------------------------------------
constexpr int OB = 256;
constexpr int OITEMS = 16;
constexpr int OTILE = OB * OITEMS;  // 4096 pairs
constexpr int OW = OB / 32;
constexpr int OMAXP = 4;            // digit passes (32-bit keys)
constexpr unsigned long long kAgg = 1ull << 62, kIncl = 2ull << 62, kValMask = (1ull << 62) - 1;

__device__ __forceinline__ u32 smem_u32(const void* p) {
    return static_cast<u32>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, u32 phase) {
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64g(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64g(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Digit histograms of every pass in one read of the keys (16-byte loads):
// counters per (digit, lane) -- lane l of every warp updates column l, so a
// warp's 32 updates never share an address or a bank whatever the digits
// (lengths crowd a few high digits). The last block to finish turns the
// histograms into each pass's bucket starts.
__global__ void __launch_bounds__(OB) k_os_hist(const u32* __restrict__ keys, u64 n, int passes, bool desc,
                                               u32* __restrict__ ghist, u32* __restrict__ gstart,
                                               u32* __restrict__ ticket) {
    extern __shared__ u32 h[];  // [passes][256][32]
    __shared__ bool s_last;
    for (int i = threadIdx.x; i < passes * 256 * 32; i += OB) h[i] = 0;
    __syncthreads();
    const unsigned lane = lane_id();
    const u64 nv = n / 4;
    const uint4* k4 = reinterpret_cast<const uint4*>(keys);
    auto add = [&](u32 k) {
        const u32 kk = desc ? ~k : k;
        for (int p = 0; p < passes; ++p) atomicAdd(&h[(p * 256 + ((kk >> (8 * p)) & 0xffu)) * 32 + lane], 1u);
    };
    // four 16-byte loads in flight per thread before their counts (one load
    // per thread at a time left the read latency-bound at ~1 TB/s)
    const u64 stride = static_cast<u64>(gridDim.x) * OB;
    u64 v = static_cast<u64>(blockIdx.x) * OB + threadIdx.x;
    for (; v + 3 * stride < nv; v += 4 * stride) {
        uint4 q[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) q[r] = k4[v + r * stride];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            add(q[r].x);
            add(q[r].y);
            add(q[r].z);
            add(q[r].w);
        }
    }
    for (; v < nv; v += stride) {
        const uint4 q = k4[v];
        add(q.x);
        add(q.y);
        add(q.z);
        add(q.w);
    }
    if (blockIdx.x == 0 && threadIdx.x < n - nv * 4) add(keys[nv * 4 + threadIdx.x]);  // the n % 4 tail
    __syncthreads();
    for (int i = threadIdx.x; i < passes * 256; i += OB) {
        u32 c = 0;
#pragma unroll 8
        for (int l = 0; l < 32; ++l) c += h[i * 32 + ((l + i) & 31)];  // rotated: no bank conflict
        if (c) atomicAdd(&ghist[i], c);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    __shared__ u32 s_red[33];
    for (int p = 0; p < passes; ++p) {
        const u32 c = *reinterpret_cast<volatile u32*>(&ghist[p * 256 + threadIdx.x]);
        u32 tot;
        gstart[p * 256 + threadIdx.x] = block_exclusive_scan<u32>(c, s_red, tot);
    }
}

// Look-back of digit d for `tile`: the exclusive count of d over the tiles
// before it -- aggregates summed back to the first inclusive count, polling
// a word not yet published. (A window of eight words per round trip spilled
// registers and measured slower.)
__device__ __forceinline__ unsigned long long look_back(const unsigned long long* __restrict__ status, u32 tile,
                                                        u32 d) {
    unsigned long long excl = 0;
    long long p = static_cast<long long>(tile) - 1;
    for (;;) {
        const unsigned long long wv = ld_relaxed_u64g(status + static_cast<u64>(p) * 256 + d);
        const unsigned long long f = wv & ~kValMask;
        if (f == 0) continue;
        excl += wv & kValMask;
        if (f == kIncl) return excl;
        --p;
    }
}

// One digit pass over a tile (dynamic tile order, so every earlier tile is
// running or done when a tile looks back).
template <bool BALLOT>
__global__ void __launch_bounds__(OB, 3) k_os_pass(const u32* __restrict__ keys_in, const u32* __restrict__ vals_in,
                                                  u32* __restrict__ keys_out, u32* __restrict__ vals_out, u64 n,
                                                  int shift, bool desc, const u32* __restrict__ gstart,
                                                  unsigned long long* __restrict__ status, u32* __restrict__ tiles,
                                                  bool bulk, int dbits) {
    extern __shared__ __align__(128) u32 os_smem[];
    u32* s_k = os_smem;  // tile as loaded
    u32* s_v = s_k + OTILE;
    auto* s_kv = reinterpret_cast<unsigned long long*>(s_v + OTILE);  // tile in digit order: key | val << 32
    __shared__ unsigned short s_wc[OW][256];
    __shared__ u32 s_lstart[256];
    __shared__ int s_gbase[256];
    __shared__ u32 s_red[33];
    __shared__ u32 s_tile;
    __shared__ alignas(8) unsigned long long s_bar;
    const unsigned tid = threadIdx.x, lane = lane_id(), w = warp_id();
    if (tid == 0) {
        s_tile = atomicAdd(tiles, 1u);
        mbar_init(&s_bar, 1);
    }
    for (int i = tid; i < OW * 256 / 2; i += OB) reinterpret_cast<u32*>(&s_wc[0][0])[i] = 0;
    __syncthreads();
    const u32 tile = s_tile;
    const u64 base = static_cast<u64>(tile) * OTILE;
    const u32 len = static_cast<u32>(base + OTILE <= n ? OTILE : n - base);
    if (bulk && len == OTILE) {
        if (tid == 0) {
            mbar_expect_tx(&s_bar, 2u * OTILE * 4u);
            bulk_g2s(s_k, keys_in + base, OTILE * 4u, &s_bar);
            bulk_g2s(s_v, vals_in + base, OTILE * 4u, &s_bar);
        }
        mbar_wait(&s_bar, 0);
    } else {
        for (u32 i = tid; i < len; i += OB) {
            s_k[i] = keys_in[base + i];
            s_v[i] = vals_in[base + i];
        }
        __syncthreads();
    }
    // stable ranks: warp w owns elements [w * 512, (w + 1) * 512), row by
    // row; rank (9 bits) and digit (9 bits, 256 = none) packed per element
    u32 rd[OITEMS], key[OITEMS];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < OITEMS; ++i) {
        const u32 e = w * (OITEMS * 32) + i * 32 + lane;
        const bool valid = e < len;
        key[i] = valid ? s_k[e] : 0u;
        const u32 d = valid ? ((desc ? ~key[i] : key[i]) >> shift) & 0xffu : 256u;
        unsigned peers;
        if (BALLOT) {  // one ballot per live digit bit instead of one match (lanes with d == 256 never match a
                       // valid digit; the bits above the key's width are zero in every digit of this pass)
            peers = __ballot_sync(0xffffffffu, valid);
            if (!valid) peers = ~peers;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                if (b >= dbits) break;
                const bool bit = (d >> b) & 1u;
                const unsigned m = __ballot_sync(0xffffffffu, bit);
                peers &= bit ? m : ~m;
            }
        } else {
            peers = __match_any_sync(0xffffffffu, d);
        }
        const u32 old = valid ? s_wc[w][d] : 0u;
        rd[i] = ((old + __popc(peers & lt)) << 16) | d;
        __syncwarp();
        if (valid && (peers & lt) == 0) s_wc[w][d] = static_cast<unsigned short>(old + __popc(peers));
        __syncwarp();
    }
    __syncthreads();
    // digit d = tid: offsets of the warps inside the tile, the tile's count
    const u32 d = tid;
    u32 run = 0;
#pragma unroll
    for (int q = 0; q < OW; ++q) {
        const u32 c = s_wc[q][d];
        s_wc[q][d] = static_cast<unsigned short>(run);
        run += c;
    }
    // publish this tile's count, then look back for the counts before it
    unsigned long long* st = status + static_cast<u64>(tile) * 256 + d;
    st_relaxed_u64g(st, (tile == 0 ? kIncl : kAgg) | run);
    u32 tot;
    const u32 lstart = block_exclusive_scan<u32>(run, s_red, tot);
    const unsigned long long excl = tile > 0 ? look_back(status, tile, d) : 0ull;
    if (tile > 0) st_relaxed_u64g(st, kIncl | (excl + run));
    s_lstart[d] = lstart;
    // global position = s_gbase[digit] + position in the digit-ordered tile (n < 2^31)
    s_gbase[d] = static_cast<int>(gstart[d] + excl) - static_cast<int>(lstart);
    __syncthreads();
    // stage in digit order, then write out coalesced
#pragma unroll
    for (int i = 0; i < OITEMS; ++i) {
        const u32 dd = rd[i] & 0xffffu;
        if (dd < 256u) {
            const u32 e = w * (OITEMS * 32) + i * 32 + lane;
            const u32 p = s_lstart[dd] + s_wc[w][dd] + (rd[i] >> 16);
            s_kv[p] = static_cast<unsigned long long>(key[i]) | (static_cast<unsigned long long>(s_v[e]) << 32);
        }
    }
    __syncthreads();
    for (u32 p = tid; p < len; p += OB) {
        const unsigned long long kv = s_kv[p];
        const u32 kk = static_cast<u32>(kv);
        const u32 dd = ((desc ? ~kk : kk) >> shift) & 0xffu;
        const u64 g = static_cast<u64>(static_cast<long long>(s_gbase[dd]) + p);
        keys_out[g] = kk;
        vals_out[g] = static_cast<u32>(kv >> 32);
    }
}

// The same pass with the tile permuted in place (32 KB of shared memory per
// CTA instead of 64 KB, no key registers kept across the look-back): ranks
// become tile positions, the keys are permuted through registers into s_k and
// written out, then the values into s_v (their digits read from the permuted
// keys). 48 registers and 38 KB per CTA: five CTAs per SM instead of three,
// so the bulk loads and look-backs of more tiles overlap the ranking.
template <int PROBE>  // 0: the pass; timing probes (wrong output): 1 no look-back, 2 no global stores
__global__ void __launch_bounds__(OB, 4) k_os_pass_ip(const u32* __restrict__ keys_in, const u32* __restrict__ vals_in,
                                                     u32* __restrict__ keys_out, u32* __restrict__ vals_out, u64 n,
                                                     int shift, bool desc, const u32* __restrict__ gstart,
                                                     unsigned long long* __restrict__ status, u32* __restrict__ tiles,
                                                     bool bulk, int dbits) {
    extern __shared__ __align__(128) u32 os_smem[];
    u32* s_k = os_smem;  // tile as loaded
    u32* s_v = s_k + OTILE;
    u32* s_x = s_v + OTILE;  // keys in digit order
    __shared__ unsigned short s_wc[OW][256];
    __shared__ int s_gbase[256];
    __shared__ u32 s_red[33];
    __shared__ u32 s_tile;
    __shared__ alignas(8) unsigned long long s_bar;
    const unsigned tid = threadIdx.x, lane = lane_id(), w = warp_id();
    if (tid == 0) {
        s_tile = atomicAdd(tiles, 1u);
        mbar_init(&s_bar, 1);
    }
    for (int i = tid; i < OW * 256 / 2; i += OB) reinterpret_cast<u32*>(&s_wc[0][0])[i] = 0;
    __syncthreads();
    const u32 tile = s_tile;
    const u64 base = static_cast<u64>(tile) * OTILE;
    const u32 len = static_cast<u32>(base + OTILE <= n ? OTILE : n - base);
    if (bulk && len == OTILE) {
        if (tid == 0) {
            mbar_expect_tx(&s_bar, 2u * OTILE * 4u);
            bulk_g2s(s_k, keys_in + base, OTILE * 4u, &s_bar);
            bulk_g2s(s_v, vals_in + base, OTILE * 4u, &s_bar);
        }
        mbar_wait(&s_bar, 0);
    } else {
        for (u32 i = tid; i < len; i += OB) {
            s_k[i] = keys_in[base + i];
            s_v[i] = vals_in[base + i];
        }
        __syncthreads();
    }
    // stable ranks as in k_os_pass (ballots on the digit's live bits)
    // stable ranks (ballots on the digit's live bits), two per word; the
    // digits are read again from the tile when the ranks become positions
    u32 pp[OITEMS / 2];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < OITEMS; ++i) {
        const u32 e = w * (OITEMS * 32) + i * 32 + lane;
        const bool valid = e < len;
        const u32 kk = valid ? s_k[e] : 0u;
        const u32 d = valid ? ((desc ? ~kk : kk) >> shift) & 0xffu : 256u;
        unsigned peers = __ballot_sync(0xffffffffu, valid);
        if (!valid) peers = ~peers;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            if (b >= dbits) break;
            const bool bit = (d >> b) & 1u;
            const unsigned m = __ballot_sync(0xffffffffu, bit);
            peers &= bit ? m : ~m;
        }
        const u32 old = valid ? s_wc[w][d] : 0u;
        const u32 r = old + __popc(peers & lt);
        if (i & 1)
            pp[i / 2] |= r << 16;
        else
            pp[i / 2] = r;
        __syncwarp();
        if (valid && (peers & lt) == 0) s_wc[w][d] = static_cast<unsigned short>(old + __popc(peers));
        __syncwarp();
    }
    __syncthreads();
    const u32 d = tid;
    u32 run = 0;
#pragma unroll
    for (int q = 0; q < OW; ++q) {
        const u32 c = s_wc[q][d];
        s_wc[q][d] = static_cast<unsigned short>(run);
        run += c;
    }
    unsigned long long* st = status + static_cast<u64>(tile) * 256 + d;
    st_relaxed_u64g(st, (tile == 0 || PROBE == 1 ? kIncl : kAgg) | run);
    u32 tot;
    const u32 lstart = block_exclusive_scan<u32>(run, s_red, tot);
    // the digit's first position in the tile, folded into the warp offsets
#pragma unroll
    for (int q = 0; q < OW; ++q) s_wc[q][d] = static_cast<unsigned short>(s_wc[q][d] + lstart);
    const unsigned long long excl = tile > 0 && PROBE != 1 ? look_back(status, tile, d) : 0ull;
    if (tile > 0 && PROBE != 1) st_relaxed_u64g(st, kIncl | (excl + run));
    s_gbase[d] = static_cast<int>(gstart[d] + excl) - static_cast<int>(lstart);
    __syncthreads();
    // keys permuted into s_x (ranks -> tile positions, 0xffff: no element)
    // and written out; values permuted into s_k (free by then) and written
    // out with the digits of the permuted keys
#pragma unroll
    for (int i = 0; i < OITEMS; ++i) {
        const u32 e = w * (OITEMS * 32) + i * 32 + lane;
        u32 pos = 0xffffu;
        if (e < len) {
            const u32 kk = s_k[e];
            pos = s_wc[w][((desc ? ~kk : kk) >> shift) & 0xffu] + ((pp[i / 2] >> (16 * (i & 1))) & 0xffffu);
            s_x[pos] = kk;
        }
        if (i & 1)
            pp[i / 2] = (pp[i / 2] & 0xffffu) | (pos << 16);
        else
            pp[i / 2] = (pp[i / 2] & 0xffff0000u) | pos;
    }
    __syncthreads();
    for (u32 p = tid; p < len; p += OB) {
        const u32 kk = s_x[p];
        if (PROBE == 2 && kk != 0x7fffffffu) continue;
        keys_out[static_cast<long long>(s_gbase[((desc ? ~kk : kk) >> shift) & 0xffu]) + p] = kk;
    }
#pragma unroll
    for (int i = 0; i < OITEMS; ++i) {
        const u32 pos = (pp[i / 2] >> (16 * (i & 1))) & 0xffffu;
        if (pos != 0xffffu) s_k[pos] = s_v[w * (OITEMS * 32) + i * 32 + lane];
    }
    __syncthreads();
    for (u32 p = tid; p < len; p += OB) {
        const u32 kk = s_x[p];
        if (PROBE == 2 && kk != 0x7fffffffu) continue;
        vals_out[static_cast<long long>(s_gbase[((desc ? ~kk : kk) >> shift) & 0xffu]) + p] = s_k[p];
    }
}


// ---------------------------------------------------------------------------
// Small sorts in one launch: up to kSmallN pairs sorted by one CTA in shared
// memory, every digit pass inside the kernel (the plans of the sweep sort
// thousands of packs or samples at a time, where the onesweep's histogram
// pass, digit passes and their launches dominate). Ranks as in k_os_pass:
// warp w owns elements [w * 256, (w + 1) * 256) row by row, ballots on the
// digit's live bits, warp counters per digit, then the digit starts.
// ---------------------------------------------------------------------------
constexpr int SB = 1024;
constexpr int kSmallN = 8192;
constexpr int SITEMS = kSmallN / SB;  // 8 rows per warp

// Stable sort of (k[0..n), v[0..n)) in shared memory by the low `bits` of the
// key (descending sorts ~key); the result ends in (k, v). tk / tv: scratch.
__device__ void small_sort_smem(u32* k, u32* v, u32* tk, u32* tv, u32 n, int bits, bool desc,
                                unsigned short (*wc)[256], u32* dstart, u32* red) {
    const unsigned tid = threadIdx.x, lane = tid & 31u, w = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int passes = bits <= 0 ? 0 : (bits + 7) / 8;
    for (int p = 0; p < passes; ++p) {
        const int shift = 8 * p;
        const int dbits = bits - shift < 8 ? bits - shift : 8;
        for (unsigned i = tid; i < 32 * 256; i += SB) (&wc[0][0])[i] = 0;
        __syncthreads();
        u32 rd[SITEMS];
#pragma unroll
        for (int i = 0; i < SITEMS; ++i) {
            const u32 e = w * (SITEMS * 32) + i * 32 + lane;
            const bool valid = e < n;
            const u32 d = valid ? (((desc ? ~k[e] : k[e]) >> shift) & 0xffu) : 256u;
            unsigned peers = __ballot_sync(0xffffffffu, valid);
            if (!valid) peers = ~peers;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                if (b >= dbits) break;
                const bool bit = (d >> b) & 1u;
                const unsigned m = __ballot_sync(0xffffffffu, bit);
                peers &= bit ? m : ~m;
            }
            const u32 old = valid ? wc[w][d] : 0u;
            rd[i] = ((old + __popc(peers & lt)) << 16) | d;
            __syncwarp();
            if (valid && (peers & lt) == 0) wc[w][d] = static_cast<unsigned short>(old + __popc(peers));
            __syncwarp();
        }
        __syncthreads();
        if (tid < 256) {  // digit tid: offsets of the warps, the digit's count
            u32 run = 0;
            for (int q = 0; q < 32; ++q) {
                const u32 c = wc[q][tid];
                wc[q][tid] = static_cast<unsigned short>(run);
                run += c;
            }
            dstart[tid] = run;
        }
        __syncthreads();
        if (w == 0) {  // exclusive scan over the 256 digit counts (8 per lane)
            u32 loc[8], sum = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                loc[q] = dstart[lane * 8 + q];
                sum += loc[q];
            }
            u32 inc = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= static_cast<unsigned>(o)) inc += t;
            }
            u32 run = inc - sum;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                dstart[lane * 8 + q] = run;
                run += loc[q];
            }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < SITEMS; ++i) {
            const u32 dd = rd[i] & 0xffffu;
            if (dd < 256u) {
                const u32 e = w * (SITEMS * 32) + i * 32 + lane;
                const u32 pos = dstart[dd] + wc[w][dd] + (rd[i] >> 16);
                tk[pos] = k[e];
                tv[pos] = v[e];
            }
        }
        __syncthreads();
        for (unsigned i = tid; i < n; i += SB) {
            k[i] = tk[i];
            v[i] = tv[i];
        }
        __syncthreads();
    }
    (void)red;
}

struct SmallSortSmem {
    u32 k[kSmallN], v[kSmallN], tk[kSmallN], tv[kSmallN];
    unsigned short wc[32][256];
    u32 dstart[256];
    u32 red[33];
};

__global__ void __launch_bounds__(SB, 1) k_small_sort_pairs(u32* __restrict__ keys, u32* __restrict__ vals, u32 n,
                                                            int bits, bool desc) {
    extern __shared__ __align__(16) unsigned char ss_raw[];
    SmallSortSmem& S = *reinterpret_cast<SmallSortSmem*>(ss_raw);
    for (unsigned i = threadIdx.x; i < n; i += SB) {
        S.k[i] = keys[i];
        S.v[i] = vals[i];
    }
    __syncthreads();
    small_sort_smem(S.k, S.v, S.tk, S.tv, n, bits, desc, S.wc, S.dstart, S.red);
    for (unsigned i = threadIdx.x; i < n; i += SB) {
        keys[i] = S.k[i];
        vals[i] = S.v[i];
    }
}

// Entries (len << 32 | idx) sorted by (length desc, key asc) in one launch:
// by key first when the input is not in key order (key = key32[idx], or idx),
// then stably by length descending; the entries are regathered.
__global__ void __launch_bounds__(SB, 1) k_small_sort_entries(u64* __restrict__ e, u32 n, const u32* __restrict__ key32,
                                                              int key_bits, int len_bits) {
    extern __shared__ __align__(16) unsigned char ss_raw[];
    SmallSortSmem& S = *reinterpret_cast<SmallSortSmem*>(ss_raw);
    for (unsigned i = threadIdx.x; i < n; i += SB) {
        const u32 idx = static_cast<u32>(e[i]);
        S.k[i] = key32 ? key32[idx] : idx;
        S.v[i] = i;
    }
    __syncthreads();
    if (key_bits > 0) small_sort_smem(S.k, S.v, S.tk, S.tv, n, key_bits, false, S.wc, S.dstart, S.red);
    for (unsigned i = threadIdx.x; i < n; i += SB) S.k[i] = static_cast<u32>(e[S.v[i]] >> 32);
    __syncthreads();
    small_sort_smem(S.k, S.v, S.tk, S.tv, n, len_bits, true, S.wc, S.dstart, S.red);
    // regather through the scratch halves (8 B per entry: tk and tv together)
    u64* out = reinterpret_cast<u64*>(S.tk);  // tk and tv are contiguous: 2 * kSmallN u32
    for (unsigned i = threadIdx.x; i < n; i += SB) out[i] = e[S.v[i]];
    __syncthreads();
    for (unsigned i = threadIdx.x; i < n; i += SB) e[i] = out[i];
}

void set_small_sort_smem_once() {
    static std::mutex mu;
    static std::set<int> done;
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    if (done.insert(dev).second) {
        CUDA_CHECK(cudaFuncSetAttribute(k_small_sort_pairs, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(sizeof(SmallSortSmem))));
        CUDA_CHECK(cudaFuncSetAttribute(k_small_sort_entries, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(sizeof(SmallSortSmem))));
    }
}

}  // namespace

void radix_sort_pairs(Ctx& c, u32* keys, u32* vals, i64 n_signed, int bits, bool descending, u32* tmp_keys,
                      u32* tmp_vals) {
    if (n_signed <= 1) return;
    const u64 n = static_cast<u64>(n_signed);
    cudaStream_t s = c.stream;
    if (n <= static_cast<u64>(kSmallN)) {  // one CTA, every pass in one launch
        set_small_sort_smem_once();
        LAUNCH_B("radix.small", 16.0 * n, k_small_sort_pairs, 1, SB, sizeof(SmallSortSmem), s, keys, vals,
                 static_cast<u32>(n), bits, descending);
        return;
    }
    DevBuf<u32> tk, tv;
    if (!tmp_keys) {
        tk.alloc(n, s);
        tmp_keys = tk.p;
    }
    if (!tmp_vals) {
        tv.alloc(n, s);
        tmp_vals = tv.p;
    }
    const int passes = std::max(1, std::min(OMAXP, (bits + 7) / 8));
    const u32 ntiles = static_cast<u32>((n + OTILE - 1) / OTILE);
    // one zeroed block: histograms, bucket starts, tickets, tile counters, look-back status
    const size_t words = static_cast<size_t>(passes) * 256 * 2 + 1 + passes;
    const size_t status_off = (words * 4 + 255) / 256 * 256;
    const size_t bytes = status_off + sizeof(unsigned long long) * static_cast<size_t>(passes) * ntiles * 256;
    DevBuf<unsigned char> scratch(bytes, s);
    CUDA_CHECK(cudaMemsetAsync(scratch.p, 0, bytes, s));
    u32* ghist = reinterpret_cast<u32*>(scratch.p);
    u32* gstart = ghist + passes * 256;
    u32* ticket = gstart + passes * 256;
    u32* tiles = ticket + 1;
    auto* status = reinterpret_cast<unsigned long long*>(scratch.p + status_off);
    int dev = 0, sms = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const size_t hsmem = sizeof(u32) * passes * 256 * 32;
    // as many histogram CTAs as fit on every SM at once (32 KB of counters per pass)
    const u64 hper = std::max<u64>(1, std::min<u64>(6, (228u * 1024u) / (hsmem + 1024u)));
    const u32 hgrid = static_cast<u32>(std::min<u64>((n / 4 + OB - 1) / OB + 1, static_cast<u64>(sms) * hper));
    constexpr size_t kSmem = sizeof(u32) * 4 * OTILE;    // the tile + the digit-ordered tile
    constexpr size_t kSmemIp = sizeof(u32) * 3 * OTILE;  // the tile + its keys in digit order
    {  // once per device (the attribute is per device; its driver lock serialises sweep workers)
        static std::mutex mu;
        static std::set<int> done;
        std::lock_guard<std::mutex> g(mu);
        if (done.insert(dev).second) {
            CUDA_CHECK(cudaFuncSetAttribute(k_os_pass<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(kSmem)));
            CUDA_CHECK(cudaFuncSetAttribute(k_os_pass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(kSmem)));
            CUDA_CHECK(cudaFuncSetAttribute(k_os_pass_ip<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(kSmemIp)));
            CUDA_CHECK(cudaFuncSetAttribute(k_os_pass_ip<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(kSmemIp)));
            CUDA_CHECK(cudaFuncSetAttribute(k_os_pass_ip<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(kSmemIp)));
            CUDA_CHECK(cudaFuncSetAttribute(k_os_hist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(sizeof(u32) * OMAXP * 256 * 32)));
        }
    }
    LAUNCH_B("radix.hist", 4.0 * n, k_os_hist, hgrid, OB, hsmem, s, keys, n, passes, descending, ghist, gstart,
             ticket);
    // the bulk copies need 16-byte aligned sources (every tile starts 16 KB in)
    const bool bulk = ((reinterpret_cast<uintptr_t>(keys) | reinterpret_cast<uintptr_t>(vals) |
                        reinterpret_cast<uintptr_t>(tmp_keys) | reinterpret_cast<uintptr_t>(tmp_vals)) & 15u) == 0;
    static const int variant = std::getenv("HBP_RADIX_VARIANT") ? std::atoi(std::getenv("HBP_RADIX_VARIANT")) : 2;
    u32 *ki = keys, *vi = vals, *ko = tmp_keys, *vo = tmp_vals;
    for (int p = 0; p < passes; ++p) {
        if (variant == 3 || variant == 4)  // timing probes (tools/radix_bench.py; wrong output)
            LAUNCH_B("radix.scatter", 16.0 * n, (variant == 3 ? k_os_pass_ip<1> : k_os_pass_ip<2>), ntiles, OB,
                     kSmemIp, s, ki, vi, ko, vo, n, 8 * p, descending, gstart + p * 256,
                     status + static_cast<size_t>(p) * ntiles * 256, tiles + p, bulk, std::min(8, bits - 8 * p));
        else if (variant == 2)
            LAUNCH_B("radix.scatter", 16.0 * n, k_os_pass_ip<0>, ntiles, OB, kSmemIp, s, ki, vi, ko, vo, n, 8 * p,
                     descending, gstart + p * 256, status + static_cast<size_t>(p) * ntiles * 256, tiles + p, bulk,
                     std::min(8, bits - 8 * p));
        else if (variant == 0)
            LAUNCH_B("radix.scatter", 16.0 * n, k_os_pass<false>, ntiles, OB, kSmem, s, ki, vi, ko, vo, n,
                     8 * p, descending, gstart + p * 256, status + static_cast<size_t>(p) * ntiles * 256, tiles + p,
                     bulk, 8);
        else
            LAUNCH_B("radix.scatter", 16.0 * n, k_os_pass<true>, ntiles, OB, kSmem, s, ki, vi, ko, vo, n,
                     8 * p, descending, gstart + p * 256, status + static_cast<size_t>(p) * ntiles * 256, tiles + p,
                     bulk, std::min(8, bits - 8 * p));
        std::swap(ki, ko);
        std::swap(vi, vo);
    }
    if (ki != keys) {
        CUDA_CHECK(cudaMemcpyAsync(keys, ki, sizeof(u32) * n, cudaMemcpyDeviceToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(vals, vi, sizeof(u32) * n, cudaMemcpyDeviceToDevice, s));
    }
}

bool sort_entries_small(Ctx& c, u64* e, i64 n, const u32* key32, int key_bits, int len_bits) {
    if (n > kSmallN) return false;
    if (n <= 1) return true;
    set_small_sort_smem_once();
    LAUNCH_B("radix.small", 32.0 * n, k_small_sort_entries, 1, SB, sizeof(SmallSortSmem), c.stream, e,
             static_cast<u32>(n), key32, key_bits, len_bits);
    return true;
}

}  // namespace hbp_b200
