// scanfit.cu — best fit (BFS) and shortest-pack-first (SPFHP) packing.
//
// Both place items one at a time in a given order into the open pack picked
// by a rule over ALL open packs, else open a new one:
//   best fit  (packing.cpp:105-127, order = seeded shuffle, :244-248)
//             tightest pack with residual >= s, lowest index on ties;
//   SPFHP     (packing.cpp:129-162, order = length desc / id asc, the
//             histogram buckets walked longest first)
//             emptiest pack (largest residual) with residual >= s, lowest
//             index on ties -- the std::map<residual, set<index>> of the
//             reference, whose last key is the largest residual.
// Neither decomposes into runs the way first fit does (the pick depends on
// every residual), so one 1024-thread CTA owns the residual array -- in
// shared memory while it fits (57K packs), else in global memory (L2) -- and
// thread t owns packs t, t + 1024, ...: per item every thread scans its
// packs, two warp REDUX steps and one cross-warp step pick the pack, and the
// owner updates its residual in place (no barrier needed: the owner is the
// only reader). One __syncthreads per item.
//
// Output matches first_fit_runs: item -> (bin, slot) and leaves
// (residual << 32 | count) per bin, bins in creation order. Slots (rank of
// an item inside its bin) come from a stable radix sort of the bin column.
#include <cstdlib>
#include <vector>

#include "radix.cuh"
#include "scan.cuh"
#include "stages.cuh"

namespace hbp_b200 {
namespace {

constexpr int kFitThreads = 1024;
constexpr int kFitWarps = kFitThreads / 32;
constexpr int kFitChunk = 1024;  // items staged per round
constexpr unsigned kFull = 0xffffffffu;

// Fixed shared memory: lengths + bins of one chunk, two reduction buffers.
constexpr size_t kFitFixedSmem = sizeof(u32) * 2 * kFitChunk + sizeof(u64) * 2 * kFitWarps;

template <bool WORST>
__device__ __forceinline__ u64 warp_pick(u32 hi, u32 lo) {
    const u32 m = WORST ? __reduce_max_sync(kFull, hi) : __reduce_min_sync(kFull, hi);
    const u32 l = WORST ? __reduce_max_sync(kFull, hi == m ? lo : 0u) : __reduce_min_sync(kFull, hi == m ? lo : ~0u);
    return (static_cast<u64>(m) << 32) | l;
}

// Best fit: this thread's tightest pack with residual >= s (lowest index on
// ties: k ascending, strict <). Eight loads in flight per step.
__device__ __forceinline__ void best_of_mine(const u32* R, u32 tid, u32 P, u32 s, u32& br, u32& bi) {
    u32 k = tid;
    for (; k + 7u * kFitThreads < P; k += 8u * kFitThreads) {
        u32 r[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) r[q] = R[k + q * kFitThreads];
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (r[q] >= s && r[q] < br) {
                br = r[q];
                bi = k + q * kFitThreads;
            }
    }
    for (; k < P; k += kFitThreads) {
        const u32 r = R[k];
        if (r >= s && r < br) {
            br = r;
            bi = k;
        }
    }
}

// SPFHP: this thread's emptiest pack (largest residual, lowest index).
__device__ __forceinline__ void max_of_mine(const u32* R, u32 tid, u32 P, u32& lm, u32& li) {
    lm = 0u;
    li = ~0u;
    u32 k = tid;
    for (; k + 7u * kFitThreads < P; k += 8u * kFitThreads) {
        u32 r[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) r[q] = R[k + q * kFitThreads];
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (r[q] > lm) {
                lm = r[q];
                li = k + q * kFitThreads;
            }
    }
    for (; k < P; k += kFitThreads) {
        const u32 r = R[k];
        if (r > lm) {
            lm = r;
            li = k;
        }
    }
}

template <bool WORST, bool SMEM>
__global__ void __launch_bounds__(kFitThreads, 1)
    k_scan_fit(const u64* __restrict__ items, i64 n, u32 cap, u32* __restrict__ g_res, u32* __restrict__ bin_out,
               u32* __restrict__ cnt, u32* __restrict__ n_bins) {
    extern __shared__ __align__(16) unsigned char smem[];
    u64* s_red = reinterpret_cast<u64*>(smem);                 // [2][32]
    u32* s_len = reinterpret_cast<u32*>(s_red + 2 * kFitWarps);
    u32* s_bin = s_len + kFitChunk;
    u32* R = SMEM ? (s_bin + kFitChunk) : g_res;
    const u32 tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;

    u32 P = 0;              // bins opened so far (identical in every thread)
    u32 lm = 0u, li = ~0u;  // SPFHP: this thread's emptiest pack, kept current
    for (i64 base = 0; base < n; base += kFitChunk) {
        const int cnt_c = static_cast<int>(n - base < kFitChunk ? n - base : kFitChunk);
        if (static_cast<int>(tid) < cnt_c) s_len[tid] = entry_len(items[base + tid]);
        __syncthreads();
        for (int j = 0; j < cnt_c; ++j) {
            const u32 s = s_len[j];
            u32 br, bi;
            if (WORST) {
                // the emptiest pack only competes when it fits (packing.cpp:
                // 147-150: lower_bound(len) == end -> new pack)
                br = lm >= s ? lm : 0u;
                bi = lm >= s ? li : ~0u;
            } else {
                br = ~0u;
                bi = ~0u;
                best_of_mine(R, tid, P, s, br, bi);
            }
            const u64 wk = warp_pick<WORST>(br, WORST ? static_cast<u32>(~bi) : bi);
            u64* red = s_red + (j & 1) * kFitWarps;
            if (lane == 0) red[warp] = wk;
            __syncthreads();
            const u64 v = red[lane];
            const u64 bk = warp_pick<WORST>(static_cast<u32>(v >> 32), static_cast<u32>(v));
            const u32 hi = static_cast<u32>(bk >> 32);
            const bool found = WORST ? hi != 0u : hi != ~0u;
            u32 b;
            u32 nr;
            if (found) {
                b = WORST ? ~static_cast<u32>(bk) : static_cast<u32>(bk);
                nr = hi - s;
            } else {
                b = P++;
                nr = cap - s;
            }
            if ((b & (kFitThreads - 1)) == tid) {
                R[b] = nr;
                atomicAdd(cnt + b, 1u);
                s_bin[j] = b;
                if (WORST) {
                    if (found) {
                        max_of_mine(R, tid, P, lm, li);  // b was this thread's emptiest pack
                    } else if (nr > lm) {
                        lm = nr;  // a new pack has the highest index: it wins strictly larger only
                        li = b;
                    }
                }
            }
        }
        __syncthreads();
        if (static_cast<int>(tid) < cnt_c) bin_out[base + tid] = s_bin[tid];
        // s_len / s_bin are rewritten next round only after this barrier
        __syncthreads();
    }
    if (SMEM)
        for (u32 k = tid; k < P; k += kFitThreads) g_res[k] = R[k];
    if (tid == 0) *n_bins = P;
}

// ---- SPFHP on one warp: a 32-ary max tree over the packs -----------------
//
// Only the emptiest pack is ever asked for, so a tournament tree answers it
// without a block barrier: the top level (<= 32 nodes) lives in the lanes'
// registers, every level below in shared memory (the leaves in global
// memory once they outgrow it). Per item: REDUX max over the top level; if it
// fits, descend one 32-wide level per step (load, ballot on == max, first
// lane: the lowest index among the emptiest), then walk back up replacing
// one child and re-reducing. A new pack raises its ancestors to max(., v).
constexpr int kTreeMaxLevels = 6;

struct TreeLevels {
    int H;                         // levels in memory (0: the leaves are the register level)
    u64 off[kTreeMaxLevels];       // shared-memory offset (u32 units) of level h, if g[h] is null
    u32* g[kTreeMaxLevels];        // global level h, else null
    u64 size[kTreeMaxLevels];      // padded entries of level h
};

__global__ void __launch_bounds__(32, 1)
    k_wfd_tree(const u64* __restrict__ items, i64 n, u32 cap, TreeLevels T, u32* __restrict__ res,
               u32* __restrict__ bin_out, u32* __restrict__ cnt, u32* __restrict__ n_bins) {
    extern __shared__ __align__(16) u32 s_tree[];
    const u32 lane = threadIdx.x;
    u32* L[kTreeMaxLevels];
#pragma unroll
    for (int h = 0; h < kTreeMaxLevels; ++h) L[h] = h < T.H ? (T.g[h] ? T.g[h] : s_tree + T.off[h]) : nullptr;
#pragma unroll
    for (int h = 0; h < kTreeMaxLevels; ++h)
        if (h < T.H && !T.g[h])
            for (u64 k = lane; k < T.size[h]; k += 32) L[h][k] = 0u;
    __syncwarp();
    u32 top = 0u;  // register level: entry `lane`
    u32 P = 0;
    // Levels in use: the register level covers 32^(hA+1) packs; it is pushed
    // down into memory level hA when the packs outgrow it, so an item pays
    // for log32 of the packs open, not of the most there could be.
    int hA = 0;
    for (i64 base = 0; base < n; base += 32) {
        const int cnt_c = static_cast<int>(n - base < 32 ? n - base : 32);
        const u32 mylen = static_cast<int>(lane) < cnt_c ? entry_len(items[base + lane]) : 0u;
        u32 mybin = 0;
        for (int j = 0; j < cnt_c; ++j) {
            const u32 s = __shfl_sync(kFull, mylen, j);
            const u32 M = __reduce_max_sync(kFull, top);
            u32 leaf;
            if (M >= s) {
                u32 node = __ffs(__ballot_sync(kFull, top == M)) - 1;
                u32 v[kTreeMaxLevels];
#pragma unroll
                for (int h = kTreeMaxLevels - 1; h >= 0; --h) {
                    if (h < hA) {
                        v[h] = L[h][node * 32 + lane];
                        node = node * 32 + (__ffs(__ballot_sync(kFull, v[h] == M)) - 1);
                    }
                }
                leaf = node;
                u32 nv = M - s, idx = leaf;
#pragma unroll
                for (int h = 0; h < kTreeMaxLevels; ++h) {
                    if (h < hA) {
                        const u32 c = idx & 31u;
                        const u32 x = lane == c ? nv : v[h];
                        if (lane == c) L[h][idx] = nv;
                        nv = __reduce_max_sync(kFull, x);
                        idx >>= 5;
                    }
                }
                if (lane == idx) top = nv;
            } else {
                // No open pack fits: this item and the rest of its run of
                // equal lengths in the batch open new packs of k = cap / s
                // items each -- a new pack is the unique emptiest until it
                // holds k (every older pack is below s) -- placed at once.
                const u32 same = __ballot_sync(kFull, mylen == s && lane >= static_cast<u32>(j) &&
                                                          lane < static_cast<u32>(cnt_c)) >> j;
                const u32 c = ~same == 0u ? 32u : static_cast<u32>(__ffs(~same) - 1);
                const u32 k = cap / s;
                const u32 npk = (c + k - 1) / k;
                while (((P + npk - 1) >> (5 * hA)) >= 32u) {
#pragma unroll
                    for (int h = 0; h < kTreeMaxLevels; ++h)
                        if (h == hA) L[h][lane] = top;
                    const u32 mx = __reduce_max_sync(kFull, top);
                    top = lane == 0 ? mx : 0u;
                    ++hA;
                    __syncwarp();
                }
                if (lane < npk) {
                    const u32 take = min(k, c - lane * k);
                    const u32 v = cap - take * s;
                    u32 idx = P + lane;
#pragma unroll
                    for (int h = 0; h < kTreeMaxLevels; ++h) {
                        if (h < hA) {
                            atomicMax(L[h] + idx, v);
                            idx >>= 5;
                        }
                    }
                    atomicAdd(cnt + P + lane, take);
                }
                for (u32 q = 0; q < npk; ++q) {
                    const u32 v = cap - min(k, c - q * k) * s;
                    if (lane == ((P + q) >> (5 * hA)) && top < v) top = v;
                }
                if (lane >= static_cast<u32>(j) && lane < static_cast<u32>(j) + c) mybin = P + (lane - j) / k;
                P += npk;
                j += static_cast<int>(c) - 1;
                __syncwarp();
                continue;
            }
            __syncwarp();
            if (lane == 0) atomicAdd(cnt + leaf, 1u);
            if (static_cast<int>(lane) == j) mybin = leaf;
        }
        if (static_cast<int>(lane) < cnt_c) bin_out[base + lane] = mybin;
    }
    // residuals of the bins: the leaf level (or the register level)
    if (hA == 0 && T.H > 0) {
        L[0][lane] = top;
        __syncwarp();
    }
    if (T.H == 0) {
        if (lane < P) res[lane] = top;
    } else if (!T.g[0]) {
        for (u32 k = lane; k < P; k += 32) res[k] = L[0][k];
    }
    if (lane == 0) *n_bins = P;
}

__global__ void k_fit_leaves(const u32* __restrict__ res, const u32* __restrict__ cnt, u64 P, u64* __restrict__ leaves) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < P;
         i += static_cast<u64>(gridDim.x) * blockDim.x)
        leaves[i] = (static_cast<u64>(res[i]) << 32) | cnt[i];
}

// sorted (bin, position) pairs -> slot of each position
__global__ void k_fit_slots(const u32* __restrict__ sbin, const u32* __restrict__ spos, u64 n,
                            const u64* __restrict__ start, u32* __restrict__ slot) {
    for (u64 j = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; j < n;
         j += static_cast<u64>(gridDim.x) * blockDim.x)
        slot[spos[j]] = static_cast<u32>(j - start[sbin[j]]);
}

__global__ void k_iota_u32(u32* __restrict__ v, u64 n) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<u64>(gridDim.x) * blockDim.x)
        v[i] = static_cast<u32>(i);
}

template <bool WORST, bool SMEM>
void launch_fit(Ctx& c, const u64* items, i64 n, u32 cap, u32* res, u32* bins, u32* cnt, u32* nb, size_t smem,
                int smem_optin) {
    set_max_dynamic_smem_once(reinterpret_cast<const void*>(&k_scan_fit<WORST, SMEM>), smem_optin);
    LAUNCH_B("fit.scan", 12.0 * static_cast<double>(n), (k_scan_fit<WORST, SMEM>), 1, kFitThreads, smem, c.stream,
             items, n, cap, res, bins, cnt, nb);
}

int fit_bits(u64 maxval) {
    int b = 0;
    while (b < 32 && (maxval >> b) != 0) ++b;
    return b;
}

}  // namespace

FitResult scan_fit(Ctx& c, const u64* items, i64 n, u64* leaves, i64 max_bins, u32 cap, bool worst, u32* item_bin,
                   u32* item_slot) {
    FitResult fr;
    if (n <= 0) return fr;
    cudaStream_t s = c.stream;
    const u64 N = static_cast<u64>(n);
    const u64 pmax = std::min<u64>(N, static_cast<u64>(max_bins));
    DevBuf<u32> res(pmax, s), cnt(pmax, s), nb(1, s);
    cnt.zero();
    int dev = 0, smem_optin = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    CUDA_CHECK(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    const size_t need = kFitFixedSmem + sizeof(u32) * pmax;
    const char* fg = std::getenv("HBP_FIT_GLOBAL");  // tests: exercise the L2-resident residual array
    const bool force_global = fg && *fg && *fg != '0';
    const bool in_smem = !force_global && need <= static_cast<size_t>(smem_optin);
    const size_t smem = in_smem ? need : kFitFixedSmem;
    const char* fb = std::getenv("HBP_SPFHP_BLOCK");  // tests: the block-wide pick for SPFHP too
    if (worst && !(fb && *fb && *fb != '0')) {
        // level sizes, leaves first, each padded to 32; the level of <= 32
        // entries stays in registers
        TreeLevels T{};
        u64 sz = (pmax + 31) / 32 * 32;
        if (pmax <= 32) sz = 0;
        while (sz > 0) {
            if (T.H == kTreeMaxLevels) throw EngineError(HBP_ERR_VALIDATION, "spfhp: too many packs");
            T.size[T.H++] = sz;
            const u64 up = (sz / 32 + 31) / 32 * 32;
            if (sz / 32 <= 32) break;
            sz = up;
        }
        // shared memory for the upper levels, top down, while they fit
        u64 used = 0;
        int h = T.H - 1;
        for (; h >= 0; --h) {
            if (force_global || (used + T.size[h]) * sizeof(u32) > static_cast<size_t>(smem_optin)) break;
            T.off[h] = used;
            used += T.size[h];
        }
        std::vector<DevBuf<u32>> glv;
        for (int k = 0; k <= h; ++k) {
            if (k == 0) {
                // leaves in global memory are the residual array itself
                T.g[0] = res.p;
                CUDA_CHECK(cudaMemsetAsync(res.p, 0, sizeof(u32) * pmax, s));
                if (T.size[0] > pmax) {
                    glv.emplace_back(T.size[0], s);
                    glv.back().zero();
                    T.g[0] = glv.back().p;
                }
            } else {
                glv.emplace_back(T.size[k], s);
                glv.back().zero();
                T.g[k] = glv.back().p;
            }
        }
        const size_t tsmem = used * sizeof(u32);
        set_max_dynamic_smem_once(reinterpret_cast<const void*>(&k_wfd_tree), smem_optin);
        LAUNCH_B("fit.tree", 12.0 * static_cast<double>(n), k_wfd_tree, 1, 32, tsmem, s, items, n, cap, T, res.p,
                 item_bin, cnt.p, nb.p);
        if (T.g[0] && T.g[0] != res.p)
            CUDA_CHECK(cudaMemcpyAsync(res.p, T.g[0], sizeof(u32) * pmax, cudaMemcpyDeviceToDevice, s));
        CUDA_CHECK(cudaStreamSynchronize(s));  // glv lives until the kernel is done
    } else if (worst) {
        if (in_smem) launch_fit<true, true>(c, items, n, cap, res.p, item_bin, cnt.p, nb.p, smem, smem_optin);
        else launch_fit<true, false>(c, items, n, cap, res.p, item_bin, cnt.p, nb.p, smem, smem_optin);
    } else {
        if (in_smem) launch_fit<false, true>(c, items, n, cap, res.p, item_bin, cnt.p, nb.p, smem, smem_optin);
        else launch_fit<false, false>(c, items, n, cap, res.p, item_bin, cnt.p, nb.p, smem, smem_optin);
    }
    const u64 P = read_vector(c, nb.p, 1)[0];
    LAUNCH(k_fit_leaves, grid_for(P, 256), 256, 0, s, res.p, cnt.p, P, leaves);
    // slots: stable sort of positions by bin, rank inside each bin
    DevBuf<u32> kb(N, s), pos(N, s), tk(N, s), tv(N, s);
    DevBuf<u64> start(P + 1, s);
    CUDA_CHECK(cudaMemcpyAsync(kb.p, item_bin, sizeof(u32) * N, cudaMemcpyDeviceToDevice, s));
    LAUNCH(k_iota_u32, grid_for(N, 256), 256, 0, s, pos.p, N);
    radix_sort_pairs(c, kb.p, pos.p, n, fit_bits(P - 1), false, tk.p, tv.p);
    {
        const u32* cp = cnt.p;
        u64* sp = start.p;
        const i64 PP = static_cast<i64>(P);
        scan_exclusive<u64>(
            PP + 1, [=] __device__(i64 i) { return i < PP ? static_cast<u64>(cp[i]) : 0ull; },
            [=] __device__(i64 i, u64 v) { sp[i] = v; }, s, c.scan, "scan.fit1");
    }
    LAUNCH(k_fit_slots, grid_for(N, 256), 256, 0, s, kb.p, pos.p, N, start.p, item_slot);
    fr.bins = static_cast<i64>(P);
    fr.records = n;
    return fr;
}

}  // namespace hbp_b200
