// shuffle.cu — exact parallel Fisher-Yates.
//
// Reference: Rng::shuffle (include/hbp/rng.hpp:61-68): for i = m .. 2,
// j_i = uniform_int(0, i-1) (rejection sampling, rng.hpp:32-41), then
// swap(v[i-1], v[j_i]). The draws form a counter-based stream (rng.cuh), so
// all targets j_i are computed in parallel; a rejected draw (probability
// < i / 2^64) shifts every later draw by one and is repaired by a single-CTA
// fix-up kernel that only does work when a rejection was flagged.
//
// Applying the swaps in parallel: write W(q, i) for the first step after
// (smaller than) i in time -- i.e. the smallest step i' > i -- that targets
// position q. Then
//   src(i)   = value at position i-1 just before step i
//            = W(i-1, i) ? src(W(i-1, i)) : in[i-1]          (a chain)
//   out[i-1] = W(j_i, i) ? src(W(j_i, i)) : in[j_i]           (i >= 2)
//   out[0]   = S_0 non-empty ? src(min S_0) : in[0]
// where S_q is the ascending list of steps targeting q. The lists come from
// a counting sort of steps by target; each chain is followed to its root
// (depth ~ log m, measured max 19 at 1M). Output: source position per slot.
#include <cstdlib>
#include <vector>

#include "engine.cuh"
#include "rng.cuh"
#include "stages.cuh"

namespace hbp_b200 {

namespace {

#include "nfround.cuh"

// Draw for step i (m >= i >= 2) with `shift` rejected draws before it.
__device__ __forceinline__ u32 fy_target(u64 seed, u64 base, u64 m, u64 i, u64 shift, bool& rejected) {
    const u64 v = splitmix_draw(seed, base + m - i + 1 + shift);
    const u64 r = v % i;
    // v >= UINT64_MAX - UINT64_MAX % i  <=>  (v - r) + i overflows
    rejected = (v - r) > (~0ull - i);
    return static_cast<u32>(r);
}

// Rare path: a draw at step `rej` was rejected. Every step i <= rej then
// uses one more draw; repeat until no rejection remains. Run by one block.
__device__ void fy_fix_block(u64 seed, u64 base, u64 m, u32* __restrict__ tgt, u32* __restrict__ cnt, u64 rej0,
                             unsigned long long* __restrict__ used) {
    __shared__ unsigned long long s_rej;
    __shared__ unsigned long long s_next;
    u64 shift = 0;
    if (threadIdx.x == 0) s_rej = rej0;
    __syncthreads();
    while (s_rej != 0) {
        const u64 upto = s_rej;
        shift += 1;
        if (threadIdx.x == 0) s_next = 0;
        __syncthreads();
        for (u64 i = 2 + threadIdx.x; i <= upto; i += blockDim.x) {
            bool bad;
            const u32 j = fy_target(seed, base, m, i, shift, bad);
            // a rejection strictly inside the shifted suffix needs another pass
            if (bad) atomicMax(&s_next, static_cast<unsigned long long>(i));
            const u32 old = tgt[i];
            if (old != j) {
                atomicSub(&cnt[old], 1u);
                atomicAdd(&cnt[j], 1u);
                tgt[i] = j;
            }
        }
        __syncthreads();
        // the step that was rejected at `upto` now uses the next draw; if that
        // one is rejected too, s_next == upto and the loop shifts again.
        if (threadIdx.x == 0) s_rej = s_next;
        __syncthreads();
    }
    // draws the shuffle consumed: one per step plus one per rejection
    if (used && threadIdx.x == 0) *used = (m - 1) + shift;
}

// Targets and their counts; rej[0]: the highest rejected step. The last
// block to finish repairs from there (fy_fix_block; it returns at once when
// there is no rejection) -- no separate launch for the rare path.
__global__ void k_fy_targets(u64 seed, u64 base, u64 m, u32* __restrict__ tgt, u32* __restrict__ cnt,
                             unsigned long long* __restrict__ rej, u64 force, unsigned long long* __restrict__ used,
                             bool split_fix, bool scan_counts) {
    for (u64 i = 2 + blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i <= m;
         i += static_cast<u64>(gridDim.x) * blockDim.x) {
        bool bad;
        const u32 j = fy_target(seed, base, m, i, 0, bad);
        bad = bad || i == force;  // tests: hbp_test_set_force_reject
        if (bad) atomicMax(rej, static_cast<unsigned long long>(i));
        tgt[i] = j;
        atomicAdd(&cnt[j], 1u);
    }
    if (split_fix) return;
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(rej + 1, 1ull) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    fy_fix_block(seed, base, m, tgt, cnt, *reinterpret_cast<volatile unsigned long long*>(rej), used);
    if (!scan_counts) return;
    // small m: the counts' exclusive scan here too (one launch fewer per
    // shuffle); each thread a contiguous chunk, read through L2
    __shared__ u32 s_red[33];
    const u64 chunk = (m + blockDim.x - 1) / blockDim.x;
    const u64 a = threadIdx.x * chunk, b = a + chunk < m ? a + chunk : m;
    u32 sum = 0;
    for (u64 q = a; q < b; ++q) sum += __ldcg(cnt + q);
    u32 tot;
    u32 run = block_exclusive_scan<u32>(sum, s_red, tot);
    for (u64 q = a; q < b; ++q) {
        const u32 x = __ldcg(cnt + q);
        cnt[q] = run;
        run += x;
    }
}

__global__ void k_fy_fix(u64 seed, u64 base, u64 m, u32* __restrict__ tgt, u32* __restrict__ cnt,
                         const unsigned long long* __restrict__ rej, unsigned long long* __restrict__ used) {
    fy_fix_block(seed, base, m, tgt, cnt, *rej, used);
}

// cur[j]: the list offsets, advanced in place (one random atomic per step);
// afterwards cur[q] is the end of S_q, i.e. the start of S_{q+1}
__global__ void k_fy_scatter(u64 m, const u32* __restrict__ tgt, u32* __restrict__ cur, u32* __restrict__ bucket) {
    for (u64 i = 2 + blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i <= m;
         i += static_cast<u64>(gridDim.x) * blockDim.x) {
        bucket[atomicAdd(&cur[tgt[i]], 1u)] = static_cast<u32>(i);
    }
}

// One thread per position q: sort S_q ascending, emit successor links.
// ends[q]: end of S_q (its start is ends[q - 1], 0 for q = 0).
__device__ __forceinline__ void fy_list(u64 q, const u32* __restrict__ ends, u32* __restrict__ bucket,
                                        u32* __restrict__ nxt, u32* __restrict__ link, u32* __restrict__ first0) {
    const u32 a = q ? ends[q - 1] : 0u, b = ends[q];
    // insertion sort (lists are short: E|S_q| = ln(m/q))
    for (u32 x = a + 1; x < b; ++x) {
        const u32 v = bucket[x];
        u32 y = x;
        while (y > a && bucket[y - 1] > v) {
            bucket[y] = bucket[y - 1];
            --y;
        }
        bucket[y] = v;
    }
    for (u32 x = a; x < b; ++x) nxt[bucket[x]] = (x + 1 < b) ? bucket[x + 1] : kNone;
    if (q == 0) {
        *first0 = b > a ? bucket[a] : kNone;
    } else {
        // link(q+1) = smallest step > q+1 in S_q (all of S_q are >= q+1)
        u32 l = kNone;
        if (b > a) {
            const u32 e0 = bucket[a];
            l = (e0 == q + 1) ? (b - a > 1 ? bucket[a + 1] : kNone) : e0;
        }
        link[q + 1] = l;
    }
}

// Four positions per thread with their loads issued together: most lists
// hold at most two steps (E|S_q| = ln(m/q)), which are ordered in registers
// (nothing reads the bucket order afterwards); longer ones take fy_list.
__global__ void k_fy_lists(u64 m, const u32* __restrict__ ends, u32* __restrict__ bucket,
                           u32* __restrict__ nxt, u32* __restrict__ link, u32* __restrict__ first0) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 q0 = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; q0 < m; q0 += 4 * stride) {
        u32 a[4], b[4], e0[4], e1[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const u64 q = q0 + u * stride;
            a[u] = q < m && q > 0 ? ends[q - 1] : 0u;
            b[u] = q < m ? ends[q] : 0u;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const u32 len = b[u] - a[u];
            e0[u] = len >= 1 ? bucket[a[u]] : kNone;
            e1[u] = len >= 2 ? bucket[a[u] + 1] : kNone;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const u64 q = q0 + u * stride;
            if (q >= m) continue;
            const u32 len = b[u] - a[u];
            if (len > 2) {
                fy_list(q, ends, bucket, nxt, link, first0);
                continue;
            }
            u32 x0 = e0[u], x1 = e1[u];
            if (len == 2 && x1 < x0) {
                x0 = e1[u];
                x1 = e0[u];
            }
            if (len >= 1) nxt[x0] = len == 2 ? x1 : kNone;
            if (len == 2) nxt[x1] = kNone;
            if (q == 0) {
                *first0 = len ? x0 : kNone;
            } else {
                // link(q+1) = smallest step > q+1 in S_q (all of S_q are >= q+1)
                u32 l = kNone;
                if (len) l = (x0 == q + 1) ? (len > 1 ? x1 : kNone) : x0;
                link[q + 1] = l;
            }
        }
    }
}

// src[p] = the source position of slot p; with `in`, out[p] = in[src[p]]
// instead (the shuffle applied in the same pass, src not stored). A chain is
// followed to its root here, once per slot that needs it.
__device__ __forceinline__ u32 chain_root(const u32* __restrict__ link, u32 r) {
    u32 l = link[r];
    while (l != kNone) {
        r = l;
        l = link[r];
    }
    return r - 1;
}

// Source position of output slot p.
__device__ __forceinline__ u32 fy_source(u64 p, const u32* __restrict__ tgt, const u32* __restrict__ nxt,
                                         const u32* __restrict__ link, const u32* __restrict__ first0) {
    if (p == 0) {
        const u32 w = *first0;
        return (w != kNone) ? chain_root(link, w) : 0u;
    }
    const u64 i = p + 1;
    const u32 w = nxt[i];
    return (w != kNone) ? chain_root(link, w) : tgt[i];
}

__global__ void k_fy_sources(u64 m, const u32* __restrict__ tgt, const u32* __restrict__ nxt,
                             const u32* __restrict__ link, const u32* __restrict__ first0,
                             u32* __restrict__ src, const u64* __restrict__ in, u64* __restrict__ out) {
    for (u64 p = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; p < m;
         p += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u32 s = fy_source(p, tgt, nxt, link, first0);
        if (in) out[p] = in[s];
        else src[p] = s;
    }
}

template <typename T>
__global__ void k_gather(const T* __restrict__ in, const u32* __restrict__ src, T* __restrict__ out, u64 m) {
    for (u64 p = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; p < m;
         p += static_cast<u64>(gridDim.x) * blockDim.x) {
        out[p] = in[src[p]];
    }
}


// The whole shuffle of a small vector in one launch: one cluster of kFyCta
// CTAs (distributed over its threads, every phase of the multi-launch path,
// hardware cluster barriers in between; the arrays stay in L2). The plans of
// the sweep shuffle pools of thousands of samples 8 times per group, where
// the five launches per shuffle, not the work, bound the throughput.
constexpr int kFyCta = 8;
constexpr int kFyThreads = 1024;
constexpr u64 kFyClusterMax = 65536;

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// Every phase of the shuffle over one cluster's threads (kFyCta CTAs of any
// size), cluster barriers in between; the arrays stay in L2.
__device__ __forceinline__ void fy_cluster_phases(u64 seed, u64 base, u64 m, u32* __restrict__ tgt,
                                                  u32* __restrict__ cnt, u32* __restrict__ bucket,
                                                  u32* __restrict__ nxt, u32* __restrict__ link,
                                                  u32* __restrict__ first0, unsigned long long* __restrict__ rej,
                                                  u32* __restrict__ part, u64 force,
                                                  unsigned long long* __restrict__ used, u32* __restrict__ src,
                                                  const u64* __restrict__ in, u64* __restrict__ out) {
    const u32 NT = blockDim.x;
    const u64 T = static_cast<u64>(kFyCta) * NT;
    const u64 tid = blockIdx.x * static_cast<u64>(NT) + threadIdx.x;
    for (u64 q = tid; q <= m; q += T) cnt[q] = 0;
    cluster_sync_all();
    // targets and their counts
    for (u64 i = 2 + tid; i <= m; i += T) {
        bool bad;
        const u32 j = fy_target(seed, base, m, i, 0, bad);
        bad = bad || i == force;
        if (bad) atomicMax(rej, static_cast<unsigned long long>(i));
        tgt[i] = j;
        atomicAdd(&cnt[j], 1u);
    }
    cluster_sync_all();
    if (blockIdx.x == 0) fy_fix_block(seed, base, m, tgt, cnt, *reinterpret_cast<volatile unsigned long long*>(rej), used);
    cluster_sync_all();
    // exclusive scan of the counts in place: each CTA a contiguous part
    __shared__ u32 s_red[33];
    const u64 per = (m + kFyCta - 1) / kFyCta;
    const u64 p0 = blockIdx.x * per, p1 = p0 + per < m ? p0 + per : m;
    const u64 chunk = p1 > p0 ? (p1 - p0 + NT - 1) / NT : 0;
    const u64 a = p0 + threadIdx.x * chunk, b = a + chunk < p1 ? a + chunk : p1;
    u32 sum = 0;
    for (u64 q = a; q < b; ++q) sum += cnt[q];
    u32 tot;
    u32 run = block_exclusive_scan<u32>(sum, s_red, tot);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
    cluster_sync_all();
    for (unsigned k = 0; k < blockIdx.x; ++k) run += part[k];
    for (u64 q = a; q < b; ++q) {
        const u32 x = cnt[q];
        cnt[q] = run;
        run += x;
    }
    cluster_sync_all();
    for (u64 i = 2 + tid; i <= m; i += T) bucket[atomicAdd(&cnt[tgt[i]], 1u)] = static_cast<u32>(i);
    cluster_sync_all();
    for (u64 q = tid; q < m; q += T) fy_list(q, cnt, bucket, nxt, link, first0);
    cluster_sync_all();
    for (u64 p = tid; p < m; p += T) {
        const u32 sp = fy_source(p, tgt, nxt, link, first0);
        if (in) out[p] = in[sp];
        else src[p] = sp;
    }
}

__global__ void __cluster_dims__(kFyCta, 1, 1) __launch_bounds__(kFyThreads, 1)
    k_fy_cluster(u64 seed, u64 base, u64 m, u32* __restrict__ tgt, u32* __restrict__ cnt, u32* __restrict__ bucket,
                 u32* __restrict__ nxt, u32* __restrict__ link, u32* __restrict__ first0,
                 unsigned long long* __restrict__ rej, u32* __restrict__ part, u64 force,
                 unsigned long long* __restrict__ used, u32* __restrict__ src, const u64* __restrict__ in,
                 u64* __restrict__ out) {
    fy_cluster_phases(seed, base, m, tgt, cnt, bucket, nxt, link, first0, rej, part, force, used, src, in, out);
}

// Every ISF round of a small pool (isf_round, packing.cpp:171-185, x the
// strategy's iterations) in one launch: one cluster shuffles (the phases
// above) and then runs the next-fit round tile by tile (nfround.cuh: tiles
// claimed in order, look-backs among the cluster's CTAs); the pool size, the
// sink counters and the round's next input stay on the device. One launch and
// one read instead of two launches and one read per round.
struct IsfSmallArgs {
    const u64* seeds;  // per round (derive_seed(seed, "isf-round", r))
    int rounds;
    u64* A;            // the pool: in, and every round's remainder
    u64* B;            // a round's shuffled pool
    u32 *tgt, *cnt, *bucket, *nxt, *link, *first0, *part;
    unsigned long long* rej;
    u64 force;
    u64* nf_status;    // 3 * ntiles_max + 1 words, re-zeroed every round
    u64 cap, tmin;
    PackSink sink;
    u64* state;        // [0] pool size, [1] sink members, [2] sink packs
};

__global__ void __cluster_dims__(kFyCta, 1, 1) __launch_bounds__(NF_B, 1) k_isf_small(IsfSmallArgs q) {
    __shared__ u32 s_claim;
    for (int r = 0; r < q.rounds; ++r) {
        cluster_sync_all();
        const u64 m = *reinterpret_cast<volatile u64*>(q.state);
        if (m == 0) break;
        const u64 mbase = *reinterpret_cast<volatile u64*>(q.state + 1);
        const u64 pbase = *reinterpret_cast<volatile u64*>(q.state + 2);
        const u32 ntiles = static_cast<u32>((m + NF_T - 1) / NF_T);
        const u64 T = static_cast<u64>(kFyCta) * blockDim.x;
        const u64 tid = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x;
        if (tid == 0) *q.rej = 0;
        for (u64 k = tid; k < 3ull * ntiles + 1; k += T) q.nf_status[k] = 0;
        cluster_sync_all();
        fy_cluster_phases(q.seeds[r], 0, m, q.tgt, q.cnt, q.bucket, q.nxt, q.link, q.first0, q.rej, q.part, q.force,
                          nullptr, nullptr, q.A, q.B);
        cluster_sync_all();
        NfRoundArgs ra;
        ra.F = q.B;
        ra.m = m;
        ra.cap = q.cap;
        ra.tmin = q.tmin;
        ra.sink = q.sink;
        ra.mbase = mbase;
        ra.pbase = pbase;
        ra.newpool = q.A;
        ra.totals = q.state;
        ra.ntiles = ntiles;
        ra.xst = q.nf_status;
        ra.tvst = q.nf_status + ntiles;
        ra.lsst = q.nf_status + 2ull * ntiles;
        ra.tile_ctr = reinterpret_cast<u32*>(q.nf_status + 3ull * ntiles);
        for (;;) {
            if (threadIdx.x == 0) s_claim = atomicAdd(ra.tile_ctr, 1u);
            __syncthreads();
            const u32 tile = s_claim;
            __syncthreads();
            if (tile >= ntiles) break;
            nf_tile(ra, tile);
            __syncthreads();
        }
    }
}
}  // namespace

namespace {
void fy_run(Ctx& c, uint64_t seed, i64 m_signed, u32* src, const u64* in, u64* out, uint64_t draw_base,
            uint64_t* draws_used) {
    if (draws_used) *draws_used = 0;
    if (m_signed <= 0) return;
    const u64 m = static_cast<u64>(m_signed);
    cudaStream_t s = c.stream;
    if (m == 1) {
        if (in) CUDA_CHECK(cudaMemcpyAsync(out, in, sizeof(u64), cudaMemcpyDeviceToDevice, s));
        else CUDA_CHECK(cudaMemsetAsync(src, 0, sizeof(u32), s));
        return;
    }
    DevBuf<unsigned long long> used(draws_used ? 1 : 0, s);
    DevBuf<u32> tgt(m + 1, s), cnt(m + 1, s), bucket(m, s), nxt(m + 2, s), link(m + 2, s);
    static const bool no_cluster = std::getenv("HBP_FY_NOCLUSTER") != nullptr;  // A/B: the multi-launch path
    if (m <= kFyClusterMax && !no_cluster) {
        DevBuf<unsigned long long> rj(1, s), usd(draws_used ? 1 : 0, s);
        DevBuf<u32> part(kFyCta, s), f0(1, s);
        rj.zero();
        LAUNCH_B(in ? "fy.cluster_gather" : "fy.cluster", 40.0 * m, k_fy_cluster, kFyCta, kFyThreads, 0, s, seed,
                 draw_base, m, tgt.p, cnt.p, bucket.p, nxt.p, link.p, f0.p, rj.p, part.p, c.test_force_reject, usd.p,
                 src, in, out);
        if (draws_used) *draws_used = read_scalar(c, usd.p);
        return;
    }
    DevBuf<unsigned long long> rej(2, s);  // highest rejected step, finished blocks
    DevBuf<u32> first0(1, s);
    cnt.zero();
    rej.zero();
    const unsigned B = 256;
    const unsigned G = grid_for(m, B, 148u * 32u);
    // tests only (hbp_test_set_force_reject): treat the first draw of one
    // step as rejected, to exercise the repair on demand (a real rejection has
    // probability < m / 2^64)
    const u64 force = c.test_force_reject;
    static const bool split_fix = std::getenv("HBP_FY_SPLITFIX") != nullptr;  // A/B: separate fix-up launch
    // small shuffles scan the target counts in the targets kernel's last block
    constexpr u64 kScanInTargets = 8192;
    const bool scan_in = !split_fix && m <= kScanInTargets;
    LAUNCH_B("fy.targets", 12.0 * m, k_fy_targets, G, B, 0, s, seed, draw_base, m, tgt.p, cnt.p, rej.p, force,
             used.p, split_fix, scan_in);
    if (split_fix) LAUNCH(k_fy_fix, 1, 1024, 0, s, seed, draw_base, m, tgt.p, cnt.p, rej.p, used.p);
    // exclusive scan of per-target counts -> list offsets, in place (the
    // scan loads a whole tile before it stores it); the scatter then
    // advances them as cursors
    u32* cntp = cnt.p;
    if (!scan_in)
        scan_exclusive<u32>(
            static_cast<i64>(m), [=] __device__(i64 i) { return cntp[i]; },
            [=] __device__(i64 i, u32 v) { cntp[i] = v; }, s, c.scan, "scan.fy1");
    LAUNCH_B("fy.scatter", 16.0 * m, k_fy_scatter, G, B, 0, s, m, tgt.p, cnt.p, bucket.p);
    LAUNCH_B("fy.lists", 20.0 * m, k_fy_lists, G, B, 0, s, m, cnt.p, bucket.p, nxt.p, link.p, first0.p);
    if (in)
        LAUNCH_B("fy.sources_gather", 32.0 * m, k_fy_sources, G, B, 0, s, m, tgt.p, nxt.p, link.p, first0.p, nullptr, in,
                 out);
    else
        LAUNCH_B("fy.sources", 16.0 * m, k_fy_sources, G, B, 0, s, m, tgt.p, nxt.p, link.p, first0.p, src, nullptr,
                 nullptr);
    if (draws_used) *draws_used = read_scalar(c, used.p);
}
}  // namespace

void fy_source_positions(Ctx& c, uint64_t seed, i64 m, u32* src, uint64_t draw_base, uint64_t* draws_used) {
    fy_run(c, seed, m, src, nullptr, nullptr, draw_base, draws_used);
}

bool isf_small(Ctx& c, const std::vector<uint64_t>& seeds, u64* A, u64& cur, u32 cap, u64 tmin, PackSink sink,
               u64& n_members, u64& n_packs) {
    static const bool off = std::getenv("HBP_ISF_SPLIT") != nullptr;  // A/B: a shuffle and a next-fit launch per round
    const u64 m = cur;
    if (off || m == 0 || m > kFyClusterMax || seeds.empty()) return false;
    cudaStream_t s = c.stream;
    const u64 ntiles = (m + NF_T - 1) / NF_T;
    DevBuf<u64> B(m, s), status(3 * ntiles + 1, s), state(3, s), dseeds(seeds.size(), s);
    DevBuf<u32> tgt(m + 1, s), cnt(m + 1, s), bucket(m, s), nxt(m + 2, s), link(m + 2, s), first0(1, s), part(kFyCta, s);
    DevBuf<unsigned long long> rej(1, s);
    const u64 h_state[3] = {m, n_members, n_packs};
    CUDA_CHECK(cudaMemcpyAsync(state.p, h_state, sizeof(h_state), cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaMemcpyAsync(dseeds.p, seeds.data(), sizeof(u64) * seeds.size(), cudaMemcpyHostToDevice, s));
    IsfSmallArgs q;
    q.seeds = dseeds.p;
    q.rounds = static_cast<int>(seeds.size());
    q.A = A;
    q.B = B.p;
    q.tgt = tgt.p;
    q.cnt = cnt.p;
    q.bucket = bucket.p;
    q.nxt = nxt.p;
    q.link = link.p;
    q.first0 = first0.p;
    q.part = part.p;
    q.rej = rej.p;
    q.force = c.test_force_reject;
    q.nf_status = status.p;
    q.cap = cap;
    q.tmin = tmin;
    q.sink = sink;
    q.state = state.p;
    // algorithmic bytes: the rounds' shuffle and next-fit of the pool
    LAUNCH_B("isf.small", 64.0 * m * seeds.size(), k_isf_small, kFyCta, NF_B, NF_SMEM_FUSED, s, q);
    const auto h = read_vector(c, state.p, 3);  // (also orders the stack copies above)
    cur = h[0];
    n_members = h[1];
    n_packs = h[2];
    return true;
}

void fy_shuffle_u64(Ctx& c, uint64_t seed, i64 m, const u64* in, u64* out) {
    fy_run(c, seed, m, nullptr, in, out, 0, nullptr);
}



void gather_u64(Ctx& c, const u64* in, const u32* src, u64* out, i64 m) {
    if (m <= 0) return;
    LAUNCH_B("gather.u64", 20.0 * m, k_gather<u64>, grid_for(m, 256, 148u * 32u), 256, 0, c.stream, in, src, out,
             static_cast<u64>(m));
}

void gather_u32(Ctx& c, const u32* in, const u32* src, u32* out, i64 m) {
    if (m <= 0) return;
    LAUNCH(k_gather<u32>, grid_for(m, 256, 148u * 32u), 256, 0, c.stream, in, src, out, static_cast<u64>(m));
}

}  // namespace hbp_b200
