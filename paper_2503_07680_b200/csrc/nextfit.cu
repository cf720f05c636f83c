// nextfit.cu — one ISF round (and plain next-fit) on the GPU.
//
// Reference: isf_round (src/packing.cpp:171-185) = shuffle, sequential_fill
// (packing.cpp:69-82, next-fit), freeze every pack whose total reaches
// double(capacity) * threshold, return the rest to the pool in pack order.
//
// Next-fit in parallel. With P the exclusive prefix sum of lengths, the pack
// opened at position s ends at next(s) = max{e : P[e] - P[s] <= cap}; the
// packs are the chain 0 -> next(0) -> ... . next() is monotone, and two
// chains in the same sequence that ever share a start coincide afterwards.
// So every tile of T positions walks a speculative chain from its first
// position; the true chain enters tile k somewhere in [a_k, next(a_k - 1)]
// and, for almost every tile, every such entry merges into the speculative
// chain inside the tile ("all-convergent"): then the tile's exit is known
// without knowing its entry and tiles resolve in parallel. Only maximal runs
// of non-convergent tiles are walked sequentially (one thread per run).
#include "engine.cuh"
#include "stages.cuh"

namespace hbp_b200 {

namespace {

constexpr int NF_T = 2048;  // positions per tile
constexpr int NF_B = 256;

__device__ __forceinline__ u32 ent_len(u64 e) { return static_cast<u32>(e >> 32); }

// next[s] by binary search over the prefix sums (pack spans <= cap items).
__global__ void k_nf_next(const u64* __restrict__ P, u64 m, u64 cap, u32* __restrict__ nxt) {
    for (u64 s = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; s < m;
         s += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u64 limit = P[s] + cap;
        const u64 top = s + cap < m ? s + cap : m;
        // gallop from s + 1 (packs hold few items: the probes stay in the
        // same cache lines), then bisect the last doubling
        u64 lo = s + 1, step = 1;
        while (lo + step <= top && P[lo + step] <= limit) {
            lo += step;
            step <<= 1;
        }
        u64 hi = lo + step - 1 < top ? lo + step - 1 : top;
        while (lo < hi) {
            const u64 mid = (lo + hi + 1) >> 1;
            if (P[mid] <= limit) lo = mid;
            else hi = mid - 1;
        }
        nxt[s] = static_cast<u32>(lo);
    }
}

// Per tile: speculative chain from the tile start, its exit, and whether all
// possible entries merge into it inside the tile.
__global__ void __launch_bounds__(NF_B) k_nf_tiles(const u32* __restrict__ nxt, u64 m, u32* __restrict__ spec,
                                                   u32* __restrict__ exitpos, u8* __restrict__ allconv) {
    __shared__ u32 s_next[NF_T];
    __shared__ u32 s_spec[NF_T / 32];
    __shared__ int s_ok;
    const u64 a = static_cast<u64>(blockIdx.x) * NF_T;
    const u64 end = a + NF_T < m ? a + NF_T : m;
    const u32 len = static_cast<u32>(end - a);
    for (u32 i = threadIdx.x; i < NF_T; i += NF_B) s_next[i] = i < len ? nxt[a + i] : static_cast<u32>(end);
    for (u32 i = threadIdx.x; i < NF_T / 32; i += NF_B) s_spec[i] = 0;
    if (threadIdx.x == 0) s_ok = 1;
    __syncthreads();
    if (threadIdx.x == 0) {
        u64 s = a;
        while (s < end) {
            const u32 r = static_cast<u32>(s - a);
            s_spec[r >> 5] |= 1u << (r & 31);
            s = s_next[r];
        }
        exitpos[blockIdx.x] = static_cast<u32>(s);
    }
    __syncthreads();
    // entries into this tile lie in [a, next(a-1)]
    if (a > 0) {
        const u64 hi_entry = nxt[a - 1];
        if (hi_entry >= end) {
            if (threadIdx.x == 0) s_ok = 0;
        } else {
            for (u64 e = a + threadIdx.x; e <= hi_entry; e += NF_B) {
                u64 s = e;
                bool conv = false;
                while (s < end) {
                    const u32 r = static_cast<u32>(s - a);
                    if (s_spec[r >> 5] & (1u << (r & 31))) {
                        conv = true;
                        break;
                    }
                    s = s_next[r];
                }
                if (!conv) s_ok = 0;
            }
        }
    }
    __syncthreads();
    for (u32 i = threadIdx.x; i < NF_T / 32; i += NF_B) spec[static_cast<u64>(blockIdx.x) * (NF_T / 32) + i] = s_spec[i];
    if (threadIdx.x == 0) allconv[blockIdx.x] = static_cast<u8>(s_ok);
}

__device__ __forceinline__ bool spec_bit(const u32* spec, u64 pos) {
    return (spec[pos >> 5] >> (pos & 31)) & 1u;
}

// Entry of every tile. Tiles after an all-convergent tile take its exit;
// a run of non-convergent tiles is walked by the thread of its first tile.
__global__ void k_nf_entries(const u32* __restrict__ nxt, const u32* __restrict__ spec,
                             const u32* __restrict__ exitpos, const u8* __restrict__ allconv, u64 m, u32 ntiles,
                             u32* __restrict__ entry) {
    for (u32 k = blockIdx.x * blockDim.x + threadIdx.x; k < ntiles; k += gridDim.x * blockDim.x) {
        if (k == 0) {
            entry[0] = 0;
            continue;
        }
        const bool prev_conv = (k - 1 == 0) || allconv[k - 1];
        if (prev_conv) {
            entry[k] = exitpos[k - 1];
            continue;
        }
        // tile k-1 is not all-convergent; only the first tile of the run walks
        const bool run_start = (k - 1 == 1) || (k - 1 == 0) || allconv[k - 2];
        if (!run_start) continue;
        u32 t = k - 1;
        u64 e = (t == 0) ? 0 : exitpos[t - 1];  // entry of tile t (tile t-1 convergent)
        while (true) {
            const u64 ta = static_cast<u64>(t) * NF_T;
            const u64 tend = ta + NF_T < m ? ta + NF_T : m;
            u64 s = e;
            while (s < tend && !spec_bit(spec, s)) s = nxt[s];
            const u64 out = (s < tend) ? exitpos[t] : s;
            entry[t + 1] = static_cast<u32>(out);
            ++t;
            if (t >= ntiles || allconv[t]) break;
            e = out;
        }
    }
}

// Final start flags: walk from the entry until the speculative chain, then copy it.
__global__ void __launch_bounds__(NF_B) k_nf_flags(const u32* __restrict__ nxt, const u32* __restrict__ spec,
                                                   const u32* __restrict__ entry, u64 m, u32* __restrict__ flags) {
    __shared__ u32 s_flags[NF_T / 32];
    __shared__ u64 s_conv;
    const u64 a = static_cast<u64>(blockIdx.x) * NF_T;
    const u64 end = a + NF_T < m ? a + NF_T : m;
    for (u32 i = threadIdx.x; i < NF_T / 32; i += NF_B) s_flags[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        u64 s = entry[blockIdx.x];
        while (s < end && !spec_bit(spec, s)) {
            const u32 r = static_cast<u32>(s - a);
            s_flags[r >> 5] |= 1u << (r & 31);
            s = nxt[s];
        }
        s_conv = s;  // from here on the speculative chain is the true chain
    }
    __syncthreads();
    const u64 conv = s_conv;
    for (u32 w = threadIdx.x; w < NF_T / 32; w += NF_B) {
        const u64 p0 = a + 32ull * w;
        if (p0 >= end) {
            flags[static_cast<u64>(blockIdx.x) * (NF_T / 32) + w] = 0;
            continue;
        }
        u32 bits = spec[static_cast<u64>(blockIdx.x) * (NF_T / 32) + w];
        // keep speculative bits at positions >= conv only
        if (conv >= p0 + 32) bits = 0;
        else if (conv > p0) bits &= ~((1u << (conv - p0)) - 1u);
        flags[static_cast<u64>(blockIdx.x) * (NF_T / 32) + w] = bits | s_flags[w];
    }
}

}  // namespace

// Packs one pool by next-fit over `F` (already in visiting order); packs
// with total >= tmin go to `sink` after the n_members / n_packs already
// there (updated), the rest to `newpool`. Returns the new pool size (one
// host sync).
i64 nextfit_freeze(Ctx& c, const u64* F, i64 m_signed, u32 cap, u64 tmin, PackSink sink, u64* newpool,
                   u64& n_members, u64& n_packs) {
    if (m_signed <= 0) return 0;
    const u64 m = static_cast<u64>(m_signed);
    cudaStream_t s = c.stream;
    DevBuf<u64> P(m + 1, s);
    DevBuf<u32> nxt(m, s);
    const u32 ntiles = static_cast<u32>((m + NF_T - 1) / NF_T);
    DevBuf<u32> spec(static_cast<size_t>(ntiles) * (NF_T / 32), s), flags(static_cast<size_t>(ntiles) * (NF_T / 32), s);
    DevBuf<u32> exitpos(ntiles, s), entry(ntiles, s);
    DevBuf<u8> allconv(ntiles, s);
    DevBuf<u64> newm(3, s);

    // prefix sums of lengths in visiting order (m + 1 entries)
    {
        u64* Pp = P.p;
        scan_exclusive<u64>(
            static_cast<i64>(m + 1), [=] __device__(i64 i) { return i < static_cast<i64>(m) ? (F[i] >> 32) : 0ull; },
            [=] __device__(i64 i, u64 v) { Pp[i] = v; }, s, c.scan);
    }
    LAUNCH_B("nf.next", 12.0 * m, k_nf_next, grid_for(m, 256, 148u * 32u), 256, 0, s, P.p, m, static_cast<u64>(cap),
             nxt.p);
    LAUNCH_B("nf.tiles", 4.25 * m, k_nf_tiles, ntiles, NF_B, 0, s, nxt.p, m, spec.p, exitpos.p, allconv.p);
    LAUNCH(k_nf_entries, grid_for(ntiles, 128), 128, 0, s, nxt.p, spec.p, exitpos.p, allconv.p, m, ntiles, entry.p);
    LAUNCH(k_nf_flags, ntiles, NF_B, 0, s, nxt.p, spec.p, entry.p, m, flags.p);
    // One scan over positions enumerates the frozen packs and emits every
    // pack from its start position: value (frozen packs << 31 | frozen
    // items) at each frozen pack start; a frozen pack goes to the sink at
    // (packs before, items before), any other pack back to the pool at its
    // position minus the frozen items before it (pack order kept).
    {
        const u32* fl = flags.p;
        const u32* nx = nxt.p;
        const u64* Pp = P.p;
        u64* nm = newm.p;
        const i64 mm = static_cast<i64>(m);
        const u64 mbase = n_members, pbase = n_packs;
        constexpr u64 kElems = (1ull << 31) - 1;
        auto frozen_value = [=] __device__(i64 i) -> u64 {
            if (!((fl[i >> 5] >> (i & 31)) & 1u)) return 0ull;
            const u32 e = nx[i];
            return Pp[e] - Pp[i] >= tmin ? ((1ull << 31) | (e - static_cast<u64>(i))) : 0ull;
        };
        scan_exclusive<u64>(
            mm, frozen_value,
            [=] __device__(i64 i, u64 v) {
                const u64 own = frozen_value(i);
                if (i == mm - 1) {  // totals: pool size and sink counters for the next round
                    const u64 t = v + own;
                    nm[0] = static_cast<u64>(mm) - (t & kElems);
                    nm[1] = mbase + (t & kElems);
                    nm[2] = pbase + (t >> 31);
                    *sink.n_members = nm[1];
                    *sink.n_packs = nm[2];
                }
                if (!((fl[i >> 5] >> (i & 31)) & 1u)) return;
                const u32 e = nx[i];
                const u64 fz_elems = v & kElems;
                if (own) {
                    const u64 q = pbase + (v >> 31);
                    const u64 dst = mbase + fz_elems;
                    u64 att = 0;
                    for (u64 k = static_cast<u64>(i); k < e; ++k) {
                        const u64 x = F[k];
                        const u64 l = ent_len(x);
                        att += l * l;
                        sink.members[dst + (k - i)] = x;
                    }
                    sink.pack_off[q] = dst;
                    sink.pack_total[q] = static_cast<u32>(Pp[e] - Pp[i]);
                    sink.pack_att[q] = att;
                } else {
                    const u64 dst = static_cast<u64>(i) - fz_elems;
                    for (u64 k = static_cast<u64>(i); k < e; ++k) newpool[dst + (k - i)] = F[k];
                }
            },
            s, c.scan, "nf.freeze_emit", 24.0);
    }
    const auto t = read_vector(c, newm.p, 3);
    n_members = t[1];
    n_packs = t[2];
    return static_cast<i64>(t[0]);
}

}  // namespace hbp_b200
