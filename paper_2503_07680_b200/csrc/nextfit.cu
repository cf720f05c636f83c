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
#include <cstdlib>

#include "engine.cuh"
#include "stages.cuh"

namespace hbp_b200 {

namespace {

#include "nfround.cuh"

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
// possible entries merge into it inside the tile. By pointer doubling in
// shared memory rather than a serial walk: with f(x) = next(x) while it
// stays in the tile (else x), F_k = f^(2^k) for k <= 11 gives every
// position's last node in the tile, last(x) = F_11(x); a chain from e
// merges into the chain from the tile start iff last(e) == last(start); the
// speculative chain's nodes f^t(start), t <= its length, are found by
// binary lifting, 11 lookups each, all in parallel.
constexpr int NF_LV = 12;  // F_0 .. F_11 (2^11 = NF_T)

__global__ void __launch_bounds__(NF_B) k_nf_tiles(const u32* __restrict__ nxt, u64 m, u32* __restrict__ spec,
                                                   u32* __restrict__ exitpos, u8* __restrict__ allconv) {
    extern __shared__ unsigned short s_F[];  // [NF_LV][NF_T]
    __shared__ u32 s_spec[NF_T / 32];
    __shared__ int s_ok;
    __shared__ u32 s_h0;
    const u64 a = static_cast<u64>(blockIdx.x) * NF_T;
    const u64 end = a + NF_T < m ? a + NF_T : m;
    const u32 len = static_cast<u32>(end - a);
    for (u32 i = threadIdx.x; i < NF_T; i += NF_B) {
        u32 f = i;
        if (i < len) {
            const u64 nx = nxt[a + i];
            if (nx < end) f = static_cast<u32>(nx - a);
        }
        s_F[i] = static_cast<unsigned short>(f);
    }
    for (u32 i = threadIdx.x; i < NF_T / 32; i += NF_B) s_spec[i] = 0;
    if (threadIdx.x == 0) s_ok = 1;
    __syncthreads();
    for (int k = 0; k + 1 < NF_LV; ++k) {
        const unsigned short* Fk = s_F + k * NF_T;
        unsigned short* Fn = s_F + (k + 1) * NF_T;
        for (u32 i = threadIdx.x; i < NF_T; i += NF_B) Fn[i] = Fk[Fk[i]];
        __syncthreads();
    }
    const unsigned short* last = s_F + (NF_LV - 1) * NF_T;
    const u32 last0 = last[0];
    if (threadIdx.x == 0) {
        // h0 = steps from the start to last0: largest t with f^t(0) != last0, plus one
        u32 x = 0, t = 0;
        for (int k = NF_LV - 2; k >= 0; --k) {
            const u32 y = s_F[k * NF_T + x];
            if (y != last0) {
                x = y;
                t += 1u << k;
            }
        }
        s_h0 = x == last0 ? t : t + 1;
        exitpos[blockIdx.x] = static_cast<u32>(nxt[a + last0]);
    }
    __syncthreads();
    const u32 h0 = s_h0;
    for (u32 t = threadIdx.x; t <= h0; t += NF_B) {
        u32 x = 0;
#pragma unroll
        for (int k = 0; k + 1 < NF_LV; ++k)
            if ((t >> k) & 1u) x = s_F[k * NF_T + x];
        atomicOr(&s_spec[x >> 5], 1u << (x & 31));
    }
    // entries into this tile lie in [a, next(a-1)]
    if (a > 0) {
        const u64 hi_entry = nxt[a - 1];
        if (hi_entry >= end) {
            if (threadIdx.x == 0) s_ok = 0;
        } else {
            for (u64 e = a + threadIdx.x; e <= hi_entry; e += NF_B)
                if (last[e - a] != last0) s_ok = 0;
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

// Final start flags: walk from the entry until the speculative chain, then
// copy it. Also the tile's freeze totals: frozen packs and their items
// among the packs starting here (fp << 31 | fe, both < 2^31), and 1 + the
// last pack start in the tile (0: none) for the emit kernel's carry-in.
__global__ void __launch_bounds__(NF_B) k_nf_flags(const u32* __restrict__ nxt, const u32* __restrict__ spec,
                                                   const u32* __restrict__ entry, const u64* __restrict__ P, u64 m,
                                                   u64 tmin, u32* __restrict__ flags, u64* __restrict__ tval,
                                                   u32* __restrict__ tlast) {
    __shared__ u32 s_flags[NF_T / 32];
    __shared__ u64 s_conv;
    __shared__ u64 s_sum[2];
    __shared__ u32 s_last[2];
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
    if (threadIdx.x < NF_T / 32) {  // two warps, one flags word each
        const u32 w = threadIdx.x;
        const u64 p0 = a + 32ull * w;
        u32 bits = 0;
        if (p0 < end) {
            bits = spec[static_cast<u64>(blockIdx.x) * (NF_T / 32) + w];
            // keep speculative bits at positions >= conv only
            if (conv >= p0 + 32) bits = 0;
            else if (conv > p0) bits &= ~((1u << (conv - p0)) - 1u);
            bits |= s_flags[w];
        }
        flags[static_cast<u64>(blockIdx.x) * (NF_T / 32) + w] = bits;
        u64 fe = 0, fp = 0;
        if (tval)  // freeze totals (next-fit rounds only)
            for (u32 b = bits; b; b &= b - 1) {
                const u64 st = p0 + __ffs(b) - 1;
                const u32 e = nxt[st];
                if (P[e] - P[st] >= tmin) {
                    fe += e - st;
                    ++fp;
                }
            }
        u64 v = warp_sum((fp << 31) | fe);
        u32 last = bits ? static_cast<u32>(p0 - a) + 32u - __clz(bits) : 0u;  // 1 + last start, tile-relative
        last = warp_max(last);
        if ((threadIdx.x & 31u) == 0) {
            s_sum[threadIdx.x >> 5] = v;
            s_last[threadIdx.x >> 5] = last;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (tval) tval[blockIdx.x] = s_sum[0] + s_sum[1];
        const u32 l = max(s_last[0], s_last[1]);
        tlast[blockIdx.x] = l ? static_cast<u32>(a) + l : 0u;
    }
}

// Freeze and emit, one tile per CTA. Every position knows its pack (the last
// start at or before it: within the thread, the block, or carried in from an
// earlier tile) and the inclusive count fz of frozen items up to it, so it
// goes to the sink at mbase + fz - (end - i) when its pack froze, else back
// to the pool at i - fz (pack order kept). Positions are read and written
// striped through shared memory; the blocked per-thread walk only computes
// destinations. Frozen pack starts also write (offset, total).

__global__ void __launch_bounds__(NF_B) k_nf_emit(const u64* __restrict__ F, u64 m, const u32* __restrict__ flags,
                                                  const u32* __restrict__ nxt, const u64* __restrict__ P, u64 tmin,
                                                  const u64* __restrict__ tpre, const u32* __restrict__ tlast,
                                                  PackSink sink, u64 mbase, u64 pbase, u64* __restrict__ newpool,
                                                  u64* __restrict__ totals, u32 ntiles) {
    constexpr u64 kElems = (1ull << 31) - 1;
    __shared__ u64 s_F[NF_T + NF_T / 32];
    __shared__ u32 s_dst[NF_T + NF_T / 32];
    __shared__ u32 s_fl[NF_T / 32];
    __shared__ u64 s_red[33];
    __shared__ u32 s_mx[NF_B / 32];
    __shared__ u32 s_carry;
    auto pad = [](u32 i) { return i + (i >> 5); };
    const u64 a = static_cast<u64>(blockIdx.x) * NF_T;
    const u32 len = static_cast<u32>((a + NF_T < m ? a + NF_T : m) - a);
    const u32 t = threadIdx.x;
    if (t < NF_T / 32) s_fl[t] = flags[static_cast<u64>(blockIdx.x) * (NF_T / 32) + t];
#pragma unroll
    for (int k = 0; k < EM_ITEMS; ++k) {
        const u32 li = k * NF_B + t;
        if (li < len) s_F[pad(li)] = F[a + li];
    }
    if (t == 0) {  // last pack start before the tile (tile 0 starts with one)
        u32 c = 0;
        for (u32 k = blockIdx.x; k > 0 && c == 0; --k) c = tlast[k - 1];
        s_carry = c;
    }
    __syncthreads();
    const u32 p0 = t * EM_ITEMS;
    const u32 bits = (s_fl[p0 >> 5] >> (p0 & 31)) & 0xffu;
    // own starts: end and frozen status
    u32 e_of[EM_ITEMS];
    u32 tot_of[EM_ITEMS];
    u64 v = 0;
#pragma unroll
    for (int j = 0; j < EM_ITEMS; ++j) {
        e_of[j] = 0;
        tot_of[j] = 0;
        if ((bits >> j) & 1u) {
            const u64 st = a + p0 + j;
            const u32 e = nxt[st];
            const u64 tot = P[e] - P[st];
            e_of[j] = e;
            tot_of[j] = static_cast<u32>(tot);
            if (tot >= tmin) v += (1ull << 31) | (e - st);
        }
    }
    u64 btot;
    const u64 ex = block_exclusive_scan<u64>(v, s_red, btot);
    const u32 my_last = bits ? static_cast<u32>(a) + p0 + 32u - __clz(bits) : 0u;  // 1 + last own start
    u32 prev = block_exclusive_max(my_last, s_mx);
    if (prev == 0) prev = s_carry;
    u64 run = tpre[blockIdx.x] + ex;  // frozen (packs << 31 | items) before my first position
    // the pack open at my first position, if it started earlier
    u32 e_cur = 0;
    bool frz = false;
    if (!(bits & 1u) && p0 < len) {
        const u64 st = prev - 1;
        e_cur = nxt[st];
        frz = P[e_cur] - P[st] >= tmin;
    }
#pragma unroll
    for (int j = 0; j < EM_ITEMS; ++j) {
        const u32 li = p0 + j;
        if (li >= len) break;
        const u64 i = a + li;
        if ((bits >> j) & 1u) {
            e_cur = e_of[j];
            frz = tot_of[j] >= tmin;
            if (frz) {
                const u64 q = pbase + (run >> 31);
                sink.pack_off[q] = mbase + (run & kElems);
                sink.pack_total[q] = tot_of[j];
                run += (1ull << 31) | (e_cur - i);
            }
        }
        const u64 fz = run & kElems;
        s_dst[pad(li)] = frz ? static_cast<u32>(mbase + fz - (e_cur - i)) | kToSink : static_cast<u32>(i - fz);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < EM_ITEMS; ++k) {
        const u32 li = k * NF_B + t;
        if (li < len) {
            const u32 d = s_dst[pad(li)];
            const u64 x = s_F[pad(li)];
            if (d & kToSink) sink.members[d & ~kToSink] = x;
            else newpool[d] = x;
        }
    }
    if (blockIdx.x == ntiles - 1 && t == 0) {  // totals: pool size and sink counters for the next round
        const u64 tt = tpre[blockIdx.x] + btot;
        totals[0] = m - (tt & kElems);
        totals[1] = mbase + (tt & kElems);
        totals[2] = pbase + (tt >> 31);
        *sink.n_members = totals[1];
        *sink.n_packs = totals[2];
    }
}


// A next-fit round in one launch: one tile per CTA (nfround.cuh nf_tile).
__global__ void __launch_bounds__(NF_B) k_nf_round(NfRoundArgs r) {
    __shared__ u32 s_claim;
    if (threadIdx.x == 0) s_claim = atomicAdd(r.tile_ctr, 1u);
    __syncthreads();
    nf_tile(r, s_claim);
}

}  // namespace

// Starts of the chain 0 -> nxt[0] -> nxt[nxt[0]] -> ... over m positions
// for any monotone nxt (nxt[s] > s): tile-parallel speculative chains,
// entries, final flags. flags: NF_T / 32 words per tile of NF_T positions
// (chain_flag_words(m) words); tlast: 1 + last start per tile (0: none).
u64 chain_flag_words(u64 m) { return ((m + NF_T - 1) / NF_T) * (NF_T / 32); }

void chain_starts(Ctx& c, const u32* nxt, u64 m, u32* flags, u32* tlast) {
    if (m == 0) return;
    cudaStream_t s = c.stream;
    const u32 ntiles = static_cast<u32>((m + NF_T - 1) / NF_T);
    DevBuf<u32> spec(static_cast<size_t>(ntiles) * (NF_T / 32), s);
    DevBuf<u32> exitpos(ntiles, s), entry(ntiles, s);
    DevBuf<u8> allconv(ntiles, s);
    const int smem = static_cast<int>(sizeof(unsigned short) * NF_LV * NF_T);
    set_max_dynamic_smem_once(reinterpret_cast<const void*>(k_nf_tiles), smem);
    LAUNCH_B("nf.tiles", 4.25 * m, k_nf_tiles, ntiles, NF_B, smem, s, nxt, m, spec.p, exitpos.p, allconv.p);
    LAUNCH(k_nf_entries, grid_for(ntiles, 128), 128, 0, s, nxt, spec.p, exitpos.p, allconv.p, m, ntiles, entry.p);
    LAUNCH_B("nf.flags", 4.25 * m, k_nf_flags, ntiles, NF_B, 0, s, nxt, spec.p, entry.p, static_cast<const u64*>(nullptr),
             m, 0ull, flags, static_cast<u64*>(nullptr), tlast);
}

// Packs one pool by next-fit over `F` (already in visiting order); packs
// with total >= tmin go to `sink` after the n_members / n_packs already
// there (updated), the rest to `newpool`. Returns the new pool size (one
// host sync).
i64 nextfit_freeze(Ctx& c, const u64* F, i64 m_signed, u32 cap, u64 tmin, PackSink sink, u64* newpool,
                   u64& n_members, u64& n_packs, const u64* P_in) {
    if (m_signed <= 0) return 0;
    const u64 m = static_cast<u64>(m_signed);
    cudaStream_t s = c.stream;
    DevBuf<u64> Pbuf;
    const u32 ntiles = static_cast<u32>((m + NF_T - 1) / NF_T);
    DevBuf<u64> newm(3, s);

    static const bool split = std::getenv("HBP_NF_SPLIT") != nullptr;  // A/B: the six-launch round
    // prefix sums of lengths in visiting order (m + 1 entries), for the
    // split round only (the fused round scans its own window), unless the
    // caller has them
    struct {
        const u64* p;
    } P{P_in};
    if (split && !P_in) {
        Pbuf.alloc(m + 1, s);
        P.p = Pbuf.p;
        u64* Pp = Pbuf.p;
        scan_exclusive<u64>(
            static_cast<i64>(m + 1), [=] __device__(i64 i) { return i < static_cast<i64>(m) ? (F[i] >> 32) : 0ull; },
            [=] __device__(i64 i, u64 v) { Pp[i] = v; }, s, c.scan, "scan.nf1");
    }
    if (split) {
        DevBuf<u32> nxt(m, s);
        DevBuf<u32> spec(static_cast<size_t>(ntiles) * (NF_T / 32), s), flags(static_cast<size_t>(ntiles) * (NF_T / 32), s);
        DevBuf<u32> exitpos(ntiles, s), entry(ntiles, s);
        DevBuf<u8> allconv(ntiles, s);
        LAUNCH_B("nf.next", 12.0 * m, k_nf_next, grid_for(m, 256, 148u * 32u), 256, 0, s, P.p, m, static_cast<u64>(cap),
                 nxt.p);
        const int smem = static_cast<int>(sizeof(unsigned short) * NF_LV * NF_T);
        set_max_dynamic_smem_once(reinterpret_cast<const void*>(k_nf_tiles), smem);
        LAUNCH_B("nf.tiles", 4.25 * m, k_nf_tiles, ntiles, NF_B, smem, s, nxt.p, m, spec.p, exitpos.p, allconv.p);
        LAUNCH(k_nf_entries, grid_for(ntiles, 128), 128, 0, s, nxt.p, spec.p, exitpos.p, allconv.p, m, ntiles, entry.p);
        DevBuf<u64> tval(ntiles, s), tpre(ntiles, s);
        DevBuf<u32> tlast(ntiles, s);
        LAUNCH_B("nf.flags", 4.25 * m, k_nf_flags, ntiles, NF_B, 0, s, nxt.p, spec.p, entry.p, P.p, m, tmin, flags.p,
                 tval.p, tlast.p);
        {
            const u64* tv = tval.p;
            u64* tp = tpre.p;
            scan_exclusive<u64>(
                static_cast<i64>(ntiles), [=] __device__(i64 i) { return tv[i]; },
                [=] __device__(i64 i, u64 v) { tp[i] = v; }, s, c.scan, "nf.tiles_scan");
        }
        LAUNCH_B("nf.freeze_emit", 16.125 * m, k_nf_emit, ntiles, NF_B, 0, s, F, m, flags.p, nxt.p, P.p, tmin, tpre.p,
                 tlast.p, sink, n_members, n_packs, newpool, newm.p, ntiles);
        const auto t = read_vector(c, newm.p, 3);
        n_members = t[1];
        n_packs = t[2];
        return static_cast<i64>(t[0]);
    }
    // status words of the fused round: exits, frozen totals, last starts, tile counter
    DevBuf<u64> st(3ull * ntiles + 1, s);
    st.zero();
    NfRoundArgs ra;
    ra.F = F;
    ra.m = m;
    ra.cap = cap;
    ra.tmin = tmin;
    ra.sink = sink;
    ra.mbase = n_members;
    ra.pbase = n_packs;
    ra.newpool = newpool;
    ra.totals = newm.p;
    ra.ntiles = ntiles;
    ra.xst = st.p;
    ra.tvst = st.p + ntiles;
    ra.lsst = st.p + 2ull * ntiles;
    ra.tile_ctr = reinterpret_cast<u32*>(st.p + 3ull * ntiles);
    set_max_dynamic_smem_once(reinterpret_cast<const void*>(k_nf_round), NF_SMEM_FUSED);
    // algorithmic bytes: entries in (lengths, then the entries) and out: 24 B
    LAUNCH_B("nf.round", 24.0 * m, k_nf_round, ntiles, NF_B, NF_SMEM_FUSED, s, ra);
    const auto t = read_vector(c, newm.p, 3);
    n_members = t[1];
    n_packs = t[2];
    return static_cast<i64>(t[0]);
}

}  // namespace hbp_b200
