// nfround.cuh — one next-fit round, tile by tile (nextfit.cu k_nf_round,
// shuffle.cu's small-pool ISF kernel). Included inside an anonymous
// namespace of hbp_b200 after stages.cuh / common.cuh.
#pragma once

constexpr int NF_T = 2048;  // positions per tile
constexpr int NF_B = 256;

// Block-wide exclusive max over threads (values >= 0; 0 before thread 0).
__device__ __forceinline__ u32 block_exclusive_max(u32 v, u32* smem) {
    const unsigned lane = lane_id(), wid = warp_id();
    u32 inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= static_cast<unsigned>(o)) inc = max(inc, t);
    }
    if (lane == 31) smem[wid] = inc;
    __syncthreads();
    u32 before = 0;
    for (unsigned q = 0; q < wid; ++q) before = max(before, smem[q]);
    u32 ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) ex = 0;
    __syncthreads();
    return max(before, ex);
}

constexpr int EM_ITEMS = NF_T / NF_B;  // 8 positions per thread
constexpr u32 kToSink = 0x80000000u;

// ---------------------------------------------------------------------------
// One next-fit round in one launch (after the prefix sums P): per tile of
// NF_T positions, in tile order claimed by an atomic counter so that every
// earlier tile is running or done:
//   next()    gallop over P for the tile's positions (no nxt array in HBM)
//   spec      pointer doubling as in k_nf_tiles: the speculative chain from
//             the tile start, its exit, all-convergence
//   entry     the exit of tile k-1, published as soon as it is known (at
//             once for an all-convergent tile, after its own entry and walk
//             otherwise); only non-convergent tiles wait on a predecessor
//   flags     walk from the entry into the speculative chain; frozen packs
//             and items among the tile's starts, its last start
//   look-back frozen totals of the tiles before (decoupled look-back) and the
//             last start before the tile (the nearest earlier tile with one)
//   emit      as k_nf_emit
// Replaces next, tiles, entries, flags, the tile scan and emit (6 launches,
// the nxt / spec / flags arrays).
// ---------------------------------------------------------------------------
constexpr u64 kXKnown = 1ull << 63;  // exit word: the tile's true exit is known
constexpr u64 kTvAgg = 1ull << 62, kTvInc = 2ull << 62, kTvMask = (1ull << 62) - 1;
constexpr u64 kLsKnown = 1ull << 63;  // last-start word: known | total of that pack << 32 | 1 + last start (0: none)

__device__ __forceinline__ u32 nf_gallop(const u64* __restrict__ P, u64 s, u64 m, u64 cap) {
    const u64 limit = P[s] + cap;
    const u64 top = s + cap < m ? s + cap : m;
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
    return static_cast<u32>(lo);
}

__device__ __forceinline__ u64 ld_acquire_u64(const u64* p) {
    u64 v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(u64* p, u64 v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct NfRoundArgs {
    const u64* F;
    u64 m, cap, tmin;
    PackSink sink;
    u64 mbase, pbase;
    u64* newpool;
    u64* totals;
    u32 ntiles;
    u32* tile_ctr;
    u64* xst;   // [ntiles] kXKnown | true exit
    u64* tvst;  // [ntiles] look-back words of the frozen totals
    u64* lsst;  // [ntiles] kLsKnown | (last pack's total << 32) | (1 + last start)
};

// a staging region (first the window's local prefix sums, last the emit's
// entries and destinations) + next + pack totals
constexpr int NF_PW = 1024;  // prefix sums staged past the tile for next()
constexpr size_t NF_STAGE = sizeof(u64) * (NF_T + NF_PW + 1) > sizeof(u64) * (NF_T + NF_T / 32) + sizeof(u32) * (NF_T + NF_T / 32)
                                ? sizeof(u64) * (NF_T + NF_PW + 1)
                                : sizeof(u64) * (NF_T + NF_T / 32) + sizeof(u32) * (NF_T + NF_T / 32);
static_assert(sizeof(unsigned short) * 5 * NF_T <= NF_STAGE, "the chain's levels fit the staging region");
constexpr int NF_SMEM_FUSED = static_cast<int>((NF_STAGE + 15) / 16 * 16 + 2 * sizeof(u32) * NF_T);

// One tile of a next-fit round (k_nf_round: one per CTA; the small-pool ISF
// kernel: a loop over the tiles its cluster claims). Every earlier tile is
// running or done when this one waits on it.
__device__ __forceinline__ void nf_tile(const NfRoundArgs& r, u32 tile) {
    constexpr u64 kElems = (1ull << 31) - 1;
    extern __shared__ __align__(16) unsigned char nf_smem[];
    auto* s_nx = reinterpret_cast<u32*>(nf_smem + (NF_STAGE + 15) / 16 * 16);  // absolute next
    auto* s_tot = s_nx + NF_T;                                        // pack total from each position
    auto* s_P = reinterpret_cast<u64*>(nf_smem);                      // first: the window's local prefix sums
    auto* s_F = reinterpret_cast<u64*>(nf_smem);                      // emit: entries (padded), over the window
    auto* s_dst = reinterpret_cast<u32*>(s_F + NF_T + NF_T / 32);     // emit: destinations (padded)
    __shared__ u32 s_spec[NF_T / 32];
    __shared__ u32 s_fl[NF_T / 32];
    __shared__ u64 s_red[33];
    __shared__ u32 s_mx[NF_B / 32];
    __shared__ u64 s_tv[2];
    __shared__ u32 s_last2[2];
    __shared__ u32 s_h0, s_hi_entry, s_carry, s_carry_tot;
    __shared__ u64 s_entry, s_conv, s_tpre;
    __shared__ int s_ok;
    auto pad = [](u32 i) { return i + (i >> 5); };
    const u32 t = threadIdx.x;
    const u64 m = r.m;
    const u64 a = static_cast<u64>(tile) * NF_T;
    const u64 end = a + NF_T < m ? a + NF_T : m;
    const u32 len = static_cast<u32>(end - a);

    // lengths of the tile and NF_PW positions past it, scanned in shared
    // memory into local prefix sums (Pl(x) = sum of lengths in [a, x)); every
    // position's next() and pack total come from a gallop over them. A pack
    // running past the window (tiny items) is summed on from the entries.
    const u64 pend = end + NF_PW < m ? end + NF_PW : m;  // window [a, pend)
    const u32 wn = static_cast<u32>(pend - a);
    const u64* __restrict__ F = r.F;
    constexpr u32 kWI = (NF_T + NF_PW + NF_B) / NF_B;  // window positions per thread (contiguous)
    for (u32 x = t; x < wn; x += NF_B) s_P[x] = F[a + x] >> 32;  // striped loads
    __syncthreads();
    {
        u64 v[kWI];
        u64 sum = 0;
#pragma unroll
        for (u32 k = 0; k < kWI; ++k) {
            const u32 x = t * kWI + k;
            v[k] = x < wn ? s_P[x] : 0ull;
            sum += v[k];
        }
        u64 tot;
        u64 run = block_exclusive_scan<u64>(sum, s_red, tot);  // (syncs: every read above is done)
#pragma unroll
        for (u32 k = 0; k < kWI; ++k) {
            const u32 x = t * kWI + k;
            if (x < wn) s_P[x] = run;
            run += v[k];
        }
        if (t == 0) s_P[wn] = tot;
    }
    __syncthreads();
    const u64 cap = r.cap;
    // the pack from position sp (local prefix base = Pl(sp), limit = base + budget):
    // its end e (largest e <= top with Pl(e) <= limit) and total Pl(e) - base
    auto pack_from = [&](u64 sp, u64 base, u64 limit, u64 top, u32& e_out, u32& tot_out) {
        const u64 wtop = top < pend ? top : pend;
        u64 lo = sp + 1, step = 1;
        while (lo + step <= wtop && s_P[lo + step - a] <= limit) {
            lo += step;
            step <<= 1;
        }
        u64 hi = lo + step - 1 < wtop ? lo + step - 1 : wtop;
        while (lo < hi) {
            const u64 mid = (lo + hi + 1) >> 1;
            if (s_P[mid - a] <= limit) lo = mid;
            else hi = mid - 1;
        }
        u64 sum = s_P[lo - a];
        if (lo == wtop && wtop < top) {  // past the window: sum on
            while (lo < top) {
                const u64 l = F[lo] >> 32;
                if (sum + l > limit) break;
                sum += l;
                ++lo;
            }
        }
        e_out = static_cast<u32>(lo);
        tot_out = static_cast<u32>(sum - base);
    };
    for (u32 i = t; i < len; i += NF_B) {
        const u64 sp = a + i;
        const u64 base = s_P[i];
        u32 e, tt;
        pack_from(sp, base, base + cap, sp + cap < m ? sp + cap : m, e, tt);
        s_nx[i] = e;
        s_tot[i] = tt;
    }
    if (t == 0) {
        s_ok = 1;
        u32 hi = 0;
        if (a > 0) {  // entries lie in [a, next(a - 1)]: the pack from a - 1 holds its item and Pl(e) <= cap - len
            const u64 l0 = F[a - 1] >> 32;
            u32 tt;
            const u64 top = a - 1 + cap < m ? a - 1 + cap : m;
            if (top <= a || s_P[1] > cap - l0) hi = static_cast<u32>(a);  // item a does not join a - 1's pack
            else pack_from(a, 0, cap - l0, top, hi, tt);                  // (it does: e >= a + 1)
        }
        s_hi_entry = hi;
    }
    for (u32 i = t; i < NF_T / 32; i += NF_B) s_spec[i] = 0;
    __syncthreads();
    // the speculative chain from the tile start: f(x) = next(x) while it
    // stays in the tile (else x, a fixed point), doubled four times in shared
    // memory (over the window, done with) to f^16; one thread jumps the
    // chain 32 nodes at a time (f^32 = f^16 o f^16) and every thread then
    // marks the nodes between jumps from the levels (node j*32 + l is
    // f^l(jump j): five lookups)
    unsigned short* s_L = reinterpret_cast<unsigned short*>(nf_smem);  // [5][NF_T]
    __shared__ unsigned short s_jump[NF_T / 32 + 1];
    __shared__ u32 s_njump;
    for (u32 i = t; i < NF_T; i += NF_B) {
        u32 f = i;
        if (i < len) {
            const u32 nx = s_nx[i];
            if (nx < end) f = static_cast<u32>(nx - a);
        }
        s_L[i] = static_cast<unsigned short>(f);
    }
    __syncthreads();
    for (int k = 0; k < 4; ++k) {
        const unsigned short* Fk = s_L + k * NF_T;
        unsigned short* Fn = s_L + (k + 1) * NF_T;
        for (u32 i = t; i < NF_T; i += NF_B) Fn[i] = Fk[Fk[i]];
        __syncthreads();
    }
    if (t == 0) {
        const unsigned short* F16 = s_L + 4 * NF_T;
        u32 x = 0, nj = 0;
        for (;;) {
            s_jump[nj++] = static_cast<unsigned short>(x);
            const u32 y = F16[F16[x]];
            if (y == x) break;
            x = y;
        }
        s_njump = nj;
    }
    __syncthreads();
    {
        const u32 nj = s_njump;
        for (u32 q = t; q < nj * 32; q += NF_B) {
            u32 x = s_jump[q >> 5];
            const u32 l = q & 31u;
#pragma unroll
            for (int k = 0; k < 5; ++k)
                if ((l >> k) & 1u) x = s_L[k * NF_T + x];
            if (x < len) atomicOr(&s_spec[x >> 5], 1u << (x & 31));
        }
        if (t == 0) s_h0 = s_jump[nj - 1];  // the chain's last node in the tile (a fixed point)
    }
    __syncthreads();
    // all-convergence: every possible entry e in [a, next(a - 1)] meets the
    // speculative chain inside the tile (a walk from e that leaves the tile
    // first means the exit depends on the entry)
    if (a > 0 && t < 32) {
        const u64 hi_entry = s_hi_entry;
        bool ok = hi_entry < end;
        for (u64 e = a + t; ok && e <= hi_entry; e += 32) {
            u64 y = e;
            while (y < end && !((s_spec[(y - a) >> 5] >> ((y - a) & 31)) & 1u)) y = s_nx[y - a];
            if (y >= end) ok = false;
        }
        if (!__all_sync(0xffffffffu, ok) && t == 0) s_ok = 0;
    }
    __syncthreads();
    const u64 exit_spec = s_nx[s_h0];
    const bool allconv = tile == 0 || s_ok;  // tile 0 is entered at its start
    if (t == 0) {
        if (allconv) st_release_u64(r.xst + tile, kXKnown | exit_spec);
        // entry: the true exit of the tile before
        u64 e = 0;
        if (tile > 0) {
            u64 w;
            while (!((w = ld_acquire_u64(r.xst + tile - 1)) & kXKnown)) {
            }
            e = w & ~kXKnown;
        }
        // walk from the entry until the speculative chain (k_nf_flags)
        for (u32 i = 0; i < NF_T / 32; ++i) s_fl[i] = 0;
        u64 x = e;
        while (x < end && !((s_spec[(x - a) >> 5] >> ((x - a) & 31)) & 1u)) {
            const u32 q = static_cast<u32>(x - a);
            s_fl[q >> 5] |= 1u << (q & 31);
            x = s_nx[q];
        }
        if (!allconv) st_release_u64(r.xst + tile, kXKnown | (x < end ? exit_spec : x));
        s_entry = e;
        s_conv = x;
    }
    __syncthreads();
    // final start flags, frozen totals among the tile's starts, last start
    const u64 conv = s_conv;
    if (t < NF_T / 32) {  // two warps, one flags word each
        const u64 p0 = a + 32ull * t;
        u32 bits = 0;
        if (p0 < end) {
            bits = s_spec[t];
            if (conv >= p0 + 32) bits = 0;
            else if (conv > p0) bits &= ~((1u << (conv - p0)) - 1u);
            bits |= s_fl[t];
            if (end < p0 + 32) bits &= (1u << (end - p0)) - 1u;
        }
        s_fl[t] = bits;
        u64 fe = 0, fp = 0;
        for (u32 b = bits; b; b &= b - 1) {
            const u64 st = p0 + __ffs(b) - 1;
            if (s_tot[st - a] >= r.tmin) {
                fe += s_nx[st - a] - st;
                ++fp;
            }
        }
        const u64 v = warp_sum((fp << 31) | fe);
        u32 lst = bits ? static_cast<u32>(p0) + 32u - __clz(bits) : 0u;  // 1 + last start, absolute
        lst = warp_max(lst);
        if ((t & 31u) == 0) {
            s_tv[t >> 5] = v;
            s_last2[t >> 5] = lst;
        }
    }
    __syncthreads();
    // publish (aggregate, last start), then look back over the tiles before
    if (t == 0) {
        const u64 tv = s_tv[0] + s_tv[1];
        const u32 lst = max(s_last2[0], s_last2[1]);
        const u64 ltot = lst ? s_tot[lst - 1 - a] : 0u;
        st_release_u64(r.lsst + tile, kLsKnown | (ltot << 32) | lst);
        st_release_u64(r.tvst + tile, (tile == 0 ? kTvInc : kTvAgg) | tv);
        u64 excl = 0;
        u32 carry = 0, carry_tot = 0;
        if (tile > 0) {
            for (long long q = static_cast<long long>(tile) - 1;; --q) {
                u64 w;
                while (((w = ld_acquire_u64(r.tvst + q)) >> 62) == 0) {
                }
                excl += w & kTvMask;
                if ((w >> 62) == 2) break;
            }
            for (long long q = static_cast<long long>(tile) - 1; q >= 0 && carry == 0; --q) {
                u64 w;
                while (!((w = ld_acquire_u64(r.lsst + q)) & kLsKnown)) {
                }
                carry = static_cast<u32>(w);
                carry_tot = static_cast<u32>((w >> 32) & 0x7fffffffu);
            }
            st_release_u64(r.tvst + tile, kTvInc | (excl + tv));
        }
        s_tpre = excl;
        s_carry = carry;
        s_carry_tot = carry_tot;
    }
    // the window is done with: the entries go where it was
#pragma unroll
    for (int k = 0; k < EM_ITEMS; ++k) {
        const u32 li = k * NF_B + t;
        if (li < len) s_F[pad(li)] = r.F[a + li];
    }
    __syncthreads();
    // emit (k_nf_emit): every position's pack and the inclusive frozen count
    const u32 p0 = t * EM_ITEMS;
    const u32 bits = (s_fl[p0 >> 5] >> (p0 & 31)) & 0xffu;
    u32 e_of[EM_ITEMS];
    u32 tot_of[EM_ITEMS];
    u64 v = 0;
#pragma unroll
    for (int j = 0; j < EM_ITEMS; ++j) {
        e_of[j] = 0;
        tot_of[j] = 0;
        if ((bits >> j) & 1u) {
            const u64 st = a + p0 + j;
            const u32 e = s_nx[p0 + j];
            const u64 tot = s_tot[p0 + j];
            e_of[j] = e;
            tot_of[j] = static_cast<u32>(tot);
            if (tot >= r.tmin) v += (1ull << 31) | (e - st);
        }
    }
    u64 btot;
    const u64 ex = block_exclusive_scan<u64>(v, s_red, btot);
    const u32 my_last = bits ? static_cast<u32>(a) + p0 + 32u - __clz(bits) : 0u;  // 1 + last own start
    u32 prev = block_exclusive_max(my_last, s_mx);
    const bool carried = prev == 0;
    if (carried) prev = s_carry;
    u64 run = s_tpre + ex;
    u32 e_cur = 0;
    bool frz = false;
    if (!(bits & 1u) && p0 < len) {
        const u64 st = prev - 1;
        // a pack carried in from an earlier tile ends at this tile's entry
        e_cur = carried ? static_cast<u32>(s_entry) : s_nx[st - a];
        frz = static_cast<u64>(carried ? s_carry_tot : s_tot[st - a]) >= r.tmin;
    }
#pragma unroll
    for (int j = 0; j < EM_ITEMS; ++j) {
        const u32 li = p0 + j;
        if (li >= len) break;
        const u64 i = a + li;
        if ((bits >> j) & 1u) {
            e_cur = e_of[j];
            frz = tot_of[j] >= r.tmin;
            if (frz) {
                const u64 q = r.pbase + (run >> 31);
                r.sink.pack_off[q] = r.mbase + (run & kElems);
                r.sink.pack_total[q] = tot_of[j];
                run += (1ull << 31) | (e_cur - i);
            }
        }
        const u64 fz = run & kElems;
        s_dst[pad(li)] = frz ? static_cast<u32>(r.mbase + fz - (e_cur - i)) | kToSink : static_cast<u32>(i - fz);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < EM_ITEMS; ++k) {
        const u32 li = k * NF_B + t;
        if (li < len) {
            const u32 d = s_dst[pad(li)];
            const u64 x = s_F[pad(li)];
            if (d & kToSink) r.sink.members[d & ~kToSink] = x;
            else r.newpool[d] = x;
        }
    }
    if (tile == r.ntiles - 1 && t == 0) {  // totals: pool size and sink counters for the next round
        const u64 tt = s_tpre + btot;
        r.totals[0] = m - (tt & kElems);
        r.totals[1] = r.mbase + (tt & kElems);
        r.totals[2] = r.pbase + (tt >> 31);
        *r.sink.n_members = r.totals[1];
        *r.sink.n_packs = r.totals[2];
    }
}
