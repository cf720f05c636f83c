// chain.cu — first fit as a systolic chain of bins.
//
// First fit (packing.cpp:55-60) puts item j into the lowest-index bin with
// room. Seen from a bin: bin b receives exactly the items that bins 0..b-1
// did not take, in item order, and takes each one that fits its current
// residual. So the bins form a pipeline through which the item sequence
// flows, and bin b's decisions depend only on what reached it. FFD's "open a
// new bin" is the same rule applied to the empty bins after the open ones
// (residual = capacity), and greedy fill (balance.cpp:62-101, in the (length
// desc, id asc) order of first_fit_runs) is the chain without empty bins.
//
// Items travel as runs of equal length: run k with c items still unplaced
// reaches a bin with residual r, which takes min(c, floor(r / s)) of them --
// the lowest ids left -- and passes the rest on. Warp j owns 32 * M
// consecutive bins (lane l holds bins j*32M + l*M + i, i < M, in registers).
// Per block of 32 runs it receives the 32 counts its predecessor left,
// marks the runs its bins can take (c > 0 and s <= its max residual), serves
// those in order and passes the 32 remaining counts on. The serve of the
// frontier warp is on the critical path of every block, so the chain keeps
// it short (see serve) and writes nothing but the input counts of its
// active cells; a replay kernel re-serves those cells in parallel and
// writes the heads (item -> bin, slot). CTAs take their chain position in
// the order they start, so once the chain has filled every resident bin
// works on a different run block at the same time.
//
// Hand-off: each count travels as one 64-bit word (block tag << 32 | count)
// that the consumer lane polls, so no flag or fence sits on the path --
// through shared memory between the warps of a CTA (a ring of kQs blocks;
// consumers publish how many blocks they have read so that producers never
// overwrite an unread slot), through global memory (L2) from the last warp of
// a CTA to the first of the next (a slot per block: a CTA never waits for a
// later one, so the chain needs no co-resident launch). Items are written
// straight to (bin, slot); bin counts give the slots.
#include "stages.cuh"

namespace hbp_b200 {

namespace {

#ifndef HBP_CHAIN_WALK
#define HBP_CHAIN_WALK 3  // lanes walked one by one before a warp scan
#endif
constexpr int kQs = 16;        // shared-memory ring depth (dynamic shared memory)
// warps per CTA (one CTA per SM): fewer for wide lanes so registers stay <= 128
// Warps per CTA. A short chain spreads over the SMs in CTAs of 4 warps
// (fewer warps per SM contend less for issue slots: C2 chain -8% against
// 16); a long one (more warps than 8 per SM) keeps CTAs of 16 so fewer
// hand-offs cross CTAs through L2.
constexpr int kShortWarps = 4;
template <int M>
__host__ __device__ constexpr int warps_for() { return M <= 4 ? 32 : 16; }
// Blocks of run data (and, for a CTA's first warp, of L2 ring words) each
// warp has in flight ahead of the block it serves. A warp whose cells are
// inactive spends only ~100 ns per block, while one L2 round trip is
// ~600 ns: fetched a block ahead, the run data and the ring word set that
// warp's pace -- and, on the C2 128K-group FFD, the whole chain's (704 ns
// per block at the first warp of a CTA, 1046 blocks). CTAs of 32 warps
// keep 4 (their shared memory holds no more).
template <int kWarps>
__host__ __device__ constexpr int prefetch_depth() { return kWarps >= 32 ? 4 : 8; }

struct ChainArgs {
    const u32* run_item;
    const u32* run_len;
    u32 n_items, n_runs, run_begin, run_end;
    u64* leaves;
    u32 live, n_bins, cap;
    u32 bin0, bin_end;     // this pass covers bins [bin0, bin_end)
    const u32* carry_in;   // per run: items the previous pass left (null: first pass)
    u32* carry_out;        // per run: items this pass leaves
    int ffd;
    u32 J, nblocks;
    u32 rb;  // runs per block (lanes 0..rb-1 carry them; 8, 16 or 32)
    unsigned long long* gring;  // CTA g -> g+1: nblocks * 32 tagged counts (every block has its slot)
    u32* cta_ctr;               // CTA ids in launch order (atomic counter)
    u32* item_bin;   // heads only: at the first item of each take
    u32* item_slot;
    u32* take;       // items in the take starting here (0: not a head)
    bool replayed;   // host: the pass ran a replay (heads only: an expand pass follows)
    u32* out;                  // [0] 1 + highest bin with items, [1] FFD overflow
    unsigned long long* prof;  // HBP_TRACE: per warp [wait in, serve, wait out, served runs]
    u32 sleep;                 // ns of back-off per failed poll (idle warps yield issue slots)
    int single;                // a lone run at the FFD frontier: plain first fit over every lane
    u32* hist;                 // [J][nblocks][32] input counts of active cells (chain -> replay)
    u32* hact;                 // [J][nblocks] active-run mask of every cell (0: nothing to serve)
    unsigned long long* tl;    // HBP_CHAIN_TL: globaltimer when block b reached warp j [J][nblocks]
};

// Per-warp prefetch ring (shared memory), filled by cp.async kPF - 1 blocks ahead.
template <int kPF>
struct ChainPF {
    unsigned long long ring[kPF][32];  // first warp of a CTA: the L2 ring words (tag checked on use)
    u32 len[kPF][32];                  // run_len
    u32 beg[kPF][32];                  // run_item (head with carry: carry_in)
    u32 end[kPF][32];                  // run_item of the next run
};

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, u32 src_bytes) {
    const u32 sa = static_cast<u32>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes) : "memory");
}
// 16 bytes through L2 only (.cg): the ring words change under the kernel
__device__ __forceinline__ void cp_async16_cg(void* smem, const void* gmem) {
    const u32 sa = static_cast<u32>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u32 ld_relaxed_u32(const u32* p) {
    u32 v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u32(u32* p, u32 v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Serves one block of 32 runs (counts c, lengths s, item ends end_item; `act`
// marks the runs with c > 0 and s <= wmax) against the warp's 32*M bins, in
// run order, and leaves in c what passes on. STORE writes one head (bin,
// slot, take) at the first item of every take; the chain serves without
// storing (scattered stores would sit on its critical path) and the replay
// re-serves with them.
//
// Per run the critical path is short: the lanes with room are known from
// each lane's max residual (one ballot); every lane computes what its M bins
// can take (independent divisions by a shuffled reciprocal) and their
// in-lane prefix; the run then walks the lanes with room in order -- one
// shuffle per lane, usually one or two lanes -- or, when it spans more,
// one saturating warp scan. The takes themselves (residuals, counts, heads)
// are off the path: every lane applies its own once it knows how many
// items it receives.
// Per-warp staging of a segment's runs for the frontier fill.
struct RunStage {
    unsigned long long incl[32];  // inclusive prefix of the runs' leftovers (run order = lane order)
    u32 s[32];                    // run length
    u32 off[32];                  // first leftover item of the run
};

// Phase cycles of the sequential serve (tools/micro/cell_micro.cu only).
#ifdef HBP_SERVE_PROF
__device__ unsigned long long g_serve_prof[8];
#define SP_BEGIN long long sp_t = clock64()
#define SP_MARK(k)                                   \
    do {                                             \
        const long long _t = clock64();              \
        if (lane == 0) g_serve_prof[k] += _t - sp_t; \
        sp_t = _t;                                   \
    } while (0)
#else
#define SP_BEGIN
#define SP_MARK(k)
#endif

// One run `r` against the lanes in `allowed` (bin order = lane order).
template <int M, int STORE>
__device__ __forceinline__ bool serve_run(const ChainArgs& a, int r, unsigned allowed, u32 s, u32 inv_own,
                                          u32 end_item, u32& c, u32 (&R)[M], u32 (&N)[M], u32& lmax, u64 base,
                                          u32 lane) {
    SP_BEGIN;
    const u32 Sraw = __shfl_sync(0xffffffffu, s, r);
    const u32 S = Sraw & 0x7fffffffu, strict = Sraw >> 31;
    const u32 inv = __shfl_sync(0xffffffffu, inv_own, r);
    const u32 C0 = __shfl_sync(0xffffffffu, c, r);
    u32 off = 0;
    if (STORE) off = __shfl_sync(0xffffffffu, end_item - c, r);
    unsigned room = __ballot_sync(0xffffffffu, lmax >= S + strict) & allowed;
    SP_MARK(0);
    if (!room) return false;
    u32 capl[M], pre[M + 1];
    pre[0] = 0;
#pragma unroll
    for (int i = 0; i < M; ++i) {
        const u32 Re = R[i] > strict ? R[i] - strict : 0u;
        // floor(Re / S): with inv = floor((2^32-1)/S) and Re < 2^31 the
        // estimate is low by at most one, so one correction is exact
        u32 q = __umulhi(Re, inv);
        q += (Re - q * S >= S) ? 1u : 0u;
        capl[i] = min(q, C0);  // no bin takes more than the run has
        pre[i + 1] = min(pre[i] + capl[i], C0);  // (a log-depth tree measured 3% slower)
    }
    const u32 lsum = pre[M];
    SP_MARK(1);
    // walk the lanes with room in bin order
    u32 left = C0, mine = 0;
    for (int k = 0; k < HBP_CHAIN_WALK && left > 0 && room; ++k) {
        const int f = __ffs(room) - 1;
        room &= room - 1;
        const u32 lf = __shfl_sync(0xffffffffu, lsum, f);
        if (static_cast<int>(lane) == f) mine = left;
        left -= min(lf, left);
    }
    if (left > 0 && room) {  // spans many lanes: one scan over the rest
        const u32 v = (room >> lane) & 1u ? lsum : 0u;
        u32 incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= static_cast<u32>(o)) incl = min(incl + t, left);
        }
        u32 excl = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) excl = 0;
        if (v > 0 && excl < left) mine = left - excl;
        left -= __shfl_sync(0xffffffffu, incl, 31);
    }
    if (static_cast<int>(lane) == r) c = left;
    SP_MARK(2);
    if (mine > 0) {  // this lane receives `mine` items of the run
        u32 nl = 0;
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const u32 t = pre[i] < mine ? min(capl[i], mine - pre[i]) : 0u;
            if (STORE && t > 0) {
                const u32 o = off + (C0 - mine) + pre[i];
                const u32 bin = static_cast<u32>(base + lane * M + i);
                a.take[o] = t;
                if (STORE == 2) {  // a chain without replay: every item (no expand pass after it)
                    for (u32 k = 0; k < t; ++k) {
                        a.item_bin[o + k] = bin;
                        a.item_slot[o + k] = N[i] + k;
                    }
                } else {
                    a.item_bin[o] = bin;
                    a.item_slot[o] = N[i];
                }
            }
            R[i] -= t * S;
            N[i] += t;
            nl = max(nl, R[i]);
        }
        lmax = nl;
    }
    SP_MARK(3);
    return true;
}

// Serves the runs of `act` against the lanes of `allowed` in run order, one
// at a time; after every take the runs that no longer fit any allowed lane
// are dropped (one reduce + one ballot) instead of each paying a serve that
// finds no room -- most active runs of greedy fill and of FFD's later
// blocks (measured on C2: 19% / 35% of the active runs take anything).
// Measured and dropped (tools/micro/cell_micro.cu on real C2 cells): a
// wavefront over the lanes (1.4x faster where every run takes, 1.3-3x
// slower elsewhere), a lane-by-lane serve without the warp prefix, a lazy
// filter, and row-major bins.
template <int M, int STORE>
__device__ __forceinline__ void serve_set(const ChainArgs& a, unsigned act, unsigned allowed, u32 s, u32 s_eff,
                                          u32 inv_own, u32 end_item, u32& c, u32 (&R)[M], u32 (&N)[M], u32& lmax,
                                          u64 base, u32 lane) {
    const bool ok = (allowed >> lane) & 1u;
    while (act) {
        const int r = __ffs(act) - 1;
        act &= act - 1;
        if (serve_run<M, STORE>(a, r, allowed, s, inv_own, end_item, c, R, N, lmax, base, lane) && act) {
            SP_BEGIN;
            act &= __ballot_sync(0xffffffffu, s_eff <= __reduce_max_sync(0xffffffffu, ok ? lmax : 0u));
            SP_MARK(4);
        }
    }
}

// FFD frontier in closed form. The runs of `seg` share k = floor(cap / s):
// their items lie in (cap / (k + 1), cap / k], so k of them always share a
// bin and k + 1 never do, and no item of the segment fits a bin that k of
// them filled. Their leftovers (what the warp's non-empty bins left) thus
// fill the empty bins in order, k items per bin, the last bin partially --
// exactly what serving them one by one would do -- with one warp scan.
template <int M, int STORE>
__device__ __forceinline__ void frontier_fill(const ChainArgs& a, unsigned seg, u32 k, u32 s, u32 end_item, u32& c,
                                              u32 (&R)[M], u32 (&N)[M], u32& lmax, u32& emask, RunStage& st,
                                              u64 base, u32 lane) {
    const u32 lv = (seg >> lane) & 1u ? c : 0u;
    if (!__any_sync(0xffffffffu, lv > 0)) return;  // the non-empty lanes took every item
    unsigned long long incl = lv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= static_cast<u32>(o)) incl += t;
    }
    const unsigned long long T = __shfl_sync(0xffffffffu, incl, 31);
    if (T == 0) return;
    const int e0 = __ffs(emask) - 1;
    const int e1 = 32 - __clz(emask);
    const unsigned long long per = static_cast<unsigned long long>(M) * k;
    const unsigned long long used = min(T, static_cast<unsigned long long>(e1 - e0) * per);
    st.incl[lane] = incl;
    st.s[lane] = s & 0x7fffffffu;
    st.off[lane] = end_item - c;
    __syncwarp();
    if (static_cast<int>(lane) >= e0 && static_cast<int>(lane) < e1) {
        const unsigned long long pos0 = static_cast<unsigned long long>(lane - e0) * per;
        if (pos0 < used) {
            int q = 0;
            while (st.incl[q] <= pos0) ++q;
            u32 nl = 0;
#pragma unroll
            for (int i = 0; i < M; ++i) {
                const unsigned long long b0 = pos0 + static_cast<unsigned long long>(i) * k;
                if (b0 < used) {
                    const unsigned long long b1 = min(b0 + k, used);
                    u32 tot = 0, nb = 0;
                    for (unsigned long long p = b0; p < b1;) {
                        while (st.incl[q] <= p) ++q;
                        const unsigned long long hi = min(b1, st.incl[q]);
                        const u32 t = static_cast<u32>(hi - p);
                        if (STORE) {
                            const unsigned long long ex_q = q ? st.incl[q - 1] : 0ull;
                            const u32 o = st.off[q] + static_cast<u32>(p - ex_q);
                            const u32 bin = static_cast<u32>(base + lane * M + i);
                            a.take[o] = t;
                            if (STORE == 2) {
                                for (u32 k = 0; k < t; ++k) {
                                    a.item_bin[o + k] = bin;
                                    a.item_slot[o + k] = nb + k;
                                }
                            } else {
                                a.item_bin[o] = bin;
                                a.item_slot[o] = nb;
                            }
                        }
                        tot += t * st.s[q];
                        nb += t;
                        p = hi;
                    }
                    R[i] = a.cap - tot;
                    N[i] = nb;
                }
                nl = max(nl, R[i]);
            }
            lmax = nl;
        }
    }
    __syncwarp();
    if (lv > 0) {
        const unsigned long long ex = incl - lv;
        const unsigned long long hi = min(incl, used);
        if (hi > ex) c -= static_cast<u32>(hi - ex);
    }
    const unsigned long long touched = (used + per - 1) / per;  // lanes no longer empty
    const int e0n = e0 + static_cast<int>(touched);
    emask = e0n >= 32 ? 0u : (emask & ~((1u << e0n) - 1u));
}

// Serves one block of 32 runs (counts c, lengths s, item ends end_item; `act`
// marks the runs with c > 0 and s <= wmax) against the warp's 32*M bins, in
// run order, and leaves in c what passes on. STORE writes one head (bin,
// slot, take) at the first item of every take; the chain serves without
// storing (scattered stores would sit on its critical path) and the replay
// re-serves with them.
//
// Per run the critical path is short: the lanes with room are known from
// each lane's max residual (one ballot); every lane computes what its M bins
// can take (independent divisions by a shuffled reciprocal) and their
// in-lane prefix; the run then walks the lanes with room in order -- one
// shuffle per lane, usually one or two lanes -- or, when it spans more,
// one saturating warp scan. The takes themselves (residuals, counts, heads)
// are off the path: every lane applies its own once it knows how many
// items it receives. At the FFD frontier (lanes whose bins are all still
// empty, emask) the runs of a block that share k = floor(cap / s) are served
// against the non-empty lanes one by one and then fill the empty ones
// together in closed form (frontier_fill).
template <int M, int STORE>
__device__ __forceinline__ void serve(const ChainArgs& a, u32 act, u32 s, u32 end_item, u32& c, u32 (&R)[M],
                                      u32 (&N)[M], u32& wmax, u32& emask, RunStage& st, u64 base, u32 lane) {
    // run_len bit 31: strict run (ids <= -2 in greedy fill, stages.cuh):
    // a bin takes floor((r - 1) / s) of its items
    const u32 s_own = s & 0x7fffffffu;
    const u32 inv_own = s_own ? 0xffffffffu / s_own : 0u;
    u32 lmax = 0;
#pragma unroll
    for (int i = 0; i < M; ++i) lmax = max(lmax, R[i]);
    u32 k_own = 0;
    if (emask && s_own) {
        k_own = __umulhi(a.cap, inv_own);
        k_own += (a.cap - k_own * s_own >= s_own) ? 1u : 0u;
    }
    // A run is active when s <= the warp's max residual at the block's
    // arrival; every take lowers residuals, so after one the runs that no
    // longer fit anywhere are dropped at once (one reduce + one ballot) instead
    // of each paying a serve that finds no room (most active runs of greedy
    // fill and of FFD's later blocks, measured on C2).
    const u32 s_eff = s_own + (s >> 31);
    while (act) {
        const int r = __ffs(act) - 1;
        if (!emask) {
            serve_set<M, STORE>(a, act, 0xffffffffu, s, s_eff, inv_own, end_item, c, R, N, lmax, base, lane);
            break;
        }
        const u32 kr = __shfl_sync(0xffffffffu, k_own, r);
        // the segment: consecutive active runs from r with the same k (runs
        // out of the block's active set are transparent); FFD's sorted runs
        // keep each k contiguous, a shuffled order (FFS) may not
        const unsigned same = __ballot_sync(0xffffffffu, k_own == kr) | ~act;
        const unsigned breaks = ~same & ~((2u << r) - 1u);
        const unsigned upto = breaks ? (1u << (__ffs(breaks) - 1)) - 1u : 0xffffffffu;
        const unsigned seg = act & upto;
        act &= ~seg;
        if (a.single && (seg & (seg - 1u)) == 0u) {
            // One run: the empty lanes follow the non-empty ones in bin
            // order, so first fit over every lane is exactly the non-empty
            // serve followed by the frontier fill; no scan, no staging. A
            // lane that received items had its first bin take them.
            serve_set<M, STORE>(a, seg, 0xffffffffu, s, s_eff, inv_own, end_item, c, R, N, lmax, base, lane);
            emask &= __ballot_sync(0xffffffffu, N[0] == 0u);
            continue;
        }
        // against the non-empty lanes only the runs that fit one of them
        const bool ne_lane = ((emask >> lane) & 1u) == 0;
        const unsigned q = seg & __ballot_sync(0xffffffffu, s_eff <= __reduce_max_sync(0xffffffffu, ne_lane ? lmax : 0u));
        serve_set<M, STORE>(a, q, ~emask, s, s_eff, inv_own, end_item, c, R, N, lmax, base, lane);
        frontier_fill<M, STORE>(a, seg, kr, s, end_item, c, R, N, lmax, emask, st, base, lane);
    }
    wmax = __reduce_max_sync(0xffffffffu, lmax);
}

// Lanes whose M bins are all fresh FFD bins (empty, inside the pass); none
// in a warp that reaches past the pass's last bin.
template <int M>
__device__ __forceinline__ u32 empty_lanes(const ChainArgs& a, u64 base, u32 lane) {
    if (!a.ffd || base + 32ull * M > a.bin_end) return 0u;
    bool e = true;
#pragma unroll
    for (int i = 0; i < M; ++i) e = e && (base + lane * M + i) >= a.live;
    return __ballot_sync(0xffffffffu, e);
}

// Loads the warp's 32*M bins (lane-major) from the leaves; empty bins past
// `live` open at capacity under FFD.
template <int M>
__device__ __forceinline__ u32 load_bins(const ChainArgs& a, u64 base, u32 lane, u32 (&R)[M], u32 (&N)[M]) {
    u32 lmax = 0;
#pragma unroll
    for (int i = 0; i < M; ++i) {
        const u64 bin = base + lane * M + i;
        u64 leaf = 0;
        if (bin < a.bin_end) {
            if (bin < a.live) leaf = a.leaves[bin];
            else if (a.ffd) leaf = static_cast<u64>(a.cap) << 32;  // empty bin
        }
        R[i] = static_cast<u32>(leaf >> 32);
        N[i] = static_cast<u32>(leaf);
        lmax = max(lmax, R[i]);
    }
    return __reduce_max_sync(0xffffffffu, lmax);
}

// 1 + the highest bin of the warp holding items (0: none); with `write`,
// stores the bins back to the leaves.
template <int M>
__device__ __forceinline__ u32 store_bins(const ChainArgs& a, u64 base, u32 lane, const u32 (&R)[M],
                                          const u32 (&N)[M], bool write) {
    u32 top = 0;
#pragma unroll
    for (int i = 0; i < M; ++i) {
        const u64 bin = base + lane * M + i;
        if (bin < a.bin_end) {
            if (write && (bin < a.live || N[i] > 0)) a.leaves[bin] = (static_cast<u64>(R[i]) << 32) | N[i];
            if (N[i] > 0) top = static_cast<u32>(bin + 1);
        }
    }
    return __reduce_max_sync(0xffffffffu, top);
}

// TRACE compiles in the per-warp counters and the per-cell timeline
// (HBP_TRACE); the product kernel keeps its per-block path short: a warp
// whose cell is inactive only forwards the counts (~40 instructions).
template <int M, int kWarps, bool TRACE>
__global__ void __launch_bounds__(kWarps * 32, 1) k_ff_chain(ChainArgs a) {
    // [kWarps][kQs][32]: warp w-1 -> w, then RunStage[kWarps], then ChainPF[kWarps]
    extern __shared__ __align__(16) unsigned long long s_ring_raw[];
    auto s_ring = reinterpret_cast<unsigned long long (*)[kQs][32]>(s_ring_raw);
    RunStage* s_stage = reinterpret_cast<RunStage*>(s_ring_raw + kWarps * kQs * 32);
    constexpr int kPF = prefetch_depth<kWarps>();
    ChainPF<kPF>* s_pf = reinterpret_cast<ChainPF<kPF>*>(s_stage + kWarps);
    __shared__ u32 s_cons[kWarps];                         // blocks warp w has read from s_ring[w]
    __shared__ u32 s_g;
    const u32 w = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    // CTA ids in the order CTAs start: CTA g only ever waits on CTA g - 1,
    // which started before it, and the L2 links hold every block (no
    // back-pressure between CTAs), so the chain needs no co-residency -- no
    // cooperative launch, and chains on other streams run alongside
    if (threadIdx.x == 0) s_g = atomicAdd(a.cta_ctr, 1u);
    for (u32 i = threadIdx.x; i < kWarps * kQs * 32; i += blockDim.x) (&s_ring[0][0][0])[i] = 0ull;
    if (threadIdx.x < kWarps) s_cons[threadIdx.x] = 0;
    __syncthreads();
    const u32 g = s_g;
    const u32 j = g * kWarps + w;
    if (j >= a.J) return;  // no CTA-wide barriers below

    // lane-major: lane l holds bins base + l*M + i (bin order = lane order)
    const u64 base = a.bin0 + static_cast<u64>(j) * 32 * M;
    u32 R[M], N[M];
    u32 wmax = load_bins<M>(a, base, lane, R, N);
    u32 emask = empty_lanes<M>(a, base, lane);
    const u32 nblocks = a.nblocks, rb = a.rb, run_begin = a.run_begin, run_end = a.run_end, n_runs = a.n_runs;
    const bool head = j == 0, tail = j + 1 == a.J;
    const bool in_global = w == 0, out_global = w + 1 == kWarps;
    const bool replay = a.hist != nullptr;
    volatile unsigned long long* sin = s_ring[w][0];
    volatile unsigned long long* sout = w + 1 < kWarps ? s_ring[w + 1][0] : nullptr;
    const unsigned long long* gin = a.gring + static_cast<u64>(g) * a.nblocks * 32;  // written by CTA g-1
    unsigned long long* gout = a.gring + static_cast<u64>(g + 1) * a.nblocks * 32;
    volatile u32* const my_scons = reinterpret_cast<volatile u32*>(s_cons) + w;
    volatile u32* const next_scons = reinterpret_cast<volatile u32*>(s_cons) + (w + 1 < kWarps ? w + 1 : w);
    u32 seen_cons = 0;  // consumer progress known to this producer

    // run data of blocks b .. b + kPF - 2 (and the first warp's L2 ring
    // words) in flight while block b is served; one cp.async group per
    // block. The chain needs run lengths only; the first warp (counts) and
    // chains that store their heads themselves (item offsets) also the
    // item bounds.
    ChainPF<kPF>& pf = s_pf[w];
    const bool carry_head = head && a.carry_in != nullptr;
    const bool want_items = head || !replay;
    const u32* const run_len = a.run_len;
    const u32* const run_item = a.run_item;
    auto prefetch = [&](u32 bb) {
        const int slot = static_cast<int>(bb % kPF);
        const u32 k = run_begin + bb * rb + lane;
        const bool valid = bb < nblocks && lane < rb && k < run_end;
        cp_async4(&pf.len[slot][lane], valid ? run_len + k : run_len, valid ? 4u : 0u);
        if (want_items) {
            cp_async4(&pf.beg[slot][lane], valid ? (carry_head ? a.carry_in + k : run_item + k) : run_item,
                      valid ? 4u : 0u);
            const bool ve = valid && k + 1 < n_runs;
            cp_async4(&pf.end[slot][lane], ve ? run_item + k + 1 : run_item, ve ? 4u : 0u);
        }
        if (in_global && !head && bb < nblocks && lane < 16)
            cp_async16_cg(&pf.ring[slot][2 * lane], gin + static_cast<u64>(bb) * 32 + 2 * lane);
        cp_async_commit();
    };
#pragma unroll 1
    for (u32 bb = 0; bb + 1 < static_cast<u32>(kPF); ++bb) prefetch(bb);

    unsigned long long pcnt[4] = {0, 0, 0, 0};
    long long t0 = 0, t1 = 0;
#pragma unroll 1
    for (u32 b = 0; b < nblocks; ++b) {
        if (TRACE && a.prof) t0 = clock64();
        __syncwarp();  // every lane is done with the slot the next prefetch refills
        prefetch(b + kPF - 1);
        cp_async_wait<kPF - 1>();
        __syncwarp();
        const int slot = static_cast<int>(b % kPF);
        const u32 s = pf.len[slot][lane];
        u32 c;
        if (head) {
            const u32 kr = run_begin + b * rb + lane;
            const bool valid = lane < rb && kr < run_end;
            const u32 e = valid ? (kr + 1 < n_runs ? pf.end[slot][lane] : a.n_items) : 0u;
            c = carry_head ? pf.beg[slot][lane] : e - pf.beg[slot][lane];
        } else if (in_global) {
            unsigned long long v = pf.ring[slot][lane];
            if ((v >> 32) != (b + 1))
                while (((v = ld_relaxed_u64(gin + static_cast<u64>(b) * 32 + lane)) >> 32) != (b + 1))
                    if (a.sleep) __nanosleep(a.sleep);
            c = static_cast<u32>(v);
        } else {
            unsigned long long v;
            while (((v = sin[(b % kQs) * 32 + lane]) >> 32) != (b + 1))
                if (a.sleep) __nanosleep(a.sleep);
            c = static_cast<u32>(v);
        }
        // every lane has its c; run_len bit 31 = strict (needs r > s)
        const unsigned act = __ballot_sync(0xffffffffu, c > 0 && (s & 0x7fffffffu) + (s >> 31) <= wmax);
        unsigned long long t_arr = 0;
        if (TRACE) {
            if (a.tl) t_arr = globaltimer();
            if (a.prof) {
                t1 = clock64();
                pcnt[0] += t1 - t0;
                pcnt[3] += __popc(act);
                t0 = t1;
            }
        }
        if (!head && !in_global && lane == 0) *my_scons = b + 1;
        if (act) {  // (the replay's hact is zeroed: inactive cells write nothing)
            const u32 kr = run_begin + b * rb + lane;
            const bool valid = lane < rb && kr < run_end;
            if (replay) {  // the replay re-serves this cell from its input counts
                if (lane < rb) a.hist[(static_cast<u64>(j) * nblocks + b) * rb + lane] = c;
                if (lane == 0) a.hact[static_cast<u64>(j) * nblocks + b] = act;
                serve<M, 0>(a, act, s, 0u, c, R, N, wmax, emask, s_stage[w], base, lane);
            } else {  // short chains store their heads directly
                const u32 end_item = valid ? (kr + 1 < n_runs ? pf.end[slot][lane] : a.n_items) : 0u;
                serve<M, 2>(a, act, s, end_item, c, R, N, wmax, emask, s_stage[w], base, lane);  // every item
            }
        }
        unsigned long long t_srv = 0;
        if (TRACE) {
            if (a.tl) t_srv = globaltimer();
            if (a.prof) {
                t1 = clock64();
                pcnt[1] += t1 - t0;
                t0 = t1;
            }
        }
        if (!tail) {
            const unsigned long long v = (static_cast<unsigned long long>(b + 1) << 32) | c;
            if (out_global) {
                st_relaxed_u64(gout + static_cast<u64>(b) * 32 + lane, v);
            } else {
                if (b >= static_cast<u32>(kQs) && seen_cons + kQs <= b) {
                    if (lane == 0)
                        while ((seen_cons = *next_scons) + kQs <= b)
                            if (a.sleep) __nanosleep(a.sleep);
                    seen_cons = __shfl_sync(0xffffffffu, seen_cons, 0);
                }
                sout[(b % kQs) * 32 + lane] = v;
            }
        } else {  // tail: hand the counts to the next pass
            const u32 k = run_begin + b * rb + lane;
            if (lane < rb && k < run_end) a.carry_out[k] = c;
            if (__any_sync(0xffffffffu, c > 0) && lane == 0) atomicOr(a.out + 1, 1u);
        }
        if (TRACE) {
            if (a.prof) pcnt[2] += clock64() - t0;
            if (a.tl && lane == 0) {  // arrival | serve ns << 40 | active runs << 56 (timeline)
                const unsigned long long d = min(t_srv - t_arr, (1ull << 16) - 1);
                a.tl[static_cast<u64>(j) * nblocks + b] =
                    (t_arr & ((1ull << 40) - 1)) | (d << 40) | (static_cast<unsigned long long>(__popc(act)) << 56);
            }
        }
    }
    if (TRACE && a.prof && lane == 0)
        for (int i = 0; i < 4; ++i) a.prof[4ull * j + i] = pcnt[i];
    // with a replay to follow, the bins stay as loaded for it
    const u32 top = store_bins<M>(a, base, lane, R, N, !replay);
    if (lane == 0 && top) atomicMax(a.out, top);
}

// Replay of a chain pass: every warp re-serves, from the input counts the
// chain recorded, the cells where runs were active, now writing the heads.
// Warps are independent here, so the scattered head stores run in parallel
// across the GPU instead of on the chain's critical path.
template <int M>
__global__ void __launch_bounds__(256) k_ff_replay(ChainArgs a) {
    const u32 lane = threadIdx.x & 31u;
    const u32 j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (j >= a.J) return;
    __shared__ RunStage s_stage[8];
    const u64 base = a.bin0 + static_cast<u64>(j) * 32 * M;
    u32 R[M], N[M];
    u32 wmax = load_bins<M>(a, base, lane, R, N);
    u32 emask = empty_lanes<M>(a, base, lane);
    for (u32 b = 0; b < a.nblocks; ++b) {
        const u32 act = a.hact[static_cast<u64>(j) * a.nblocks + b];
        if (!act) continue;
        const u32 k = a.run_begin + b * a.rb + lane;
        const bool valid = lane < a.rb && k < a.run_end;
        const u32 s = valid ? a.run_len[k] : 0u;
        const u32 end_item = valid ? (k + 1 < a.n_runs ? a.run_item[k + 1] : a.n_items) : 0u;
        u32 c = valid ? a.hist[(static_cast<u64>(j) * a.nblocks + b) * a.rb + lane] : 0u;
        serve<M, 1>(a, act, s, end_item, c, R, N, wmax, emask, s_stage[threadIdx.x >> 5], base, lane);  // heads
    }
    store_bins<M>(a, base, lane, R, N, true);
}

// Bins one resident chain of width M can hold (per device, queried once).
template <int M, int kWarps = warps_for<M>()>
u64 chain_capacity(int sms) {
    const size_t smem = sizeof(unsigned long long) * kWarps * kQs * 32 + (sizeof(RunStage) + sizeof(ChainPF<prefetch_depth<kWarps>()>)) * kWarps;
    static std::mutex mu;
    static std::map<int, int> per_sm_of;
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    auto it = per_sm_of.find(dev);
    if (it == per_sm_of.end()) {
        CUDA_CHECK(cudaFuncSetAttribute(k_ff_chain<M, kWarps, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
        CUDA_CHECK(cudaFuncSetAttribute(k_ff_chain<M, kWarps, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
        int per_sm = 0;
        CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ff_chain<M, kWarps, false>, kWarps * 32, smem));
        it = per_sm_of.emplace(dev, per_sm).first;
    }
    return static_cast<u64>(it->second > 0 ? it->second : 0) * sms * kWarps * 32 * M;
}

// One pass over bins [a.bin0, a.bin_end); returns {1 + highest bin used, any carry}.
template <int M>
std::pair<u32, bool> run_pass(Ctx& c, ChainArgs& a, const char* name) {
    const u64 pass_bins = a.bin_end - a.bin0;
    const u32 J = static_cast<u32>((pass_bins + 32ull * M - 1) / (32ull * M));
    int sms = 0, dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const bool short_chain = J <= 2u * kShortWarps * static_cast<u32>(sms) &&
                             chain_capacity<M, kShortWarps>(sms) >= pass_bins;
    const int kWarps = short_chain ? kShortWarps : warps_for<M>();
    const u32 G = (J + kWarps - 1) / kWarps;
    const size_t smem = sizeof(unsigned long long) * kWarps * kQs * 32 +
                        (sizeof(RunStage) + (short_chain ? sizeof(ChainPF<prefetch_depth<kShortWarps>()>)
                                                         : sizeof(ChainPF<prefetch_depth<warps_for<M>()>()>))) *
                            kWarps;
    if (short_chain) (void)chain_capacity<M, kShortWarps>(sms);  // attribute set
    else (void)chain_capacity<M>(sms);
    cudaStream_t s = c.stream;
    a.J = J;
    DevBuf<unsigned long long> gring(static_cast<size_t>(G + 1) * a.nblocks * 32, s);
    DevBuf<u32> out(4, s);  // [0] top, [1] overflow, [2] CTA id counter
    gring.zero();
    out.zero();
    a.gring = gring.p;
    a.out = out.p;
    a.cta_ctr = out.p + 2;
    DevBuf<unsigned long long> prof, tl;
    a.prof = nullptr;
    a.tl = nullptr;
    if (c.trace) {
        prof.alloc(4ull * J, s);
        prof.zero();
        a.prof = prof.p;
        if (std::getenv("HBP_CHAIN_TL")) {
            tl.alloc(static_cast<size_t>(J) * a.nblocks, s);
            tl.zero();
            a.tl = tl.p;
        }
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c.trace) {
        CUDA_CHECK(cudaEventCreate(&e0));
        CUDA_CHECK(cudaEventCreate(&e1));
        CUDA_CHECK(cudaEventRecord(e0, s));
    }
    // the chain serves without head stores and records the input counts of
    // its active cells; the replay then writes the heads in parallel
    // A short chain's critical path is its blocks walking a few warps, and a
    // replay would repeat that walk warp by warp: short chains store the
    // heads themselves. Long chains (the head stores on every warp's
    // critical path) hand them to the parallel replay.
    const char* er = std::getenv("HBP_CHAIN_REPLAY_MIN");
    const u32 replay_min = er ? static_cast<u32>(std::atoi(er)) : 64u;
    const bool replay = J >= replay_min && std::getenv("HBP_CHAIN_NOREPLAY") == nullptr;
    DevBuf<u32> hist, hact;
    a.hist = a.hact = nullptr;
    if (replay) {
        hist.alloc(static_cast<size_t>(J) * a.nblocks * a.rb, s);
        hact.alloc(static_cast<size_t>(J) * a.nblocks, s);
        hact.zero();  // the chain writes the active cells only
        a.hist = hist.p;
        a.hact = hact.p;
    }
    a.replayed = replay;
    // algorithmic bytes (FFD residue): 12 B per item + 12 B per bin of the pass
    const double alg = 12.0 * a.n_items + 12.0 * (a.bin_end - a.bin0);
    static const bool coop = std::getenv("HBP_CHAIN_COOP") != nullptr;  // A/B: co-resident launch
    if (coop) {
        void* args[] = {&a};
        if (short_chain) LAUNCH_COOP(name, alg, (k_ff_chain<M, kShortWarps, false>), dim3(G), dim3(kWarps * 32), smem, s, args);
        else LAUNCH_COOP(name, alg, (k_ff_chain<M, warps_for<M>(), false>), dim3(G), dim3(kWarps * 32), smem, s, args);
    } else if (c.trace) {
        if (short_chain) LAUNCH_B(name, alg, (k_ff_chain<M, kShortWarps, true>), G, kWarps * 32, smem, s, a);
        else LAUNCH_B(name, alg, (k_ff_chain<M, warps_for<M>(), true>), G, kWarps * 32, smem, s, a);
    } else {
        if (short_chain) LAUNCH_B(name, alg, (k_ff_chain<M, kShortWarps, false>), G, kWarps * 32, smem, s, a);
        else LAUNCH_B(name, alg, (k_ff_chain<M, warps_for<M>(), false>), G, kWarps * 32, smem, s, a);
    }
    if (c.trace) CUDA_CHECK(cudaEventRecord(e1, s));
    if (replay) LAUNCH_B("fit.replay", 12.0 * a.n_items + 16.0 * (a.bin_end - a.bin0), k_ff_replay<M>, (J + 7) / 8, 256, 0, s, a);
    const auto o = read_vector(c, out.p, 2);
    if (c.trace) {
        float ms = 0;
        CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        std::fprintf(stderr,
                     "[hbp trace] fit chain %s: runs %u..%u (%u blocks) bins %u..%u (live %u) M %d warps %u ctas %u "
                     "used %u carry %u: %.3f ms\n",
                     a.ffd ? "ffd" : "fill", a.run_begin, a.run_end, a.nblocks, a.bin0, a.bin_end, a.live, M, J, G,
                     o[0], o[1], ms);
        const auto pf = read_vector(c, prof.p, 4ull * J);
        if (const char* tlf = std::getenv("HBP_CHAIN_TL")) {  // [J, nblocks, ffd, M] + timeline, appended
            const auto tv = read_vector(c, tl.p, static_cast<size_t>(J) * a.nblocks);
            if (FILE* f = std::fopen(tlf, "ab")) {
                const u32 hdr[4] = {J, a.nblocks, static_cast<u32>(a.ffd), static_cast<u32>(M)};
                std::fwrite(hdr, 4, 4, f);
                std::fwrite(tv.data(), 8, tv.size(), f);
                std::fclose(f);
            }
        }
        if (const char* dump = std::getenv("HBP_CHAIN_DUMP")) {  // per-warp counters, appended
            if (FILE* f = std::fopen(dump, "ab")) {
                const u32 hdr[4] = {J, a.nblocks, static_cast<u32>(M), static_cast<u32>(a.ffd)};
                std::fwrite(hdr, 4, 4, f);
                std::fwrite(pf.data(), 8, pf.size(), f);
                std::fclose(f);
            }
        }
        double sum[4] = {0, 0, 0, 0}, mx[4] = {0, 0, 0, 0};
        u32 arg[4] = {0, 0, 0, 0};
        for (u32 jj = 0; jj < J; ++jj)
            for (int i = 0; i < 4; ++i) {
                const double v = static_cast<double>(pf[4ull * jj + i]);
                sum[i] += v;
                if (v > mx[i]) {
                    mx[i] = v;
                    arg[i] = jj;
                }
            }
        std::fprintf(stderr,
                     "[hbp trace]   per warp: wait-in avg %.2fM max %.2fM | serve avg %.3fM max %.2fM (warp %u) | "
                     "wait-out avg %.3fM max %.2fM | served runs %.0f, max %.0f (warp %u)\n",
                     sum[0] / J / 1e6, mx[0] / 1e6, sum[1] / J / 1e6, mx[1] / 1e6, arg[1], sum[2] / J / 1e6,
                     mx[2] / 1e6, sum[3], mx[3], arg[3]);
    }
    a.out = nullptr;
    return {o[0], o[1] != 0};
}

}  // namespace

// Heads -> every item: item x belongs to the last head h <= x when
// x < h + take[h] (same bin, slot + x - h), else it stays unassigned.
__global__ void k_expand_heads(const u32* __restrict__ take, const u32* __restrict__ q, const u32* __restrict__ pos,
                               u64 n, u32* __restrict__ item_bin, u32* __restrict__ item_slot) {
    // four items per thread, each level of the lookups issued for all four
    // before the next (heads already hold (bin, slot) and are not written)
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 x0 = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; x0 < n; x0 += 4 * stride) {
        u32 k[4], h[4], t[4], b[4], sl[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const u64 x = x0 + u * stride;
            k[u] = x < n && !take[x] ? q[x] : kNone;  // kNone: head or past the end
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) h[u] = k[u] != kNone && k[u] > 0 ? pos[k[u] - 1] : kNone;
#pragma unroll
        for (int u = 0; u < 4; ++u) t[u] = h[u] != kNone ? take[h[u]] : 0u;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const u64 x = x0 + u * stride;
            const bool in = h[u] != kNone && x - h[u] < t[u];
            b[u] = in ? item_bin[h[u]] : kNone;
            sl[u] = in ? item_slot[h[u]] + static_cast<u32>(x - h[u]) : kNone;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (k[u] == kNone) continue;
            item_bin[x0 + u * stride] = b[u];
            item_slot[x0 + u * stride] = sl[u];
        }
    }
}

void expand_heads(Ctx& c, u64 n, u32* item_bin, u32* item_slot, const u32* take) {
    cudaStream_t s = c.stream;
    DevBuf<u32> q(n, s), pos(n, s);
    u32* qp = q.p;
    u32* pp = pos.p;
    // the scan's store also records each head's position (no separate pass)
    scan_exclusive_v<u32>(
        static_cast<i64>(n), [=] __device__(i64 x) { return take[x] ? 1u : 0u; },
        [=] __device__(i64 x, u32 v, u32 h) {
            qp[x] = v + h;
            if (h) pp[v] = static_cast<u32>(x);
        },
        s, c.scan, "scan.chain1", 12.0);
    LAUNCH_B("chain.expand", 24.0 * n, k_expand_heads, grid_for(n, 256), 256, 0, s, take, q.p, pos.p, n, item_bin,
             item_slot);
}

bool chain_fit(Ctx& c, const ChainRuns& runs, u64* leaves, u32 live, u32 n_bins, u32 cap, bool ffd, u32* item_bin,
               u32* item_slot, u32* take, u32 first_pass_bins, u32& used, bool expand) {
    used = live;
    if (runs.run_begin >= runs.run_end || n_bins == 0) {
        if (expand) expand_heads(c, runs.n_items, item_bin, item_slot, take);
        return true;
    }
    cudaStream_t s = c.stream;
    if (c.trace) {
        if (const char* rf = std::getenv("HBP_CHAIN_RUNS")) {  // the chain's input, appended (analysis tools)
            const auto rl = read_vector(c, runs.run_len, runs.n_runs);
            const auto ri = read_vector(c, runs.run_item, runs.n_runs);
            const auto lv = read_vector(c, leaves, live);
            if (FILE* f = std::fopen(rf, "ab")) {
                const u32 hdr[8] = {runs.n_runs, runs.n_items, live, n_bins, cap, static_cast<u32>(ffd),
                                    runs.run_begin, runs.run_end};
                std::fwrite(hdr, 4, 8, f);
                std::fwrite(rl.data(), 4, rl.size(), f);
                std::fwrite(ri.data(), 4, ri.size(), f);
                std::fwrite(lv.data(), 8, lv.size(), f);
                std::fclose(f);
            }
        }
    }
    int dev = 0, sms = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    ChainArgs a{};
    a.run_item = runs.run_item;
    a.run_len = runs.run_len;
    a.n_items = runs.n_items;
    a.n_runs = runs.n_runs;
    a.run_begin = runs.run_begin;
    a.run_end = runs.run_end;
    a.leaves = leaves;
    a.live = live;
    a.n_bins = n_bins;
    a.cap = cap;
    a.ffd = ffd ? 1 : 0;
    // runs per block: small blocks shorten each warp's serve of the block
    // that walks the whole chain last; large ones amortise the hand-off
    const char* erb = std::getenv("HBP_CHAIN_RB");
    a.rb = erb ? static_cast<u32>(std::atoi(erb)) : 32u;
    if (a.rb != 8 && a.rb != 16) a.rb = 32;
    a.nblocks = (runs.run_end - runs.run_begin + a.rb - 1) / a.rb;
    a.item_bin = item_bin;
    a.item_slot = item_slot;
    a.take = take;
    a.single = std::getenv("HBP_CHAIN_NOSINGLE") == nullptr ? 1 : 0;
    const char* es = std::getenv("HBP_CHAIN_SLEEP");
    a.sleep = es ? static_cast<u32>(std::atoi(es)) : 0u;
    // Bins are covered by consecutive passes: a pass's tail hands the counts
    // its bins left (per run) to the next pass's head, exactly as one longer
    // chain would. A pass uses the fewest rows per warp (>= HBP_CHAIN_M,
    // default 8, measured best on C2) whose chain is resident; FFD's first
    // pass is sized by the caller's estimate of the bins FFD opens, so the
    // 2x bin bound costs a second pass only when the estimate is short.
    // Lane width: a run's serve costs about M-proportional work on the
    // frontier warp (divisions, prefix and takes over the lane's M bins),
    // while every extra warp adds a hop to the path of each block. Measured
    // (tools/chain_env_ab.sh): chains of up to ~5K bins (C1/C3 plans) run
    // 1.3-2.2x faster at M = 1-2 than at 8; C2's 90-150K-bin chains are
    // fastest at M = 8. So: the narrowest lanes that keep the chain within
    // kMaxNarrowWarps warps, else M = 8.
    const char* em = std::getenv("HBP_CHAIN_M");
    constexpr u64 kMaxNarrowWarps = 160;
    const u64 cap_of[5] = {chain_capacity<1>(sms), chain_capacity<2>(sms), chain_capacity<4>(sms),
                           chain_capacity<8>(sms), chain_capacity<16>(sms)};
    const int widths[5] = {1, 2, 4, 8, 16};
    DevBuf<u32> carry[2] = {DevBuf<u32>(runs.n_runs + 1, s), DevBuf<u32>(runs.n_runs + 1, s)};
    u32 pos = 0, top = live;
    bool left_over = false, any_replay = false;
    for (int pass = 0; pos < n_bins; ++pass) {
        u64 want = n_bins - pos;
        if (pass == 0 && first_pass_bins > 0 && first_pass_bins < want) want = first_pass_bins;
        int m0 = 8;
        if (em) {
            m0 = std::atoi(em);
        } else {
            for (int w : {1, 2, 4})
                if ((want + 32ull * w - 1) / (32ull * w) <= kMaxNarrowWarps) {
                    m0 = w;
                    break;
                }
        }
        int wi = 0;
        while (wi < 5 && (widths[wi] < m0 || cap_of[wi] < want)) ++wi;
        if (wi == 5) {
            wi = 4;
            want = cap_of[4];
        }
        if (want == 0) return false;
        a.bin0 = pos;
        a.bin_end = static_cast<u32>(pos + want);
        a.carry_in = pass == 0 ? nullptr : carry[(pass + 1) & 1].p;
        a.carry_out = carry[pass & 1].p;
        std::pair<u32, bool> r;
        switch (widths[wi]) {
            case 1: r = run_pass<1>(c, a, "fit.chain"); break;
            case 2: r = run_pass<2>(c, a, "fit.chain"); break;
            case 4: r = run_pass<4>(c, a, "fit.chain"); break;
            case 8: r = run_pass<8>(c, a, "fit.chain"); break;
            default: r = run_pass<16>(c, a, "fit.chain"); break;
        }
        top = std::max(top, r.first);
        left_over = r.second;
        any_replay = any_replay || a.replayed;
        pos = a.bin_end;
        if (!left_over) break;
    }
    // FFD never runs past its bin bound; greedy fill leaves what no pack took
    if (ffd && left_over) throw EngineError(HBP_ERR_CUDA, "first-fit chain: bin capacity exceeded");
    used = top;
    // replays wrote heads only: expand them (items the chains wrote in full are
    // rewritten with the same values); without replays every take is written
    // and items no take covers keep the caller's kNone
    if (expand && any_replay) expand_heads(c, runs.n_items, item_bin, item_slot, take);
    return true;
}

}  // namespace hbp_b200
