// firstfit.cu — first-fit by runs: the FFD residue pass of ISF and greedy
// fill, exactly as the reference orders them.
//
// Reference: first_fit over sort_decreasing (src/packing.cpp:55-60, 86-103)
// places each item (length desc, id asc) into the first pack with room,
// else opens a pack. For a run of c equal items of size s this means: visit
// bins in index order, every bin with residual r >= s takes floor(r / s)
// items (the run's next ids), until the run is used up; then open bins of
// floor(cap / s) items. greedy_fill (src/balance.cpp:62-101) -- each pack,
// nearest pool first, repeatedly takes the largest sample that fits, lowest
// id first -- assigns exactly the same way when its candidate samples are
// visited by (length desc, id asc): pools are disjoint length ranges and a
// pack only ever receives decreasing lengths. It never opens bins.
//
// Engine: one warp walks the runs over a 32-ary max-residual tree whose
// leaves are (residual << 32 | count) per bin: a ballot per level finds the
// first child with max >= s, the leaf chunk is filled with one warp scan of
// floor(r / s), maxima are written back up the path and the search resumes
// from the path (finger search) instead of the root. Items larger than
// cap / 2 can never share a bin; in FFD mode they are placed in bulk by a
// parallel kernel before the walk. Output is a compact record list expanded
// to per-item (bin, slot) by a parallel kernel.
#include "stages.cuh"
#include "radix.cuh"

namespace hbp_b200 {

namespace {

constexpr int kMaxLevels = 8;

struct TreeLayout {
    u32* base;                  // all levels >= 1, concatenated
    u64 off[kMaxLevels + 1];    // offset of level h (h >= 1) inside base
    u64 size[kMaxLevels + 1];   // entries at level h (size[0] = max_bins leaves)
    int H;                      // root level (size[H] == 1)
};

TreeLayout make_layout(u64 max_bins) {
    TreeLayout t{};
    t.size[0] = max_bins;
    u64 total = 0;
    int h = 0;
    u64 sz = max_bins;
    do {
        ++h;
        sz = (sz + 31) / 32;
        t.size[h] = sz;
        t.off[h] = total;
        total += sz;
    } while (sz > 1 && h < kMaxLevels);
    t.H = h;
    if (t.size[h] != 1) throw EngineError(HBP_ERR_VALIDATION, "first-fit tree too deep");
    t.off[0] = total;  // total entries (stashed)
    return t;
}

// Run heads: a new length, or (fill with negative ids) the first item of
// the non-negative class within a length.
__device__ __forceinline__ bool neg_item(u64 e, const u32* key32, u64 neg_keys) {
    const u32 ix = entry_idx(e);
    return (key32 ? key32[ix] : ix) < neg_keys;
}
__device__ __forceinline__ bool run_head(const u64* items, u64 i, const u32* key32, u64 neg_keys) {
    if (i == 0 || entry_len(items[i]) != entry_len(items[i - 1])) return true;
    return neg_keys && neg_item(items[i], key32, neg_keys) != neg_item(items[i - 1], key32, neg_keys);
}

// Level h >= 1 from level h-1 (h-1 == 0: leaves).
__global__ void k_tree_level(const u64* __restrict__ leaves, u32* __restrict__ base, TreeLayout t, int h, u64 lo,
                             u64 hi) {
    // recompute entries [lo, hi) of level h
    for (u64 i = lo + blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < hi;
         i += static_cast<u64>(gridDim.x) * blockDim.x) {
        u32 m = 0;
        for (int k = 0; k < 32; ++k) {
            const u64 c = 32 * i + k;
            if (c >= t.size[h - 1]) break;
            const u32 v = (h == 1) ? static_cast<u32>(leaves[c] >> 32) : base[t.off[h - 1] + c];
            m = v > m ? v : m;
        }
        base[t.off[h] + i] = m;
    }
}

// FFD bulk: items [0, k) all longer than cap / 2 -> bin i each.
__global__ void k_bulk_big(const u64* __restrict__ items, u64 k, u32 cap, u64* __restrict__ leaves,
                           u32* __restrict__ item_bin, u32* __restrict__ item_slot, u32* __restrict__ take) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < k;
         i += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u32 l = entry_len(items[i]);
        leaves[i] = (static_cast<u64>(cap - l) << 32) | 1u;
        if (item_bin) {  // chain path: each bulk item is a head of one
            item_bin[i] = static_cast<u32>(i);
            item_slot[i] = 0;
            take[i] = 1;
        }
    }
}

struct EngineArgs {
    const u64* items;
    u32 n_items;
    const u32* run_item;
    const u32* run_len;
    u32 n_runs;
    u32 run_begin;
    u32 run_end;  // runs [run_begin, run_end) are processed
    u64* leaves;
    TreeLayout t;
    u32 bins0;
    u32 max_bins;
    u32 cap;
    int ffd;
    FitRecords rec;
    u32 rec0;
    u32 max_records;
    u32* out;  // [0] bins, [1] records, [2] overflow flag
    unsigned long long* prof;  // optional cycle counters (HBP_TRACE)
};

__device__ __forceinline__ u32 tree_get(const TreeLayout& t, int h, u64 i) {
    return i < t.size[h] ? t.base[t.off[h] + i] : 0u;
}

// One warp. Shared: children values held along the current path.
__global__ void __launch_bounds__(32) k_fit_engine(EngineArgs a) {
    __shared__ u32 s_held[kMaxLevels + 1][32];
    __shared__ u64 s_node[kMaxLevels + 1];
    const unsigned lane = threadIdx.x;
    const TreeLayout& t = a.t;
    const int H = t.H;
    u32 B = a.bins0;
    u32 nrec = a.rec0;
    bool overflow = false;

    // loads the children of node n at level h into s_held[h]; for h == 1 also
    // returns this lane's leaf word
    auto load_children = [&](int h, u64 n) -> u64 {
        u64 leaf = 0;
        const u64 ci = 32 * n + lane;
        if (h == 1) {
            leaf = ci < t.size[0] ? a.leaves[ci] : 0ull;
            s_held[1][lane] = static_cast<u32>(leaf >> 32);
        } else {
            s_held[h][lane] = tree_get(t, h - 1, ci);
        }
        s_node[h] = n;
        __syncwarp();
        return leaf;
    };
    // after s_held[1] changed: write maxima up to the root
    auto propagate = [&]() {
        for (int h = 1; h <= H; ++h) {
            const u32 m = warp_max(s_held[h][lane]);
            const u64 n = s_node[h];
            if (lane == 0) t.base[t.off[h] + n] = m;
            if (h < H && lane == static_cast<unsigned>(n & 31)) s_held[h + 1][lane] = m;
            __syncwarp();
        }
    };

    for (u32 k = a.run_begin; k < a.run_end; ++k) {
        const u32 s = a.run_len[k];
        u32 item = a.run_item[k];
        const u32 end_item = (k + 1 < a.n_runs) ? a.run_item[k + 1] : a.n_items;
        u32 c = end_item - item;

        const u32 rootmax = t.base[t.off[H]];
        if (rootmax >= s && B > 0) {
            // fresh descent from the root
            u64 leaf = load_children(H, 0);
            int h = H;
            int after = -1;
            while (c > 0) {
                const unsigned mask = __ballot_sync(0xffffffffu, s_held[h][lane] >= s) &
                                      (after >= 31 ? 0u : (~0u << (after + 1)));
                if (mask == 0) {
                    if (h == H) break;  // nothing left with room
                    after = static_cast<int>(s_node[h] & 31);
                    ++h;
                    continue;
                }
                const int f = __ffs(mask) - 1;
                if (h > 1) {
                    const u64 child = 32 * s_node[h] + f;
                    leaf = load_children(h - 1, child);
                    --h;
                    after = -1;
                    continue;
                }
                // h == 1: fill the eligible bins of this chunk in order
                const u32 res = s_held[1][lane];
                const bool elig = static_cast<int>(lane) >= f && res >= s;
                const u32 capl = elig ? res / s : 0u;
                const u32 incl = warp_inclusive_scan(capl);
                const u32 excl = incl - capl;
                const u32 take = excl >= c ? 0u : (capl < c - excl ? capl : c - excl);
                const unsigned tm = __ballot_sync(0xffffffffu, take > 0);
                const u32 r = __popc(tm & ((1u << lane) - 1u));
                if (take > 0) {
                    const u32 ri = nrec + r;
                    if (ri < a.max_records) {
                        a.rec.item[ri] = item + excl;
                        a.rec.count[ri] = take;
                        a.rec.bin[ri] = static_cast<u32>(32 * s_node[1] + lane);
                        a.rec.per_bin[ri] = take;
                        a.rec.slot0[ri] = static_cast<u32>(leaf);
                    }
                    const u32 nres = res - take * s;
                    const u32 ncnt = static_cast<u32>(leaf) + take;
                    leaf = (static_cast<u64>(nres) << 32) | ncnt;
                    a.leaves[32 * s_node[1] + lane] = leaf;
                    s_held[1][lane] = nres;
                }
                __syncwarp();
                const u32 used = __shfl_sync(0xffffffffu, incl, 31);
                const u32 got = used < c ? used : c;
                nrec += __popc(tm);
                c -= got;
                item += got;
                propagate();
                // every eligible bin of the chunk is now below s: continue right
                after = 31;
            }
        }
        if (c > 0 && a.ffd) {
            const u32 per = a.cap / s;
            const u32 nb = (c + per - 1) / per;
            if (B + nb > a.max_bins) {
                overflow = true;
                break;
            }
            if (nrec < a.max_records && lane == 0) {
                a.rec.item[nrec] = item;
                a.rec.count[nrec] = c;
                a.rec.bin[nrec] = B;
                a.rec.per_bin[nrec] = per;
                a.rec.slot0[nrec] = 0;
            }
            ++nrec;
            const u32 res_full = a.cap - per * s;
            const u32 last_cnt = c - (nb - 1) * per;
            const u32 res_last = a.cap - last_cnt * s;
            for (u32 b = lane; b < nb; b += 32) {
                const bool last = (b == nb - 1);
                a.leaves[B + b] = (static_cast<u64>(last ? res_last : res_full) << 32) | (last ? last_cnt : per);
            }
            // raise maxima over the new range at every level
            const u64 lo = B, hi = static_cast<u64>(B) + nb - 1;  // inclusive
            const u64 full_hi = nb > 1 ? hi - 1 : lo;              // last full bin (if nb > 1)
            for (int h = 1; h <= H; ++h) {
                const u64 ilo = lo >> (5 * h), ihi = hi >> (5 * h);
                for (u64 i = ilo + lane; i <= ihi; i += 32) {
                    const u64 slo = i << (5 * h), shi = ((i + 1) << (5 * h)) - 1;
                    u32 v = t.base[t.off[h] + i];
                    if (nb > 1 && slo <= full_hi && shi >= lo) v = v > res_full ? v : res_full;
                    if (slo <= hi && shi >= hi) v = v > res_last ? v : res_last;
                    t.base[t.off[h] + i] = v;
                }
                __syncwarp();
            }
            B += nb;
            c = 0;
        }
        __syncwarp();
    }
    if (lane == 0) {
        a.out[0] = B;
        a.out[1] = nrec;
        a.out[2] = (overflow || nrec > a.max_records) ? 1u : 0u;
    }
}

// ---------------------------------------------------------------------------
// Engine v3: the whole max tree (levels >= 1) lives in shared memory as
// saturated u16 maxima (min(max, 65535)); leaves stay in HBM/L2. For s <=
// 65535 a saturated comparison is exact; for larger s a saturated entry is
// only a candidate and the leaf check decides. Per run the warp descends
// from the root to the first candidate chunk, collects up to 32 candidate
// chunks in index order with one ballot per tree node, copies all their
// leaves into shared memory with cp.async (one L2 round trip for the whole
// batch), then fills them in order.
// ---------------------------------------------------------------------------

constexpr u32 kSat = 65535u;
__device__ __forceinline__ unsigned short sat16(u32 v) { return static_cast<unsigned short>(v > kSat ? kSat : v); }

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

__global__ void __launch_bounds__(32) k_fit_engine_smem(EngineArgs a) {
    extern __shared__ unsigned short st[];  // tree levels 1..H
    __shared__ u64 s_cand[32];
    __shared__ __align__(16) u64 s_leaf[32][32];
    const unsigned lane = threadIdx.x;
    const unsigned lt = (1u << lane) - 1u;
    const TreeLayout& t = a.t;
    const int H = t.H;
    const u64 total = t.off[0];
    for (u64 i = lane; i < total; i += 32) st[i] = sat16(t.base[i]);
    __syncwarp();

    auto getL = [&](int h, u64 i) -> u32 { return i < t.size[h] ? st[t.off[h] + i] : 0u; };
    // first level-1 index with saturated max >= q (caller checked the root)
    auto find_first = [&](u32 q) -> u64 {
        u64 idx = 0;
        for (int h = H; h > 1; --h) {
            const u64 base = idx << 5;
            const unsigned m = __ballot_sync(0xffffffffu, getL(h - 1, base + lane) >= q);
            if (!m) return ~0ull;
            idx = base + (__ffs(m) - 1);
        }
        return idx;
    };
    // smallest level-1 index >= j with saturated max >= q, or ~0
    auto find_next = [&](u64 j, u32 q) -> u64 {
        int h = 1;
        u64 idx = j;
        while (true) {
            const u64 base = idx & ~31ull;
            const unsigned m = __ballot_sync(0xffffffffu, getL(h, base + lane) >= q && base + lane >= idx);
            if (m) {
                idx = base + (__ffs(m) - 1);
                break;
            }
            if (h == H) return ~0ull;
            idx = (base >> 5) + 1;
            ++h;
        }
        while (h > 1) {
            const u64 base = idx << 5;
            const unsigned m = __ballot_sync(0xffffffffu, getL(h - 1, base + lane) >= q);
            idx = base + (__ffs(m) - 1);
            --h;
        }
        return idx;
    };
    // level-1 entry j decreased to `v` (true max): rewrite ancestors. Values
    // only decrease here, so a parent needs recomputing only when the child
    // was (one of) its maxima.
    auto update_up = [&](u64 j, u32 v) {
        u32 old_child = getL(1, j);
        const u32 nv = sat16(v);
        if (old_child == nv) return;
        if (lane == 0) st[t.off[1] + j] = static_cast<unsigned short>(nv);
        __syncwarp();
        u64 idx = j;
        for (int h = 2; h <= H; ++h) {
            const u64 p = idx >> 5;
            const u32 old = getL(h, p);
            if (old_child < old) break;  // another child holds the max
            const u32 m = warp_max(getL(h - 1, (p << 5) + lane));
            if (old == m) break;
            if (lane == 0) st[t.off[h] + p] = static_cast<unsigned short>(m);
            __syncwarp();
            old_child = old;
            idx = p;
        }
    };

    u32 B = a.bins0;
    u32 nrec = a.rec0;
    bool overflow = false;
    u32 win_base = a.run_begin;
    u32 my_len = 0, my_item = 0;
    auto load_window = [&](u32 base) {
        win_base = base;
        const u32 r = base + lane;
        my_len = r < a.n_runs ? a.run_len[r] : 0u;
        my_item = r < a.n_runs ? a.run_item[r] : a.n_items;
    };
    load_window(a.run_begin);
    // cycle counters: 0 collect, 1 load, 2 process, 3 new bins, 4 searched runs, 5 candidates, 6 collect rounds
    unsigned long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long t0 = 0;
    const bool prof = a.prof != nullptr;

    for (u32 k = a.run_begin; k < a.run_end; ++k) {
        if (k - win_base == 32) load_window(k);
        const unsigned wl = k - win_base;
        const u32 s = __shfl_sync(0xffffffffu, my_len, wl);
        u32 item = __shfl_sync(0xffffffffu, my_item, wl);
        u32 end_item;
        if (wl < 31) {
            end_item = __shfl_sync(0xffffffffu, my_item, wl + 1);
        } else {
            end_item = (k + 1 < a.n_runs) ? a.run_item[k + 1] : a.n_items;
        }
        u32 c = end_item - item;
        const u32 q = s > kSat ? kSat : s;

        if (B > 0 && getL(H, 0) >= q) {
            u64 pos = 0;
            bool first = true;
            pc[4] += 1;
            while (c > 0) {
                if (prof) t0 = clock64();
                const u32 K = c < 32 ? c : 32u;
                u32 ncand = 0;
                pc[6] += 1;
                while (ncand < K) {
                    const u64 j = first ? find_first(q) : find_next(pos, q);
                    first = false;
                    if (j == ~0ull) break;
                    const u64 base = j & ~31ull;
                    const unsigned m =
                        __ballot_sync(0xffffffffu, getL(1, base + lane) >= q && base + lane >= j);
                    const u32 cnt = __popc(m);
                    const u32 room = K - ncand;
                    const u32 r = __popc(m & lt);
                    if (((m >> lane) & 1u) && r < room) s_cand[ncand + r] = base + lane;
                    __syncwarp();
                    if (cnt <= room) {
                        ncand += cnt;
                        pos = base + 32;
                    } else {
                        ncand += room;
                        pos = s_cand[ncand - 1] + 1;
                    }
                }
                if (prof) {
                    const long long t1 = clock64();
                    pc[0] += t1 - t0;
                    t0 = t1;
                }
                if (ncand == 0) break;
                pc[5] += ncand;
                for (u32 qq = 0; qq < ncand; ++qq) {
                    const u64 li = s_cand[qq] * 32 + lane;
                    if (li < a.max_bins) cp_async8(&s_leaf[qq][lane], &a.leaves[li]);
                    else s_leaf[qq][lane] = 0ull;
                }
                cp_async_wait_all();
                __syncwarp();
                if (prof) {
                    const long long t1 = clock64();
                    pc[1] += t1 - t0;
                    t0 = t1;
                }
                for (u32 qq = 0; qq < ncand && c > 0; ++qq) {
                    const u64 leaf = s_leaf[qq][lane];
                    const u32 res = static_cast<u32>(leaf >> 32);
                    const u32 capl = res >= s ? res / s : 0u;
                    const u32 incl = warp_inclusive_scan(capl);
                    const u32 excl = incl - capl;
                    const u32 take = excl >= c ? 0u : (capl < c - excl ? capl : c - excl);
                    const unsigned tm = __ballot_sync(0xffffffffu, take > 0);
                    const u64 chunk = s_cand[qq];
                    u32 nres = res;
                    if (take > 0) {
                        const u32 ri = nrec + __popc(tm & lt);
                        if (ri < a.max_records) {
                            a.rec.item[ri] = item + excl;
                            a.rec.count[ri] = take;
                            a.rec.bin[ri] = static_cast<u32>(chunk * 32 + lane);
                            a.rec.per_bin[ri] = take;
                            a.rec.slot0[ri] = static_cast<u32>(leaf);
                        }
                        nres = res - take * s;
                        a.leaves[chunk * 32 + lane] = (static_cast<u64>(nres) << 32) | (static_cast<u32>(leaf) + take);
                    }
                    const u32 used = __shfl_sync(0xffffffffu, incl, 31);
                    const u32 got = used < c ? used : c;
                    nrec += __popc(tm);
                    c -= got;
                    item += got;
                    if (tm) update_up(chunk, warp_max(nres));
                }
                if (prof) {
                    const long long t1 = clock64();
                    pc[2] += t1 - t0;
                    t0 = t1;
                }
            }
        }
        if (prof) t0 = clock64();
        if (c > 0 && a.ffd) {
            const u32 per = a.cap / s;
            const u32 nb = (c + per - 1) / per;
            if (static_cast<u64>(B) + nb > a.max_bins) {
                overflow = true;
                break;
            }
            if (nrec < a.max_records && lane == 0) {
                a.rec.item[nrec] = item;
                a.rec.count[nrec] = c;
                a.rec.bin[nrec] = B;
                a.rec.per_bin[nrec] = per;
                a.rec.slot0[nrec] = 0;
            }
            ++nrec;
            const u32 res_full = a.cap - per * s;
            const u32 last_cnt = c - (nb - 1) * per;
            const u32 res_last = a.cap - last_cnt * s;
            for (u32 b = lane; b < nb; b += 32) {
                const bool last = (b == nb - 1);
                a.leaves[B + b] = (static_cast<u64>(last ? res_last : res_full) << 32) | (last ? last_cnt : per);
            }
            const u64 lo = B, hi = static_cast<u64>(B) + nb - 1;
            const u64 full_hi = nb > 1 ? hi - 1 : lo;
            for (int h = 1; h <= H; ++h) {
                const u64 ilo = lo >> (5 * h), ihi = hi >> (5 * h);
                for (u64 i = ilo + lane; i <= ihi; i += 32) {
                    const u64 slo = i << (5 * h), shi = ((i + 1) << (5 * h)) - 1;
                    u32 val = getL(h, i);
                    if (nb > 1 && slo <= full_hi && shi >= lo) val = val > res_full ? val : res_full;
                    if (slo <= hi && shi >= hi) val = val > res_last ? val : res_last;
                    if (i < t.size[h]) st[t.off[h] + i] = sat16(val);
                }
                __syncwarp();
            }
            B += nb;
        }
        if (prof) pc[3] += clock64() - t0;
        __syncwarp();
    }
    if (lane == 0) {
        a.out[0] = B;
        a.out[1] = nrec;
        a.out[2] = (overflow || nrec > a.max_records) ? 1u : 0u;
        if (prof)
            for (int i = 0; i < 8; ++i) a.prof[i] = pc[i];
    }
}

// ---------------------------------------------------------------------------
// Engine v4: fixed three-level max structure in shared memory (u16,
// saturated): L1 = max of 32 leaves (a chunk), L2 = max of 32 chunks, L3 =
// max of 32 L2 entries (<= 128 entries, scanned by the warp). Fixed depth,
// offsets in registers, warp maxima with REDUX, and a 32-chunk leaf cache in
// shared memory (direct-mapped by chunk index, write-through to HBM) so
// that consecutive runs touching the same chunks skip the L2 round trip.
// Bins <= 128 * 32768; larger trees use v3.
// ---------------------------------------------------------------------------

struct V4Layout {
    u32 n1, n2, n3;      // live entries per level
    u32 o2, o3;          // offsets of L2 / L3 in the smem array (L1 at 0)
    u32 total;           // padded entries
};

V4Layout make_v4(u64 bins) {
    V4Layout v{};
    v.n1 = static_cast<u32>((bins + 31) / 32);
    v.n2 = (v.n1 + 31) / 32;
    v.n3 = (v.n2 + 31) / 32;
    const u32 p1 = (v.n1 + 31) / 32 * 32, p2 = (v.n2 + 31) / 32 * 32;
    v.o2 = p1;
    v.o3 = p1 + p2;
    v.total = p1 + p2 + 128;
    return v;
}

__global__ void __launch_bounds__(32) k_fit_engine_v4(EngineArgs a, V4Layout L) {
    extern __shared__ unsigned short st4[];
    __shared__ __align__(16) u64 s_cache[32][32];
    __shared__ u32 s_tag[32];
    __shared__ u32 s_cand[32];
    const unsigned lane = threadIdx.x;
    const unsigned lt = (1u << lane) - 1u;
    unsigned short* L1 = st4;
    unsigned short* L2 = st4 + L.o2;
    unsigned short* L3 = st4 + L.o3;
    // build the levels from the global tree (levels 1..3 of TreeLayout are
    // exactly L1..L3 here; deeper levels are not needed)
    {
        const TreeLayout& t = a.t;
        for (u32 i = lane; i < L.total; i += 32) st4[i] = 0;
        __syncwarp();
        for (u32 i = lane; i < L.n1; i += 32) L1[i] = sat16(t.base[t.off[1] + i]);
        for (u32 i = lane; i < L.n2; i += 32) L2[i] = t.H >= 2 ? sat16(t.base[t.off[2] + i]) : 0;
        __syncwarp();
        if (t.H < 2) {  // derive L2 / L3 from L1
            for (u32 i = lane; i < L.n2; i += 32) {
                u32 m = 0;
                for (u32 k = 0; k < 32 && 32 * i + k < L.n1; ++k) m = max(m, static_cast<u32>(L1[32 * i + k]));
                L2[i] = static_cast<unsigned short>(m);
            }
        }
        __syncwarp();
        for (u32 i = lane; i < L.n3; i += 32) {
            u32 m = 0;
            for (u32 k = 0; k < 32 && 32 * i + k < L.n2; ++k) m = max(m, static_cast<u32>(L2[32 * i + k]));
            L3[i] = static_cast<unsigned short>(m);
        }
        s_tag[lane] = kNone;
        __syncwarp();
    }
    auto root = [&]() -> u32 {
        u32 m = max(max(L3[lane], L3[lane + 32]), max(L3[lane + 64], L3[lane + 96]));
        return __reduce_max_sync(0xffffffffu, m);
    };
    // descend into L3 entry i3 / L2 entry i2 to the first chunk >= q
    auto down_from_l2 = [&](u32 i2, u32 q) -> u32 {
        const unsigned m1 = __ballot_sync(0xffffffffu, L1[32 * i2 + lane] >= q);
        return 32 * i2 + (__ffs(m1) - 1);
    };
    auto down_from_l3 = [&](u32 i3, u32 q) -> u32 {
        const unsigned m2 = __ballot_sync(0xffffffffu, L2[32 * i3 + lane] >= q);
        return down_from_l2(32 * i3 + (__ffs(m2) - 1), q);
    };
    // first L3 entry > after (after = -1: any) with max >= q, or kNone
    auto scan_l3 = [&](int after, u32 q) -> u32 {
#pragma unroll
        for (int part = 0; part < 4; ++part) {
            const int idx = part * 32 + static_cast<int>(lane);
            const unsigned m = __ballot_sync(0xffffffffu, idx > after && L3[idx] >= q);
            if (m) return static_cast<u32>(part * 32 + __ffs(m) - 1);
        }
        return kNone;
    };
    // smallest chunk >= j with max >= q
    auto find_next = [&](u32 j, u32 q) -> u32 {
        if (j >= L.n1) return kNone;
        const u32 b1 = j & ~31u;
        const unsigned m1 = __ballot_sync(0xffffffffu, L1[b1 + lane] >= q && b1 + lane >= j);
        if (m1) return b1 + (__ffs(m1) - 1);
        const u32 j2 = (j >> 5) + 1;
        const u32 b2 = (j2 & ~31u);
        if (j2 < L.n2 && (j2 & 31u)) {
            const unsigned m2 = __ballot_sync(0xffffffffu, L2[b2 + lane] >= q && b2 + lane >= j2);
            if (m2) return down_from_l2(b2 + (__ffs(m2) - 1), q);
        }
        const u32 i3 = scan_l3(static_cast<int>((j2 + 31) / 32) - 1, q);
        return i3 == kNone ? kNone : down_from_l3(i3, q);
    };
    auto find_first = [&](u32 q) -> u32 {
        const u32 i3 = scan_l3(-1, q);
        return i3 == kNone ? kNone : down_from_l3(i3, q);
    };
    // chunk j's max decreased to v
    auto update_down = [&](u32 j, u32 v) {
        const u32 old1 = L1[j];
        const u32 n1 = v > kSat ? kSat : v;
        if (old1 == n1) return;
        if (lane == 0) L1[j] = static_cast<unsigned short>(n1);
        __syncwarp();
        const u32 p2 = j >> 5;
        const u32 old2 = L2[p2];
        if (old1 < old2) return;
        const u32 m2 = __reduce_max_sync(0xffffffffu, static_cast<u32>(L1[32 * p2 + lane]));
        if (m2 == old2) return;
        if (lane == 0) L2[p2] = static_cast<unsigned short>(m2);
        __syncwarp();
        const u32 p3 = p2 >> 5;
        const u32 old3 = L3[p3];
        if (old2 < old3) return;
        const u32 m3 = __reduce_max_sync(0xffffffffu, static_cast<u32>(L2[32 * p3 + lane]));
        if (lane == 0) L3[p3] = static_cast<unsigned short>(m3);
        __syncwarp();
    };

    u32 B = a.bins0;
    u32 nrec = a.rec0;
    bool overflow = false;
    u32 win_base = a.run_begin;
    u32 my_len = 0, my_item = 0;
    auto load_window = [&](u32 base) {
        win_base = base;
        const u32 r = base + lane;
        my_len = r < a.n_runs ? a.run_len[r] : 0u;
        my_item = r < a.n_runs ? a.run_item[r] : a.n_items;
    };
    load_window(a.run_begin);
    u32 rmax = root();
    // cycle counters (HBP_TRACE): 0 collect 1 load 2 process 3 new bins 4 searched runs 5 candidates 6 rounds 7 misses
    unsigned long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const bool prof = a.prof != nullptr;
    long long t0 = 0;

    for (u32 k = a.run_begin; k < a.run_end; ++k) {
        if (k - win_base == 32) load_window(k);
        const unsigned wl = k - win_base;
        const u32 s = __shfl_sync(0xffffffffu, my_len, wl);
        u32 item = __shfl_sync(0xffffffffu, my_item, wl);
        const u32 nxt = __shfl_sync(0xffffffffu, my_item, wl < 31 ? wl + 1 : 31);
        const u32 end_item = wl < 31 ? nxt : ((k + 1 < a.n_runs) ? a.run_item[k + 1] : a.n_items);
        u32 c = end_item - item;
        const u32 q = s > kSat ? kSat : s;

        if (B > 0 && rmax >= q) {
            u32 pos = 0;
            bool first = true;
            pc[4] += 1;
            while (c > 0) {
                if (prof) t0 = clock64();
                pc[6] += 1;
                // candidates with distinct cache slots, in chunk order
                const u32 K = c < 32 ? c : 32u;
                u32 ncand = 0, used_slots = 0;
                bool stop = false;
                while (ncand < K && !stop) {
                    const u32 j = first ? find_first(q) : find_next(pos, q);
                    first = false;
                    if (j == kNone) break;
                    const u32 b1 = j & ~31u;
                    const unsigned m = __ballot_sync(0xffffffffu, L1[b1 + lane] >= q && b1 + lane >= j);
                    // take candidates in order while slots stay distinct
                    unsigned mm = m;
                    while (mm && ncand < K) {
                        const u32 cj = b1 + (__ffs(mm) - 1);
                        const u32 slot = cj & 31u;
                        if (used_slots & (1u << slot)) {
                            stop = true;
                            break;
                        }
                        used_slots |= 1u << slot;
                        if (lane == 0) s_cand[ncand] = cj;
                        ++ncand;
                        mm &= mm - 1;
                        pos = cj + 1;
                    }
                    if (!mm && !stop) pos = b1 + 32;
                }
                __syncwarp();
                if (prof) {
                    const long long t1 = clock64();
                    pc[0] += t1 - t0;
                    t0 = t1;
                }
                if (ncand == 0) break;
                pc[5] += ncand;
                // fill misses with cp.async (hits are already in s_cache)
                bool any_miss = false;
                for (u32 qq = 0; qq < ncand; ++qq) {
                    const u32 cj = s_cand[qq];
                    const u32 slot = cj & 31u;
                    if (s_tag[slot] != cj) {
                        any_miss = true;
                        pc[7] += 1;
                        const u64 li = static_cast<u64>(cj) * 32 + lane;
                        if (li < a.max_bins) cp_async8(&s_cache[slot][lane], &a.leaves[li]);
                        else s_cache[slot][lane] = 0ull;
                    }
                }
                if (any_miss) cp_async_wait_all();
                __syncwarp();
                if (lane < ncand) s_tag[s_cand[lane] & 31u] = s_cand[lane];
                __syncwarp();
                if (prof) {
                    const long long t1 = clock64();
                    pc[1] += t1 - t0;
                    t0 = t1;
                }
                for (u32 qq = 0; qq < ncand && c > 0; ++qq) {
                    const u32 cj = s_cand[qq];
                    const u32 slot = cj & 31u;
                    const u64 leaf = s_cache[slot][lane];
                    const u32 res = static_cast<u32>(leaf >> 32);
                    const bool elig = res >= s;
                    const unsigned em = __ballot_sync(0xffffffffu, elig);
                    if (!em) continue;
                    const u32 capl = elig ? res / s : 0u;
                    u32 incl;
                    if ((em & (em - 1)) == 0) {  // one eligible lane: no scan needed
                        const int f = __ffs(em) - 1;
                        const u32 only = __shfl_sync(0xffffffffu, capl, f);
                        incl = static_cast<int>(lane) >= f ? only : 0u;
                    } else {
                        incl = warp_inclusive_scan(capl);
                    }
                    const u32 excl = incl - capl;
                    const u32 take = excl >= c ? 0u : (capl < c - excl ? capl : c - excl);
                    const unsigned tm = __ballot_sync(0xffffffffu, take > 0);
                    u32 nres = res;
                    if (take > 0) {
                        const u32 ri = nrec + __popc(tm & lt);
                        if (ri < a.max_records) {
                            a.rec.item[ri] = item + excl;
                            a.rec.count[ri] = take;
                            a.rec.bin[ri] = cj * 32 + lane;
                            a.rec.per_bin[ri] = take;
                            a.rec.slot0[ri] = static_cast<u32>(leaf);
                        }
                        nres = res - take * s;
                        const u64 nl = (static_cast<u64>(nres) << 32) | (static_cast<u32>(leaf) + take);
                        s_cache[slot][lane] = nl;
                        a.leaves[static_cast<u64>(cj) * 32 + lane] = nl;
                    }
                    const u32 used = __shfl_sync(0xffffffffu, incl, 31);
                    const u32 got = used < c ? used : c;
                    nrec += __popc(tm);
                    c -= got;
                    item += got;
                    if (tm) update_down(cj, __reduce_max_sync(0xffffffffu, nres));
                }
                __syncwarp();
                if (prof) pc[2] += clock64() - t0;
            }
            rmax = root();
        }
        if (prof) t0 = clock64();
        if (c > 0 && a.ffd) {
            const u32 per = a.cap / s;
            const u32 nb = (c + per - 1) / per;
            if (static_cast<u64>(B) + nb > a.max_bins) {
                overflow = true;
                break;
            }
            if (nrec < a.max_records && lane == 0) {
                a.rec.item[nrec] = item;
                a.rec.count[nrec] = c;
                a.rec.bin[nrec] = B;
                a.rec.per_bin[nrec] = per;
                a.rec.slot0[nrec] = 0;
            }
            ++nrec;
            const u32 res_full = a.cap - per * s;
            const u32 last_cnt = c - (nb - 1) * per;
            const u32 res_last = a.cap - last_cnt * s;
            for (u32 b = lane; b < nb; b += 32) {
                const bool last = (b == nb - 1);
                a.leaves[B + b] = (static_cast<u64>(last ? res_last : res_full) << 32) | (last ? last_cnt : per);
            }
            const u32 lo = B, hi = B + nb - 1;
            const u32 full_hi = nb > 1 ? hi - 1 : lo;
            // cached chunks overlapping the new range are stale
            if (s_tag[lane] != kNone && s_tag[lane] >= (lo >> 5) && s_tag[lane] <= (hi >> 5)) s_tag[lane] = kNone;
            auto raise = [&](unsigned short* Lv, int shift) {
                const u32 ilo = lo >> shift, ihi = hi >> shift;
                for (u32 i = ilo + lane; i <= ihi; i += 32) {
                    const u32 slo = i << shift, shi = ((i + 1) << shift) - 1;
                    u32 val = Lv[i];
                    if (nb > 1 && slo <= full_hi && shi >= lo) val = max(val, res_full);
                    if (slo <= hi && shi >= hi) val = max(val, res_last);
                    Lv[i] = static_cast<unsigned short>(val > kSat ? kSat : val);
                }
                __syncwarp();
            };
            raise(L1, 5);
            raise(L2, 10);
            raise(L3, 15);
            rmax = max(rmax, min(kSat, max(nb > 1 ? res_full : 0u, res_last)));
            B += nb;
        }
        if (prof) pc[3] += clock64() - t0;
        __syncwarp();
    }
    if (lane == 0) {
        a.out[0] = B;
        a.out[1] = nrec;
        a.out[2] = (overflow || nrec > a.max_records) ? 1u : 0u;
        if (prof)
            for (int i = 0; i < 8; ++i) a.prof[i] = pc[i];
    }
}

__global__ void k_expand(FitRecords rec, const u32* __restrict__ nrec_p, u64 n_items, u32* __restrict__ item_bin,
                         u32* __restrict__ item_slot) {
    const u32 nrec = *nrec_p;
    for (u64 j = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; j < n_items;
         j += static_cast<u64>(gridDim.x) * blockDim.x) {
        // last record with item <= j
        u32 lo = 0, hi = nrec;
        while (lo < hi) {
            const u32 mid = (lo + hi) >> 1;
            if (rec.item[mid] <= j) lo = mid + 1;
            else hi = mid;
        }
        u32 b = kNone, sl = kNone;
        if (lo > 0) {
            const u32 r = lo - 1;
            const u64 off = j - rec.item[r];
            if (off < rec.count[r]) {
                const u32 per = rec.per_bin[r];
                b = rec.bin[r] + static_cast<u32>(off / per);
                sl = rec.slot0[r] + static_cast<u32>(off % per);
            }
        }
        item_bin[j] = b;
        item_slot[j] = sl;
    }
}

// ---------------------------------------------------------------------------
// Fill mode, consuming runs in parallel.
//
// While no length runs out, greedy fill is bin-independent: a pack with
// residual r takes floor(r / L) samples of the largest pool length L <= r,
// then continues with r mod L, and so on. Every pack computes that
// trajectory on its own thread against the remaining runs; per run, the
// demand is compared with the run's count. Runs before the first
// over-subscribed ("scarce") run are exact and committed in parallel:
// records sorted (run, pack) give each pick its item offset. The scarce
// region goes to the sequential engine, then the next parallel pass starts.
// ---------------------------------------------------------------------------

// first run index in [lo, hi) with run_len <= r (run_len is decreasing)
__device__ __forceinline__ u32 first_run_le(const u32* __restrict__ run_len, u32 lo, u32 hi, u32 r) {
    while (lo < hi) {
        const u32 mid = (lo + hi) >> 1;
        if (run_len[mid] <= r) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

template <bool EMIT>
__global__ void k_traj(const u64* __restrict__ leaves, u32 P, const u32* __restrict__ run_len, u32 pos, u32 n_runs,
                       u32* __restrict__ npick, const u64* __restrict__ off, u32* __restrict__ r_run,
                       u32* __restrict__ r_take, u32* __restrict__ r_slot0, u32* __restrict__ r_after,
                       unsigned long long* __restrict__ demand) {
    for (u32 b = blockIdx.x * blockDim.x + threadIdx.x; b < P; b += gridDim.x * blockDim.x) {
        const u64 leaf = leaves[b];
        u32 r = static_cast<u32>(leaf >> 32);
        u32 cnt = static_cast<u32>(leaf);
        u32 k = pos, n = 0;
        u64 o = EMIT ? off[b] : 0;
        while (r > 0) {
            k = first_run_le(run_len, k, n_runs, r);
            if (k >= n_runs) break;
            const u32 L = run_len[k];
            const u32 t = r / L;
            r -= t * L;
            if (EMIT) {
                r_run[o + n] = k;
                r_take[o + n] = t;
                r_slot0[o + n] = cnt;
                r_after[o + n] = r;
                atomicAdd(&demand[k], static_cast<unsigned long long>(t));
            }
            cnt += t;
            ++n;
            ++k;
        }
        if (!EMIT) npick[b] = n;
    }
}

__global__ void k_scarce(const unsigned long long* __restrict__ demand, const u32* __restrict__ run_item, u32 pos,
                         u32 n_runs, u32 n_items, u8* __restrict__ scarce, u32* __restrict__ kstar) {
    for (u32 k = pos + blockIdx.x * blockDim.x + threadIdx.x; k < n_runs; k += gridDim.x * blockDim.x) {
        const u32 count = (k + 1 < n_runs ? run_item[k + 1] : n_items) - run_item[k];
        const bool sc = demand[k] > count;
        scarce[k] = sc;
        if (sc) atomicMin(kstar, k);
    }
}

// bin-major records: valid = run < kstar; a pack's last valid record
// carries its final state into the leaf
__global__ void k_traj_commit_leaves(u32 P, const u64* __restrict__ off, const u32* __restrict__ npick,
                                     const u32* __restrict__ r_run, const u32* __restrict__ r_take,
                                     const u32* __restrict__ r_slot0, const u32* __restrict__ r_after,
                                     const u32* __restrict__ kstar_p, u64* __restrict__ leaves,
                                     u32* __restrict__ sort_key, u32 n_runs) {
    const u32 kstar = *kstar_p;
    for (u32 b = blockIdx.x * blockDim.x + threadIdx.x; b < P; b += gridDim.x * blockDim.x) {
        const u64 o = off[b];
        const u32 n = npick[b];
        u32 last = kNone;
        for (u32 i = 0; i < n; ++i) {
            const bool valid = r_run[o + i] < kstar;
            sort_key[o + i] = valid ? r_run[o + i] : n_runs;
            if (valid) last = i;
        }
        if (last != kNone)
            leaves[b] = (static_cast<u64>(r_after[o + last]) << 32) | (r_slot0[o + last] + r_take[o + last]);
    }
}

__device__ __forceinline__ u32 bin_of_record(const u64* __restrict__ off, u32 P, u64 i) {
    // last pack b with off[b] <= i
    u32 lo = 0, hi = P;
    while (lo + 1 < hi) {
        const u32 mid = (lo + hi) >> 1;
        if (off[mid] <= i) lo = mid;
        else hi = mid;
    }
    return lo;
}

__global__ void k_traj_first_of_run(const u32* __restrict__ sorted_idx, const u32* __restrict__ r_run, u64 V,
                                    const u64* __restrict__ take_scan, u64* __restrict__ run_base) {
    for (u64 j = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; j < V;
         j += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u32 run = r_run[sorted_idx[j]];
        if (j == 0 || r_run[sorted_idx[j - 1]] != run) run_base[run] = take_scan[j];
    }
}

__global__ void k_traj_records(const u32* __restrict__ sorted_idx, u64 V, const u64* __restrict__ off, u32 P,
                               const u32* __restrict__ r_run, const u32* __restrict__ r_take,
                               const u32* __restrict__ r_slot0, const u64* __restrict__ take_scan,
                               const u64* __restrict__ run_base, const u32* __restrict__ run_item, FitRecords rec,
                               u32 rec_base) {
    for (u64 j = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; j < V;
         j += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u32 i = sorted_idx[j];
        const u32 run = r_run[i];
        const u32 t = r_take[i];
        const u64 r = rec_base + j;
        rec.item[r] = run_item[run] + static_cast<u32>(take_scan[j] - run_base[run]);
        rec.count[r] = t;
        rec.bin[r] = bin_of_record(off, P, i);
        rec.per_bin[r] = t;
        rec.slot0[r] = r_slot0[i];
    }
}

}  // namespace

// One parallel pass from run `pos`: commits every run before the first
// scarce one; returns that run index (n_runs when none) and the scarce flags.
static u32 fill_parallel_pass(Ctx& c, u64* leaves, u32 P, const u32* run_len, const u32* run_item, u32 pos,
                              u32 n_runs, u32 n_items, FitRecords rec, u32& nrec, u32 max_records,
                              std::vector<u8>& scarce_host) {
    cudaStream_t s = c.stream;
    DevBuf<u32> npick(P + 1, s);
    DevBuf<u64> off(P + 1, s);
    LAUNCH(k_traj<false>, grid_for(P, 256, 148u * 16u), 256, 0, s, leaves, P, run_len, pos, n_runs, npick.p, nullptr,
           nullptr, nullptr, nullptr, nullptr, nullptr);
    {
        const u32* np = npick.p;
        u64* op = off.p;
        const i64 PP = P;
        scan_exclusive<u64>(
            PP + 1, [=] __device__(i64 i) { return i < PP ? static_cast<u64>(np[i]) : 0ull; },
            [=] __device__(i64 i, u64 v) { op[i] = v; }, s, c.scan, "scan.ff1");
    }
    const u64 R = read_vector(c, off.p + P, 1)[0];
    DevBuf<unsigned long long> demand(n_runs + 1, s);
    demand.zero();
    DevBuf<u32> r_run(R + 1, s), r_take(R + 1, s), r_slot0(R + 1, s), r_after(R + 1, s);
    if (R > 0)
        LAUNCH(k_traj<true>, grid_for(P, 256, 148u * 16u), 256, 0, s, leaves, P, run_len, pos, n_runs, npick.p, off.p,
               r_run.p, r_take.p, r_slot0.p, r_after.p, demand.p);
    DevBuf<u8> scarce(n_runs + 1, s);
    DevBuf<u32> kstar(1, s);
    CUDA_CHECK(cudaMemcpyAsync(kstar.p, &n_runs, 4, cudaMemcpyHostToDevice, s));
    LAUNCH(k_scarce, grid_for(n_runs - pos, 256, 148u * 16u), 256, 0, s, demand.p, run_item, pos, n_runs, n_items,
           scarce.p, kstar.p);
    const u32 ks = read_scalar(c, kstar.p);
    scarce_host.assign(n_runs, 0);
    if (n_runs > pos)
        CUDA_CHECK(cudaMemcpyAsync(scarce_host.data() + pos, scarce.p + pos, n_runs - pos, cudaMemcpyDeviceToHost, s));
    if (ks == pos || R == 0) {
        CUDA_CHECK(cudaStreamSynchronize(s));
        return ks;
    }
    // commit runs [pos, ks)
    DevBuf<u32> key(R, s), idx(R, s);
    LAUNCH(k_traj_commit_leaves, grid_for(P, 256, 148u * 16u), 256, 0, s, P, off.p, npick.p, r_run.p, r_take.p,
           r_slot0.p, r_after.p, kstar.p, leaves, key.p, n_runs);
    for_each_index(c, R, [ip = idx.p] __device__(u64 i) { ip[i] = static_cast<u32>(i); });
    int bits = 1;
    while (bits < 32 && (static_cast<u64>(n_runs) >> bits) != 0) ++bits;
    radix_sort_pairs(c, key.p, idx.p, static_cast<i64>(R), bits, false);
    // valid records are the prefix with key < ks
    DevBuf<u64> take_scan(R + 1, s), run_base(n_runs + 1, s), vcount(1, s);
    vcount.zero();  // stays 0 when no record belongs to a committed run
    {
        const u32* kp = key.p;
        const u32* ip = idx.p;
        const u32* tp = r_take.p;
        u64* sp = take_scan.p;
        u64* vc = vcount.p;
        const i64 RR = static_cast<i64>(R);
        const u32 kk = ks;
        scan_exclusive<u64>(
            RR, [=] __device__(i64 j) { return kp[j] < kk ? static_cast<u64>(tp[ip[j]]) : 0ull; },
            [=] __device__(i64 j, u64 v) {
                sp[j] = v;
                if (kp[j] < kk && (j == RR - 1 || kp[j + 1] >= kk)) *vc = static_cast<u64>(j + 1);
            },
            s, c.scan, "scan.ff2");
    }
    const u64 V = read_scalar(c, vcount.p);
    if (V > 0) {
        if (nrec + V > max_records) throw EngineError(HBP_ERR_CUDA, "fill: record capacity exceeded");
        LAUNCH(k_traj_first_of_run, grid_for(V, 256, 148u * 16u), 256, 0, s, idx.p, r_run.p, V, take_scan.p,
               run_base.p);
        LAUNCH(k_traj_records, grid_for(V, 256, 148u * 16u), 256, 0, s, idx.p, V, off.p, P, r_run.p, r_take.p,
               r_slot0.p, take_scan.p, run_base.p, run_item, rec, nrec);
        nrec += static_cast<u32>(V);
    }
    CUDA_CHECK(cudaStreamSynchronize(s));
    return ks;
}

// FFD's shape from its runs: [0] runs, [1] the first run no longer than
// cap / 2 (with bulk; the runs before it each hold items that never share
// a bin), [3] the items' total length; k_ffd_bulk then writes [2] = the
// item that run starts at (the bulk-placed items before it).
__global__ void k_ffd_shape(const u32* __restrict__ run_len, const u32* __restrict__ run_item,
                            const u32* __restrict__ n_runs_p, u64 n, u32 cap, bool bulk,
                            unsigned long long* __restrict__ out) {
    const u32 nr = *n_runs_p;
    unsigned long long sum = 0, first_short = ~0ull;
    for (u64 k = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; k < nr;
         k += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u64 len = run_len[k] & 0x7fffffffu;
        const u64 e = k + 1 < nr ? run_item[k + 1] : n;
        sum += len * (e - run_item[k]);
        if (bulk && 2ull * len <= cap && k < first_short) first_short = k;
    }
    sum = warp_sum(sum);
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, first_short, o);
        first_short = t < first_short ? t : first_short;
    }
    if ((threadIdx.x & 31u) == 0) {
        if (sum) atomicAdd(out + 3, sum);
        if (first_short != ~0ull) atomicMin(out + 1, first_short);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = nr;
}

__global__ void k_ffd_bulk(const u32* __restrict__ run_item, u64 n, bool bulk, unsigned long long* __restrict__ out) {
    const u64 nr = out[0];
    const u64 rb = bulk ? (out[1] < nr ? out[1] : nr) : 0;
    out[1] = rb;
    out[2] = rb == 0 ? 0 : (rb < nr ? run_item[rb] : n);
}

void prepare_runs(Ctx& c, const u64* items, i64 n_items, const u32* key32, u64 neg_keys, FitRuns r) {
    if (n_items <= 0) return;
    u32* ri = r.run_item;
    u32* rl = r.run_len;
    u32* sc = r.n_runs;
    const i64 nn = n_items;
    // one scan over run-head flags; each head writes its run's first item
    // and length (bit 31: strict) at its run index
    auto store = [=] __device__(i64 i, u32 v, u32 x) {
        const bool head = x != 0;
        if (head) {
            const bool strict = neg_keys && neg_item(items[i], key32, neg_keys);
            ri[v] = static_cast<u32>(i);
            rl[v] = entry_len(items[i]) | (strict ? 0x80000000u : 0u);
        }
        if (i == nn - 1) sc[0] = v + (head ? 1u : 0u);
    };
    if (neg_keys == 0) {
        // lengths only: a branch-free flag, so the tile's loads are issued
        // together (the id-class test below kept them one item at a time:
        // 9.8M items 115 us)
        scan_exclusive_v<u32>(
            nn,
            [=] __device__(i64 i) {
                const u64 e = items[i], p = items[i > 0 ? i - 1 : 0];
                return (i == 0 || entry_len(e) != entry_len(p)) ? 1u : 0u;
            },
            store, c.stream, c.scan, "scan.ff3", 8.0);
    } else {
        scan_exclusive_v<u32>(
            nn,
            [=] __device__(i64 i) {
                const u64 e = items[i], p = items[i > 0 ? i - 1 : 0];
                bool head = i == 0 || entry_len(e) != entry_len(p);
                if (!head) head = neg_item(e, key32, neg_keys) != neg_item(p, key32, neg_keys);
                return head ? 1u : 0u;
            },
            store, c.stream, c.scan, "scan.ff3", 8.0);
    }
}

FitResult first_fit_runs(Ctx& c, const u64* items, i64 n_items_s, u64* leaves, i64 bins0, i64 max_bins, u32 cap,
                         FitMode mode, u32* item_bin, u32* item_slot, const u32* key32, u64 neg_keys,
                         const FitRuns* pre) {
    FitResult out;
    out.bins = bins0;
    if (n_items_s <= 0) return out;
    const u64 n = static_cast<u64>(n_items_s);
    cudaStream_t s = c.stream;
    const bool ffd = mode == FitMode::Ffd;
    if (max_bins < 1) max_bins = 1;
    const char* eng = std::getenv("HBP_ENGINE");
    const std::string engine = eng ? eng : "";
    const bool use_chain = engine.empty() || engine == "chain";
    if (mode == FitMode::Ffd) neg_keys = 0;  // first_fit compares totals, no probe quirk
    if (neg_keys > 0 && !use_chain)
        throw EngineError(HBP_ERR_CUDA, "greedy fill with sample ids <= -2 needs the chain engine (HBP_ENGINE)");

    // runs of equal length (or precomputed by the caller with the same key rules)
    DevBuf<u32> run_item, run_len, scal;
    FitRuns fr;
    if (pre) {
        fr = *pre;
    } else {
        run_item.alloc(n, s);
        run_len.alloc(n, s);
        scal.alloc(4, s);
        fr = FitRuns{run_item.p, run_len.p, scal.p};
        prepare_runs(c, items, static_cast<i64>(n), key32, neg_keys, fr);
    }

    // bulk-place the items that can never share a bin (FFD with no live bins)
    u32 bulk = 0;
    u32 run_begin = 0;
    u32 n_runs = 0;
    // First fit never leaves two bins at most half full (the later bin's
    // first item would have fitted the earlier), so FFD opens at most
    // 2 * ceil(sum / cap) + 1 bins: size the tree by that, not by n.
    i64 tree_bins = max_bins;
    i64 est_bins = 0;
    if (ffd) {
        // the runs' count, the leading runs longer than cap / 2 (sorted
        // decreasing: a prefix) with their items, and the items' total
        // length, on the device and in one read
        DevBuf<unsigned long long> shape(4, s);
        shape.zero();
        CUDA_CHECK(cudaMemsetAsync(shape.p + 1, 0xff, sizeof(unsigned long long), s));  // first short run: none yet
        LAUNCH(k_ffd_shape, grid_for(n, 256, 148u * 4u), 256, 0, s, fr.run_len, fr.run_item, fr.n_runs, n, cap,
               bins0 == 0, shape.p);
        LAUNCH(k_ffd_bulk, 1, 1, 0, s, fr.run_item, n, bins0 == 0, shape.p);
        const auto h = read_vector(c, shape.p, 4);
        n_runs = static_cast<u32>(h[0]);
        run_begin = static_cast<u32>(h[1]);
        bulk = static_cast<u32>(h[2]);
        const long double sum = static_cast<long double>(h[3]);
        const i64 bound = static_cast<i64>(2 * std::ceil(sum / cap)) + 2 + bins0;
        // FFD of sorted items is near the volume bound for small items and
        // one bin per item above cap / 2: first chain pass sized by both
        const long double vol = std::ceil(sum / cap);
        est_bins = static_cast<i64>(std::max<long double>(static_cast<long double>(bins0 + bulk) * 1.02L, vol * 1.02L)) +
                   1024;
        if (bound < tree_bins) tree_bins = bound;
    } else {
        n_runs = read_scalar(c, fr.n_runs);
    }
    const u64 live = static_cast<u64>(bins0) + bulk;
    if (use_chain) {
        DevBuf<u32> take(n, s);
        take.zero();
        // items no take covers stay unassigned (chains without replay skip the expand)
        CUDA_CHECK(cudaMemsetAsync(item_bin, 0xff, sizeof(u32) * n, s));
        if (bulk > 0)
            LAUNCH(k_bulk_big, grid_for(bulk, 256, 148u * 16u), 256, 0, s, items, static_cast<u64>(bulk), cap, leaves,
                   item_bin, item_slot, take.p);
        ChainRuns cr{fr.run_item, fr.run_len, static_cast<u32>(n), n_runs, run_begin, n_runs};
        u32 used = 0;
        if (chain_fit(c, cr, leaves, static_cast<u32>(live), static_cast<u32>(ffd ? tree_bins : live), cap, ffd,
                      item_bin, item_slot, take.p, static_cast<u32>(std::min<i64>(est_bins, tree_bins)), used)) {
            out.bins = ffd ? std::max<i64>(static_cast<i64>(live), used) : bins0;
            return out;
        }
    }
    const u64 max_records = 2 * n + 2;
    DevBuf<u32> r_item(max_records, s), r_count(max_records, s), r_bin(max_records, s), r_per(max_records, s),
        r_slot0(max_records, s);
    FitRecords rec{r_item.p, r_count.p, r_bin.p, r_per.p, r_slot0.p};
    TreeLayout t = make_layout(static_cast<u64>(tree_bins));
    DevBuf<u32> tree(t.off[0], s);
    t.base = tree.p;
    if (bulk > 0) {
        LAUNCH(k_bulk_big, grid_for(bulk, 256, 148u * 16u), 256, 0, s, items, static_cast<u64>(bulk), cap, leaves,
               nullptr, nullptr, nullptr);
    }
    // leaves beyond the live ones start empty
    if (static_cast<u64>(max_bins) > live)
        CUDA_CHECK(cudaMemsetAsync(leaves + live, 0, sizeof(u64) * (max_bins - live), s));
    CUDA_CHECK(cudaMemsetAsync(tree.p, 0, sizeof(u32) * t.off[0], s));
    for (int h = 1; h <= t.H; ++h) {
        const u64 hi = (live + (1ull << (5 * h)) - 1) >> (5 * h);
        if (hi == 0) break;
        LAUNCH(k_tree_level, grid_for(hi, 256, 148u * 16u), 256, 0, s, leaves, tree.p, t, h, 0ull, hi);
    }
    u32 rec0 = 0;
    if (bulk > 0) {
        // one record covers the bulk: item i -> bin i
        const u32 one[5] = {0u, bulk, 0u, 1u, 0u};
        CUDA_CHECK(cudaMemcpyAsync(rec.item, &one[0], 4, cudaMemcpyHostToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(rec.count, &one[1], 4, cudaMemcpyHostToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(rec.bin, &one[2], 4, cudaMemcpyHostToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(rec.per_bin, &one[3], 4, cudaMemcpyHostToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(rec.slot0, &one[4], 4, cudaMemcpyHostToDevice, s));
        CUDA_CHECK(cudaStreamSynchronize(s));  // `one` is a stack buffer
        rec0 = 1;
    }
    EngineArgs a;
    a.items = items;
    a.n_items = static_cast<u32>(n);
    a.run_item = fr.run_item;
    a.run_len = fr.run_len;
    a.n_runs = n_runs;
    a.run_begin = run_begin;
    a.leaves = leaves;
    a.t = t;
    a.bins0 = static_cast<u32>(live);
    a.max_bins = static_cast<u32>(tree_bins);
    a.cap = cap;
    a.ffd = ffd ? 1 : 0;
    a.rec = rec;
    a.rec0 = rec0;
    a.max_records = static_cast<u32>(max_records);
    a.out = fr.n_runs;
    DevBuf<unsigned long long> prof;
    a.prof = nullptr;
    if (c.trace) {
        prof.alloc(8, s);
        prof.zero();
        a.prof = prof.p;
    }
    const size_t smem = sizeof(unsigned short) * t.off[0];
    constexpr size_t kSmemLimit = 216 * 1024;  // + 8.4 KB static (candidates, leaf stage) <= 227 KB
    const V4Layout vl = make_v4(static_cast<u64>(tree_bins));
    const size_t smem4 = sizeof(unsigned short) * vl.total;
    const bool force_v3 = engine == "v3", force_v1 = engine == "v1";
    cudaFuncAttributes fa4{};
    CUDA_CHECK(cudaFuncGetAttributes(&fa4, k_fit_engine_v4));
    const size_t limit4 = 227 * 1024 - fa4.sharedSizeBytes;  // dynamic + static <= 227 KB per CTA
    const bool v4ok = vl.n3 <= 128 && smem4 <= limit4 && !force_v3 && !force_v1;
    a.run_end = n_runs;
    if (v4ok && !ffd && !std::getenv("HBP_NO_HYBRID")) {
        // fill: parallel passes over the non-scarce runs, the engine over
        // each scarce cluster (runs within kGap of a scarce run)
        constexpr u32 kGap = 64;
        CUDA_CHECK(cudaFuncSetAttribute(k_fit_engine_v4, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(limit4)));
        const u32 P = static_cast<u32>(live);
        u32 nrec = rec0, pos = run_begin, passes = 0, engine_runs = 0;
        // a pass costs about as much as the engine on ~kGap / 2 runs: when
        // passes stop paying (few runs committed), hand the engine
        // exponentially longer stretches
        u32 stretch = kGap;
        std::vector<u8> scarce;
        while (pos < n_runs) {
            const u32 ks = fill_parallel_pass(c, leaves, P, fr.run_len, fr.run_item, pos, n_runs, static_cast<u32>(n),
                                              rec, nrec, static_cast<u32>(max_records), scarce);
            ++passes;
            if (ks >= n_runs) break;
            if (ks - pos < kGap / 2) stretch = stretch * 2 < n_runs ? stretch * 2 : n_runs;
            else stretch = kGap;
            u32 last = ks;
            for (u32 k = ks + 1; k < n_runs && k - last <= kGap; ++k)
                if (scarce[k]) last = k;
            u32 end = last + 1;
            if (end - ks < stretch) end = ks + stretch < n_runs ? ks + stretch : n_runs;
            CUDA_CHECK(cudaMemsetAsync(tree.p, 0, sizeof(u32) * t.off[0], s));
            for (int h = 1; h <= t.H; ++h) {
                const u64 hi = (live + (1ull << (5 * h)) - 1) >> (5 * h);
                if (hi == 0) break;
                LAUNCH(k_tree_level, grid_for(hi, 256, 148u * 16u), 256, 0, s, leaves, tree.p, t, h, 0ull, hi);
            }
            a.run_begin = ks;
            a.run_end = end;
            a.rec0 = nrec;
            LAUNCH_B("fit.engine", 0.0, k_fit_engine_v4, 1, 32, smem4, s, a, vl);
            const auto o = read_vector(c, fr.n_runs, 3);
            if (o[2]) throw EngineError(HBP_ERR_CUDA, "first-fit engine: record or bin capacity exceeded");
            nrec = o[1];
            engine_runs += end - ks;
            pos = end;
        }
        if (c.trace)
            std::fprintf(stderr, "[hbp trace] fit fill (hybrid): runs %u bins %u passes %u engine runs %u records %u\n",
                         n_runs, P, passes, engine_runs, nrec);
        out.bins = live;
        out.records = nrec;
        expand_fit_records(c, rec, out.records, static_cast<i64>(n), item_bin, item_slot);
        return out;
    }
    if (v4ok) {
        CUDA_CHECK(cudaFuncSetAttribute(k_fit_engine_v4, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(limit4)));
        LAUNCH_B("fit.engine", 0.0, k_fit_engine_v4, 1, 32, smem4, s, a, vl);
    } else if (smem <= kSmemLimit && !force_v1) {
        CUDA_CHECK(cudaFuncSetAttribute(k_fit_engine_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kSmemLimit)));
        LAUNCH_B("fit.engine", 0.0, k_fit_engine_smem, 1, 32, smem, s, a);
    } else {
        LAUNCH_B("fit.engine.v1", 0.0, k_fit_engine, 1, 32, 0, s, a);
    }
    const auto o = read_vector(c, fr.n_runs, 3);
    if (o[2]) throw EngineError(HBP_ERR_CUDA, "first-fit engine: record or bin capacity exceeded");
    if (c.trace) {
        const auto pc = read_vector(c, prof.p, 8);
        std::fprintf(stderr,
                     "[hbp trace] fit %s: runs %u (from %u) bins %u tree_bins %lld H %d | collect %.2fM load %.2fM "
                     "process %.2fM newbins %.2fM cycles | searched %llu cands %llu rounds %llu misses %llu\n",
                     ffd ? "ffd" : "fill", n_runs, run_begin, o[0], static_cast<long long>(tree_bins), t.H,
                     pc[0] / 1e6, pc[1] / 1e6, pc[2] / 1e6, pc[3] / 1e6, pc[4], pc[5], pc[6], pc[7]);
    }
    out.bins = o[0];
    out.records = o[1];
    expand_fit_records(c, rec, out.records, static_cast<i64>(n), item_bin, item_slot);
    return out;
}

void expand_fit_records(Ctx& c, FitRecords rec, i64 n_records, i64 n_items, u32* item_bin, u32* item_slot) {
    if (n_items <= 0) return;
    DevBuf<u32> nrec(1, c.stream);
    const u32 nr = static_cast<u32>(n_records);
    CUDA_CHECK(cudaMemcpyAsync(nrec.p, &nr, 4, cudaMemcpyHostToDevice, c.stream));
    LAUNCH(k_expand, grid_for(n_items, 256, 148u * 16u), 256, 0, c.stream, rec, nrec.p, static_cast<u64>(n_items),
           item_bin, item_slot);
    CUDA_CHECK(cudaStreamSynchronize(c.stream));  // nr lives on the host stack
}

}  // namespace hbp_b200
