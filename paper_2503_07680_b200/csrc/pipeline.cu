// pipeline.cu — build_plan on the GPU (reference src/balance.cpp:207-258).
//
//   ingest      SampleSet::validate (types.cpp:8-24) + lengths to u32
//   group_data  stable partition by group (balance.cpp:25-44): one radix pass
//   per group, largest first:
//     pack      ISF rounds (shuffle.cu + nextfit.cu), residue FFD (firstfit.cu)
//     fill      greedy_fill from the smaller pools (firstfit.cu, fill mode)
//     layout    members of every pack contiguous; totals and Σ L²
//     batching  stable attention sort + chunks of N, spill tail (balance.cpp:105-192)
//   plan shuffle (balance.cpp:255-256) and CSR output.
// The host only synchronises for data-dependent sizes (pool sizes per ISF
// round, pack counts, record counts); all data stays in HBM.
#include <algorithm>
#include <cmath>
#include <numeric>

#include "pipeline.cuh"
#include "radix.cuh"
#include "rng.cuh"

namespace hbp_b200 {

namespace {

constexpr int kB = 256;

inline unsigned G(u64 n) { return grid_for(n, kB, 148u * 16u); }

inline int bits_for(u64 maxval) {
    int b = 1;
    while (b < 32 && (maxval >> b) != 0) ++b;
    return b;
}

#define GRID_STRIDE(i, n) \
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < (n); i += static_cast<u64>(gridDim.x) * blockDim.x)

// Grid-stride loop in two phases per U elements: every load first (ld(i),
// predicated on i < n), then every store (st(i, v)). A plain grid-stride loop
// keeps one load per thread in flight (its next load waits behind the bound
// check), which held these passes at 1.6-3.7 TB/s.
template <int U, typename Ld, typename St>
__device__ __forceinline__ void grid_stride_2phase(u64 n, Ld ld, St st) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i0 = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i0 < n; i0 += U * stride) {
        decltype(ld(u64{0})) v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const u64 i = i0 + u * stride;
            if (i < n) v[u] = ld(i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const u64 i = i0 + u * stride;
            if (i < n) st(i, v[u]);
        }
    }
}

// ---------------------------------------------------------------------------
// ingest
// ---------------------------------------------------------------------------

struct IngestFlags {
    unsigned long long first_bad_len;  // length < 1
    unsigned long long first_over;     // length > limit
    unsigned long long neg;            // ids <= -2
    unsigned long long not_ascending;
};

__global__ void k_ingest(const int64_t* __restrict__ len64, const int64_t* __restrict__ ids, u64 n, int64_t limit,
                         u32* __restrict__ len32, IngestFlags* __restrict__ f) {
    GRID_STRIDE(i, n) {
        const int64_t L = len64[i];
        if (L < 1) atomicMin(&f->first_bad_len, static_cast<unsigned long long>(i));
        if (L > limit) atomicMin(&f->first_over, static_cast<unsigned long long>(i));
        len32[i] = L < 1 ? 0u : (L > 0x7fffffffLL ? 0x7fffffffu : static_cast<u32>(L));
        if (ids) {
            if (ids[i] <= -2) atomicAdd(&f->neg, 1ull);
            if (i + 1 < n && ids[i] >= ids[i + 1]) f->not_ascending = 1ull;
        }
    }
}

__global__ void k_id_words(const int64_t* __restrict__ ids, const u32* __restrict__ order, u64 n, bool high,
                           u32* __restrict__ out) {
    GRID_STRIDE(i, n) {
        const u64 v = static_cast<u64>(ids[order[i]]) ^ (1ull << 63);  // order-preserving for signed
        out[i] = high ? static_cast<u32>(v >> 32) : static_cast<u32>(v);
    }
}

__global__ void k_iota(u32* __restrict__ a, u64 n) {
    GRID_STRIDE(i, n) a[i] = static_cast<u32>(i);
}

__global__ void k_ranks_dups(const int64_t* __restrict__ ids, const u32* __restrict__ order, u64 n,
                             u32* __restrict__ rank, unsigned long long* __restrict__ first_dup) {
    GRID_STRIDE(r, n) {
        const u32 i = order[r];
        rank[i] = static_cast<u32>(r);
        if (r >= 1 && ids[order[r - 1]] == ids[i]) {
            // the second occurrence (in input order) of an id is the first duplicate seen
            if (r == 1 || ids[order[r - 2]] != ids[i]) atomicMin(first_dup, static_cast<unsigned long long>(i));
        }
    }
}

// ---------------------------------------------------------------------------
// group_data + entries
// ---------------------------------------------------------------------------

// Group of every sample (and group_data's l_max check, balance.cpp:32-36:
// counts[64] <- the first sample longer than lm, in the same read).
__global__ void k_group_keys(const u32* __restrict__ len32, u64 n, const int64_t* __restrict__ glen, int ng, u32 lm,
                             u32* __restrict__ key, u32* __restrict__ val, unsigned long long* __restrict__ counts) {
    __shared__ unsigned long long s_cnt[64];
    for (int g = threadIdx.x; g < 64; g += blockDim.x) s_cnt[g] = 0;
    __syncthreads();
    GRID_STRIDE(i, n) {
        const u32 L = len32[i];
        if (L > lm) atomicMin(&counts[64], static_cast<unsigned long long>(i));
        int g = 0;
        while (g < ng - 1 && static_cast<int64_t>(L) > glen[g]) ++g;
        key[i] = static_cast<u32>(g);
        val[i] = static_cast<u32>(i);
        // one shared atomic per group present in the warp (not per sample:
        // with two groups every lane hits the same counter)
        const unsigned peers = __match_any_sync(__activemask(), g);
        if ((threadIdx.x & 31u) == static_cast<unsigned>(__ffs(peers) - 1))
            atomicAdd(&s_cnt[g < 64 ? g : 63], static_cast<unsigned long long>(__popc(peers)));
    }
    __syncthreads();
    for (int g = threadIdx.x; g < ng && g < 64; g += blockDim.x)
        if (s_cnt[g]) atomicAdd(&counts[g], s_cnt[g]);
}

__global__ void k_entries_from_idx(const u32* __restrict__ len32, const u32* __restrict__ idx, u64 n,
                                   u64* __restrict__ out) {
    grid_stride_2phase<4>(
        n, [&](u64 i) { const u32 j = idx[i]; return make_entry(len32[j], j); },
        [&](u64 i, u64 e) { out[i] = e; });
}

// ---------------------------------------------------------------------------
// entry sorting: (length desc, key asc)
// ---------------------------------------------------------------------------

__global__ void k_keys_of_entries(const u64* __restrict__ e, const u32* __restrict__ key32, u64 n,
                                  u32* __restrict__ k, u32* __restrict__ v) {
    grid_stride_2phase<4>(
        n, [&](u64 i) { const u32 idx = entry_idx(e[i]); return key32 ? key32[idx] : idx; },
        [&](u64 i, u32 key) {
            k[i] = key;
            v[i] = static_cast<u32>(i);
        });
}

__global__ void k_lens_of(const u64* __restrict__ e, const u32* __restrict__ perm, u64 n, u32* __restrict__ k) {
    grid_stride_2phase<4>(n, [&](u64 i) { return entry_len(e[perm[i]]); }, [&](u64 i, u32 l) { k[i] = l; });
}

__global__ void k_gather_entries(const u64* __restrict__ in, const u32* __restrict__ perm, u64 n,
                                 u64* __restrict__ out) {
    grid_stride_2phase<4>(n, [&](u64 i) { return in[perm[i]]; }, [&](u64 i, u64 x) { out[i] = x; });
}

// ---------------------------------------------------------------------------
// pack layout, fill, stats
// ---------------------------------------------------------------------------

__global__ void k_isf_leaves(const u64* __restrict__ pack_off, const u32* __restrict__ pack_total, u64 np,
                             u64 n_members, u32 cap, u64* __restrict__ leaves) {
    GRID_STRIDE(p, np) {
        const u64 end = (p + 1 < np) ? pack_off[p + 1] : n_members;
        const u64 size = end - pack_off[p];
        leaves[p] = (static_cast<u64>(cap - pack_total[p]) << 32) | static_cast<u32>(size);
    }
}

__global__ void k_mark_consumed(const u64* __restrict__ items, const u32* __restrict__ item_bin, u64 n,
                                u8* __restrict__ consumed) {
    grid_stride_2phase<4>(
        n, [&](u64 i) { return item_bin[i] != kNone ? entry_idx(items[i]) : kNone; },
        [&](u64, u32 ix) {
            if (ix != kNone) consumed[ix] = 1;
        });
}

__global__ void k_place_isf(const u64* __restrict__ sink_members, const u64* __restrict__ pack_off, u64 np,
                            u64 n_members, const u64* __restrict__ out_off, u64* __restrict__ out) {
    // eight lanes per pack (packs hold ~10 members): four packs per warp
    const u64 groups = (static_cast<u64>(gridDim.x) * blockDim.x) >> 3;
    const u32 sub = threadIdx.x & 7u;
    for (u64 p = (blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x) >> 3; p < np; p += groups) {
        const u64 a = pack_off[p];
        const u64 b = (p + 1 < np) ? pack_off[p + 1] : n_members;
        const u64 d = out_off[p];
        for (u64 k = a + sub; k < b; k += 8) out[d + (k - a)] = sink_members[k];
    }
}

__global__ void k_place_items(const u64* __restrict__ items, const u32* __restrict__ item_bin,
                              const u32* __restrict__ item_slot, u64 n, u64 bin_base,
                              const u64* __restrict__ out_off, u64* __restrict__ out) {
    struct Item {
        u64 dst, v;
    };
    grid_stride_2phase<4>(
        n,
        [&](u64 i) {
            const u32 b = item_bin[i];
            return b != kNone ? Item{out_off[bin_base + b] + item_slot[i], items[i]} : Item{~0ull, 0};
        },
        [&](u64, Item it) {
            if (it.dst != ~0ull) out[it.dst] = it.v;
        });
}

__global__ void k_pack_stats(const u64* __restrict__ members, const u64* __restrict__ off, u64 np, u64 mbase,
                             u64 pbase, u32 cap, u64* __restrict__ g_moff, u32* __restrict__ g_cnt,
                             u32* __restrict__ g_cap, u32* __restrict__ g_total, u64* __restrict__ g_att) {
    GRID_STRIDE(p, np) {
        const u64 a = off[p], b = off[p + 1];
        u64 tot = 0, att = 0;
        for (u64 k = a; k < b; ++k) {
            const u64 l = entry_len(members[k]);
            tot += l;
            att += l * l;
        }
        g_moff[pbase + p] = mbase + a;
        g_cnt[pbase + p] = static_cast<u32>(b - a);
        g_cap[pbase + p] = cap;
        g_total[pbase + p] = static_cast<u32>(tot);
        g_att[pbase + p] = att;
    }
}

// ---------------------------------------------------------------------------
// batching
// ---------------------------------------------------------------------------

__global__ void k_att_words(const u64* __restrict__ att, const u32* __restrict__ perm, u64 n, bool high,
                            u32* __restrict__ out) {
    GRID_STRIDE(i, n) {
        const u64 v = att[perm[i]];
        out[i] = high ? static_cast<u32>(v >> 32) : static_cast<u32>(v);
    }
}

__global__ void k_full_iterations(const u32* __restrict__ order, u64 nfull, u32 N, u32 pbase, int gi, u64 ibase,
                                  u32* __restrict__ slots, int32_t* __restrict__ igroup) {
    GRID_STRIDE(x, nfull * N) {
        const u64 k = x / N;
        slots[(ibase + k) * N + (x % N)] = pbase + order[x];
        if (x % N == 0) igroup[ibase + k] = gi;
    }
}

// Spill tail (balance.cpp:121-151): samples sorted (length desc, id asc)
// go one by one to the device with the least attention that still fits
// (lowest device on ties); unpadded capacity; fallback keeps the packs.
// device_count > 256: one thread (the warp version keeps 8 devices per lane)
__global__ void k_spill_serial(const u64* __restrict__ sorted, u64 k, u32 N, u32 cap, const u32* __restrict__ tail_packs,
                        u32 rem, u32 spill_pbase, u64 spill_mbase, int gi, u64 iter, u64* __restrict__ g_members,
                        u64* __restrict__ g_moff, u32* __restrict__ g_cnt, u32* __restrict__ g_cap,
                        u32* __restrict__ g_total, u64* __restrict__ g_att, u32* __restrict__ dev_of,
                        u32* __restrict__ slots, int32_t* __restrict__ igroup) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    // device totals / attention in registers of one thread (N small)
    bool ok = true;
    for (u32 d = 0; d < N; ++d) {
        g_total[spill_pbase + d] = 0;
        g_att[spill_pbase + d] = 0;
        g_cnt[spill_pbase + d] = 0;
    }
    for (u64 i = 0; i < k; ++i) {
        const u32 L = entry_len(sorted[i]);
        u32 target = N;
        u64 best = 0;
        for (u32 d = 0; d < N; ++d) {
            if (cap - g_total[spill_pbase + d] < L) continue;
            const u64 a = g_att[spill_pbase + d];
            if (target == N || a < best) {
                target = d;
                best = a;
            }
        }
        if (target == N) {
            ok = false;
            break;
        }
        dev_of[i] = target;
        g_total[spill_pbase + target] += L;
        g_att[spill_pbase + target] += static_cast<u64>(L) * L;
        g_cnt[spill_pbase + target] += 1;
    }
    igroup[iter] = gi;
    if (ok) {
        // members grouped by device, in assignment order
        u64 off = spill_mbase;
        for (u32 d = 0; d < N; ++d) {
            g_moff[spill_pbase + d] = off;
            off += g_cnt[spill_pbase + d];
            g_cap[spill_pbase + d] = g_total[spill_pbase + d];
        }
        for (u32 d = 0; d < N; ++d) g_cnt[spill_pbase + d] = 0;
        for (u64 i = 0; i < k; ++i) {
            const u32 d = dev_of[i];
            g_members[g_moff[spill_pbase + d] + g_cnt[spill_pbase + d]++] = sorted[i];
        }
        for (u32 d = 0; d < N; ++d) slots[iter * N + d] = g_cnt[spill_pbase + d] ? spill_pbase + d : kNone;
    } else {
        for (u32 d = 0; d < N; ++d) slots[iter * N + d] = d < rem ? tail_packs[d] : kNone;
    }
}

// One warp: device d's running total / attention live in lane d % 32 (slot
// d / 32), so each sample is one warp argmin over (attention, device) among
// the devices it fits -- no dependent global memory on the sample loop.
constexpr u32 kSpillSlots = 8;  // devices per lane: device_count <= 256 on this path
template <u32 kSlots>
__global__ void k_spill(const u64* __restrict__ sorted, u64 k, u32 N, u32 cap, const u32* __restrict__ tail_packs,
                        u32 rem, u32 spill_pbase, u64 spill_mbase, int gi, u64 iter, u64* __restrict__ g_members,
                        u64* __restrict__ g_moff, u32* __restrict__ g_cnt, u32* __restrict__ g_cap,
                        u32* __restrict__ g_total, u64* __restrict__ g_att, u32* __restrict__ dev_of,
                        u32* __restrict__ slots, int32_t* __restrict__ igroup) {
    if (blockIdx.x != 0 || threadIdx.x >= 32) return;
    const u32 lane = threadIdx.x;
    u32 tot[kSlots], cnt[kSlots];
    u64 att[kSlots];
#pragma unroll
    for (u32 q = 0; q < kSlots; ++q) {
        tot[q] = 0;
        cnt[q] = 0;
        att[q] = 0;
    }
    bool ok = true;
    u32 chunk = 0;  // lengths of items [i & ~31, +32), one per lane, loaded together
    for (u64 i = 0; i < k; ++i) {
        if ((i & 31u) == 0) chunk = i + lane < k ? entry_len(sorted[i + lane]) : 0u;
        const u32 L = __shfl_sync(0xffffffffu, chunk, static_cast<int>(i & 31u));
        // this lane's best fitting device (least attention, lowest index)
        u64 ba = ~0ull;
        u32 bd = 0xffffffffu;
#pragma unroll
        for (u32 q = 0; q < kSlots; ++q) {
            const u32 d = q * 32 + lane;
            if (d < N && cap - tot[q] >= L && (att[q] < ba || (att[q] == ba && d < bd))) {
                ba = att[q];
                bd = d;
            }
        }
        // warp argmin of (attention, device): three REDUX steps (high word,
        // low word, device) instead of five shuffle rounds on the item's path
        {
            const u32 h = static_cast<u32>(ba >> 32);
            const u32 mh = __reduce_min_sync(0xffffffffu, h);
            const u32 l = h == mh ? static_cast<u32>(ba) : 0xffffffffu;
            const u32 ml = __reduce_min_sync(0xffffffffu, l);
            bd = __reduce_min_sync(0xffffffffu, h == mh && static_cast<u32>(ba) == ml ? bd : 0xffffffffu);
        }
        if (bd == 0xffffffffu) {
            ok = false;
            break;
        }
        if (lane == (bd & 31u)) {
            const u32 q = bd >> 5;
#pragma unroll
            for (u32 qq = 0; qq < kSlots; ++qq)
                if (qq == q) {
                    tot[qq] += L;
                    att[qq] += static_cast<u64>(L) * L;
                    dev_of[i] = bd | (cnt[qq] << 16);  // device | slot within it (both < 2^16)
                    cnt[qq] += 1;
                }
        }
    }
    if (lane == 0) igroup[iter] = gi;
    if (ok) {
        // members grouped by device, in assignment order
        u64 base = spill_mbase;  // members of the devices before each slot row
#pragma unroll
        for (u32 q = 0; q < kSlots; ++q) {
            const u32 d = q * 32 + lane;
            const u32 c = d < N ? cnt[q] : 0u;
            u32 incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= static_cast<u32>(o)) incl += t;
            }
            const u32 row_total = __shfl_sync(0xffffffffu, incl, 31);
            if (d < N) {
                g_moff[spill_pbase + d] = base + (incl - c);
                g_cap[spill_pbase + d] = tot[q];
                g_total[spill_pbase + d] = tot[q];
                g_att[spill_pbase + d] = att[q];
                g_cnt[spill_pbase + d] = c;
                slots[iter * N + d] = c ? spill_pbase + d : kNone;
            }
            base += row_total;
        }
        __syncwarp();
        // members in assignment order within each device: every item knows
        // its slot, so the lanes place them independently
        for (u64 i = lane; i < k; i += 32) {
            const u32 w = dev_of[i];
            g_members[g_moff[spill_pbase + (w & 0xffffu)] + (w >> 16)] = sorted[i];
        }
    } else {
        for (u32 d = lane; d < N; d += 32) {
            g_total[spill_pbase + d] = 0;
            g_att[spill_pbase + d] = 0;
            g_cnt[spill_pbase + d] = 0;
            slots[iter * N + d] = d < rem ? tail_packs[d] : kNone;
        }
    }
}

__global__ void k_gather_spill(const u64* __restrict__ g_members, const u64* __restrict__ g_moff,
                               const u32* __restrict__ g_cnt, const u32* __restrict__ tail_packs, u32 rem,
                               const u64* __restrict__ tail_off, u64* __restrict__ out) {
    // one block per tail pack
    for (u32 t = blockIdx.x; t < rem; t += gridDim.x) {
        const u32 p = tail_packs[t];
        const u64 a = g_moff[p];
        const u32 c = g_cnt[p];
        for (u32 k = threadIdx.x; k < c; k += blockDim.x) out[tail_off[t] + k] = g_members[a + k];
    }
}

// ---------------------------------------------------------------------------
// plan output
// ---------------------------------------------------------------------------

__global__ void k_out_iterations(const u32* __restrict__ src, u64 I, u32 N, const int32_t* __restrict__ igroup,
                                 int32_t* __restrict__ out_group, int64_t* __restrict__ out_doff,
                                 int32_t* __restrict__ out_dindex) {
    GRID_STRIDE(p, I) {
        out_group[p] = igroup[src[p]];
        out_doff[p] = static_cast<int64_t>(p * N);
        for (u32 d = 0; d < N; ++d) out_dindex[p * N + d] = static_cast<int32_t>(d);
        if (p == I - 1) out_doff[I] = static_cast<int64_t>(I * N);
    }
}

__global__ void k_out_packs(const u32* __restrict__ src, u64 I, u32 N, const u32* __restrict__ slots,
                            const int64_t* __restrict__ dev_pack_off, const u32* __restrict__ g_cnt,
                            const u32* __restrict__ g_cap, const u32* __restrict__ g_total,
                            const u64* __restrict__ g_att, int64_t* __restrict__ pcap, int64_t* __restrict__ ptot,
                            int64_t* __restrict__ patt, u32* __restrict__ pglobal, u64* __restrict__ pcnt) {
    GRID_STRIDE(x, I * N) {
        const u64 p = x / N, d = x % N;
        const u32 g = slots[static_cast<u64>(src[p]) * N + d];
        if (g == kNone) continue;
        const int64_t q = dev_pack_off[x];
        pcap[q] = g_cap[g];
        ptot[q] = g_total[g];
        patt[q] = static_cast<int64_t>(g_att[g]);
        pglobal[q] = g;
        pcnt[q] = g_cnt[g];
    }
}

__global__ void k_out_members(const u32* __restrict__ pglobal, u64 P, const int64_t* __restrict__ moff,
                              const u64* __restrict__ g_moff, const u32* __restrict__ g_cnt,
                              const u64* __restrict__ g_members, int32_t* __restrict__ out) {
    // eight lanes per output pack (packs hold ~10 members): four packs in
    // flight per warp
    const u64 groups = (static_cast<u64>(gridDim.x) * blockDim.x) >> 3;
    const u32 sub = threadIdx.x & 7u;
    for (u64 q = (blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x) >> 3; q < P; q += groups) {
        const u32 g = pglobal[q];
        const u64 a = g_moff[g];
        const u32 c = g_cnt[g];
        const int64_t d = moff[q];
        for (u32 k = sub; k < c; k += 8) out[d + k] = static_cast<int32_t>(entry_idx(g_members[a + k]));
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------

void validate_groups(const std::vector<hbp_group_config>& g, int64_t l_max) {
    if (g.empty()) fail_validation("no packing groups");
    int64_t prev = 0;
    for (const auto& x : g) {
        if (x.length <= prev) fail_validation("group lengths must be strictly increasing");
        if (x.sp < 1 || x.ckpt < 0) fail_validation("invalid group runtime config");
        prev = x.length;
    }
    if (g.back().length != l_max) fail_validation("last group must carry l_max");
}

void validate_strategy(const hbp_strategy& s) {
    if (s.kind == HBP_STRATEGY_ISF) {
        if (s.isf_iterations < 1) fail_validation("isf_iterations must be >= 1");
        if (s.isf_fill_threshold <= 0.0 || s.isf_fill_threshold > 1.0)
            fail_validation("isf fill threshold must lie in (0, 1]");
    }
    if (s.kind < HBP_STRATEGY_RANDOM || s.kind > HBP_STRATEGY_SPFHP) fail_validation("unknown packing strategy");
}

namespace {

struct IngestResult {
    IngestFlags f;
};

// Uploads lengths (and ids), converts, and collects the flags. `limit` is
// the largest admissible length (l_max or the pack capacity).
IngestFlags upload_and_scan(Ctx& c, const hbp_samples* in, DeviceCorpus& corpus, int64_t limit,
                            DevBuf<int64_t>& dids) {
    const u64 n = static_cast<u64>(in->n);
    cudaStream_t s = c.stream;
    corpus.n = in->n;
    corpus.len32.alloc(n, s);
    DevBuf<int64_t> dlen;
    const int64_t* len_dev = in->lengths;
    const int64_t* ids_dev = in->ids;
    if (in->memory == HBP_MEM_HOST) {
        dlen.alloc(n, s);
        CUDA_CHECK(cudaMemcpyAsync(dlen.p, in->lengths, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
        len_dev = dlen.p;
        if (in->ids) {
            dids.alloc(n, s);
            CUDA_CHECK(cudaMemcpyAsync(dids.p, in->ids, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
            ids_dev = dids.p;
        }
    }
    DevBuf<IngestFlags> f(1, s);
    IngestFlags init{~0ull, ~0ull, 0ull, 0ull};
    CUDA_CHECK(cudaMemcpyAsync(f.p, &init, sizeof(init), cudaMemcpyHostToDevice, s));
    LAUNCH(k_ingest, G(n), kB, 0, s, len_dev, ids_dev, n, limit, corpus.len32.p, f.p);
    IngestFlags out = read_scalar(c, f.p);
    corpus.neg_ids = static_cast<i64>(out.neg);
    corpus.ids_ascending = out.not_ascending == 0;
    corpus.key_bits = bits_for(n > 0 ? n - 1 : 0);
    if (in->ids) {
        if (in->memory == HBP_MEM_HOST) {
            corpus.ids_host = in->ids;
        } else {
            corpus.h_ids = read_vector(c, in->ids, n);
            corpus.ids_host = corpus.h_ids.data();
        }
    } else {
        corpus.ids_host = nullptr;
    }
    return out;
}

// Ranks of general (non-ascending) ids; returns the first duplicate index.
u64 rank_ids(Ctx& c, const int64_t* ids_dev, DeviceCorpus& corpus) {
    const u64 n = static_cast<u64>(corpus.n);
    cudaStream_t s = c.stream;
    DevBuf<u32> order(n, s), words(n, s), tk(n, s), tv(n, s);
    LAUNCH(k_iota, G(n), kB, 0, s, order.p, n);
    for (int pass = 0; pass < 2; ++pass) {
        LAUNCH(k_id_words, G(n), kB, 0, s, ids_dev, order.p, n, pass == 1, words.p);
        radix_sort_pairs(c, words.p, order.p, static_cast<i64>(n), 32, false, tk.p, tv.p);
    }
    corpus.key32.alloc(n, s);
    DevBuf<unsigned long long> dup(1, s);
    const unsigned long long none = ~0ull;
    CUDA_CHECK(cudaMemcpyAsync(dup.p, &none, sizeof(none), cudaMemcpyHostToDevice, s));
    LAUNCH(k_ranks_dups, G(n), kB, 0, s, ids_dev, order.p, n, corpus.key32.p, dup.p);
    return read_scalar(c, dup.p);
}

// Sorts entries by (length desc, key asc) in place.
void sort_entries(Ctx& c, const DeviceCorpus& corpus, u64* e, u64 n, bool key_ordered, u32 max_len) {
    if (n <= 1) return;
    if (sort_entries_small(c, e, static_cast<i64>(n), corpus.key32.p, key_ordered ? 0 : corpus.key_bits,
                           bits_for(max_len)))
        return;
    cudaStream_t s = c.stream;
    DevBuf<u32> k(n, s), v(n, s), tk(n, s), tv(n, s);
    LAUNCH(k_keys_of_entries, G(n), kB, 0, s, e, corpus.key32.p, n, k.p, v.p);
    if (!key_ordered) radix_sort_pairs(c, k.p, v.p, static_cast<i64>(n), corpus.key_bits, false, tk.p, tv.p);
    LAUNCH(k_lens_of, G(n), kB, 0, s, e, v.p, n, k.p);
    radix_sort_pairs(c, k.p, v.p, static_cast<i64>(n), bits_for(max_len), true, tk.p, tv.p);
    DevBuf<u64> tmp(n, s);
    LAUNCH(k_gather_entries, G(n), kB, 0, s, e, v.p, n, tmp.p);
    CUDA_CHECK(cudaMemcpyAsync(e, tmp.p, sizeof(u64) * n, cudaMemcpyDeviceToDevice, s));
}

// Global pack table being built.
struct PackTable {
    DevBuf<u64> members;   // entries
    DevBuf<u64> moff;      // first member per pack
    DevBuf<u32> cnt, cap, total;
    DevBuf<u64> att;
    u64 n_packs = 0, n_members = 0;
};

// Result of packing one group (members laid out contiguously).
struct GroupPacks {
    u64 P = 0;  // packs in PackList order
    u64 M = 0;  // members
    DevBuf<u64> members;
    DevBuf<u64> off;  // P + 1
};

// Stage 1 of one group: pack(pool, cap, strategy, seed) -> ISF packs +
// FFD bins with their leaves (residual, count) for greedy fill.
struct PackedGroup {
    u64 n_isf = 0;
    u64 n_isf_members = 0;
    DevBuf<u64> isf_members, isf_off;
    DevBuf<u32> isf_total;
    u64 n_ffd = 0;
    u64 n_residue = 0;
    DevBuf<u64> residue;       // sorted residue items
    DevBuf<u32> res_bin, res_slot;
    DevBuf<u64> leaves;        // all packs: ISF then FFD bins
    u64 P() const { return n_isf + n_ffd; }
};

void pack_pool(Ctx& c, const DeviceCorpus& corpus, const u64* pool_in, u64 m, u32 cap, const hbp_strategy& st,
               uint64_t seed, PackedGroup& out) {
    cudaStream_t s = c.stream;
    out.isf_members.alloc(m, s);
    out.isf_off.alloc(m + 1, s);
    out.isf_total.alloc(m + 1, s);
    DevBuf<u64> counters(2, s);
    counters.zero();
    PackSink sink{out.isf_members.p, out.isf_off.p, out.isf_total.p, counters.p, counters.p + 1};
    u64 n_members = 0, n_packs = 0;  // host copies of the sink counters
    DevBuf<u64> A(m, s), Bf(m, s);
    CUDA_CHECK(cudaMemcpyAsync(A.p, pool_in, sizeof(u64) * m, cudaMemcpyDeviceToDevice, s));
    u64 cur = m;
    bool residue_ffd = false;
    bool key_ordered = corpus.key32.p == nullptr;  // pool in input order == key order
    if (st.kind == HBP_STRATEGY_ISF || st.kind == HBP_STRATEGY_RANDOM) {
        const int rounds = st.kind == HBP_STRATEGY_ISF ? st.isf_iterations : 1;
        u64 tmin = 0;
        if (st.kind == HBP_STRATEGY_ISF) {
            const double min_fill = static_cast<double>(cap) * st.isf_fill_threshold;  // packing.cpp:177-178
            tmin = static_cast<u64>(std::ceil(min_fill));
        }
        std::vector<uint64_t> seeds(static_cast<size_t>(rounds > 0 ? rounds : 0));
        for (int r = 0; r < rounds; ++r)
            seeds[r] = st.kind == HBP_STRATEGY_ISF ? derive_seed(seed, "isf-round", static_cast<uint64_t>(r))
                                                   : derive_seed(seed, "random-pack");
        // small pools: every round in one launch
        const bool done = isf_small(c, seeds, A.p, cur, cap, tmin, sink, n_members, n_packs);
        for (int r = 0; !done && r < rounds && cur > 0; ++r) {
            const uint64_t rs = seeds[r];
            fy_shuffle_u64(c, rs, static_cast<i64>(cur), A.p, Bf.p);
            trace_mark(c, "isf.shuffle");
            cur = static_cast<u64>(nextfit_freeze(c, Bf.p, static_cast<i64>(cur), cap, tmin, sink, A.p, n_members, n_packs));
            trace_mark(c, "isf.nextfit+freeze");
        }
        residue_ffd = st.kind == HBP_STRATEGY_ISF;
        key_ordered = false;  // the residue is in shuffled order
    } else if (st.kind == HBP_STRATEGY_FFD) {
        residue_ffd = true;
    } else if (st.kind == HBP_STRATEGY_FFS) {
        // first fit over a seeded shuffle (packing.cpp:239-243)
        fy_shuffle_u64(c, derive_seed(seed, "ffs"), static_cast<i64>(m), A.p, Bf.p);
        CUDA_CHECK(cudaMemcpyAsync(A.p, Bf.p, sizeof(u64) * m, cudaMemcpyDeviceToDevice, s));
    } else if (st.kind == HBP_STRATEGY_BFS) {
        // best fit over a seeded shuffle (packing.cpp:244-248)
        fy_shuffle_u64(c, derive_seed(seed, "bfs"), static_cast<i64>(m), A.p, Bf.p);
        CUDA_CHECK(cudaMemcpyAsync(A.p, Bf.p, sizeof(u64) * m, cudaMemcpyDeviceToDevice, s));
    } else {
        residue_ffd = true;  // SPFHP walks lengths longest first, ids ascending (packing.cpp:135-137)
    }
    out.n_isf_members = n_members;
    out.n_isf = n_packs;
    out.n_residue = cur;
    out.leaves.alloc(out.n_isf + cur + 1, s);
    if (out.n_isf > 0) {
        LAUNCH(k_isf_leaves, G(out.n_isf), kB, 0, s, out.isf_off.p, out.isf_total.p, out.n_isf, out.n_isf_members,
               cap, out.leaves.p);
    }
    if (cur > 0) {
        out.residue.alloc(cur, s);
        CUDA_CHECK(cudaMemcpyAsync(out.residue.p, A.p, sizeof(u64) * cur, cudaMemcpyDeviceToDevice, s));
        if (residue_ffd) sort_entries(c, corpus, out.residue.p, cur, key_ordered, cap);
        trace_mark(c, "ffd.sort");
        out.res_bin.alloc(cur, s);
        out.res_slot.alloc(cur, s);
        const bool scan_rule = st.kind == HBP_STRATEGY_BFS || st.kind == HBP_STRATEGY_SPFHP;
        const FitResult fr =
            scan_rule ? scan_fit(c, out.residue.p, static_cast<i64>(cur), out.leaves.p + out.n_isf,
                                 static_cast<i64>(cur), cap, st.kind == HBP_STRATEGY_SPFHP, out.res_bin.p, out.res_slot.p)
                      : first_fit_runs(c, out.residue.p, static_cast<i64>(cur), out.leaves.p + out.n_isf, 0,
                                       static_cast<i64>(cur), cap, FitMode::Ffd, out.res_bin.p, out.res_slot.p);
        out.n_ffd = static_cast<u64>(fr.bins);
        trace_mark(c, "ffd.engine");
    }
}

// Lays the group's packs out contiguously (after an optional fill) and
// appends them to the pack table. Returns the group pack count.
u64 layout_group(Ctx& c, PackedGroup& pg, const u64* fill_items, u64 n_fill, const u32* fill_bin,
                 const u32* fill_slot, u32 cap, PackTable& T) {
    cudaStream_t s = c.stream;
    const u64 P = pg.P();
    if (P == 0) return 0;
    DevBuf<u64> off(P + 1, s);
    {
        const u64* lv = pg.leaves.p;
        u64* op = off.p;
        const i64 PP = static_cast<i64>(P);
        scan_exclusive<u64>(
            PP + 1, [=] __device__(i64 i) { return i < PP ? static_cast<u64>(static_cast<u32>(lv[i])) : 0ull; },
            [=] __device__(i64 i, u64 v) { op[i] = v; }, s, c.scan, "scan.plan1");
    }
    const u64 M = read_vector(c, off.p + P, 1)[0];
    u64* dst = T.members.p + T.n_members;
    if (pg.n_isf > 0)
        LAUNCH(k_place_isf, grid_for(pg.n_isf * 8, kB, 148u * 64u), kB, 0, s, pg.isf_members.p, pg.isf_off.p, pg.n_isf, pg.n_isf_members, off.p,
               dst);
    if (pg.n_residue > 0)
        LAUNCH(k_place_items, G(pg.n_residue), kB, 0, s, pg.residue.p, pg.res_bin.p, pg.res_slot.p, pg.n_residue,
               pg.n_isf, off.p, dst);
    if (n_fill > 0)
        LAUNCH(k_place_items, G(n_fill), kB, 0, s, fill_items, fill_bin, fill_slot, n_fill, 0ull, off.p, dst);
    LAUNCH(k_pack_stats, G(P), kB, 0, s, dst, off.p, P, T.n_members, T.n_packs, cap, T.moff.p, T.cnt.p, T.cap.p,
           T.total.p, T.att.p);
    T.n_members += M;
    T.n_packs += P;
    return P;
}

// Orders the group's packs (stable attention desc, or seeded shuffle) and
// writes its iterations. Returns iterations written.
u64 batch_group(Ctx& c, const DeviceCorpus& corpus, PackTable& T, u64 pbase, u64 P, u32 N, u32 cap, int gi,
                bool balance, uint64_t seed, u64 ibase, DevBuf<u32>& slots, DevBuf<int32_t>& igroup) {
    cudaStream_t s = c.stream;
    if (P == 0) return 0;
    DevBuf<u32> order(P, s);
    if (balance) {
        DevBuf<u32> w(P, s), tk(P, s), tv(P, s);
        LAUNCH(k_iota, G(P), kB, 0, s, order.p, P);
        const u64* att = T.att.p + pbase;
        // attention <= cap^2: sort only the bits it can have (one 32-bit
        // pass set when cap^2 < 2^32, else the low word then the few high bits)
        const u64 amax = static_cast<u64>(cap) * cap;
        const int hi_bits = bits_for(amax >> 32);
        LAUNCH(k_att_words, G(P), kB, 0, s, att, order.p, P, false, w.p);
        radix_sort_pairs(c, w.p, order.p, static_cast<i64>(P), (amax >> 32) ? 32 : bits_for(amax), true, tk.p, tv.p);
        if (amax >> 32) {
            LAUNCH(k_att_words, G(P), kB, 0, s, att, order.p, P, true, w.p);
            radix_sort_pairs(c, w.p, order.p, static_cast<i64>(P), hi_bits, true, tk.p, tv.p);
        }
    } else {
        fy_source_positions(c, derive_seed(seed, "pack-batching", static_cast<uint64_t>(gi)), static_cast<i64>(P),
                            order.p);
    }
    const u64 nfull = P / N;
    const u32 rem = static_cast<u32>(P % N);
    if (nfull > 0)
        LAUNCH(k_full_iterations, G(nfull * N), kB, 0, s, order.p, nfull, N, static_cast<u32>(pbase), gi, ibase,
               slots.p, igroup.p);
    if (rem == 0) return nfull;
    // spill tail: gather its samples, sort (length desc, id asc), redistribute
    // tail packs and their sizes in one read-back
    DevBuf<u32> dtail(rem, s), dtcnt(rem, s);
    {
        const u32* op = order.p + nfull * N;
        const u32* cp = T.cnt.p;
        u32* tp = dtail.p;
        u32* np = dtcnt.p;
        const u32 pb = static_cast<u32>(pbase);
        for_each_index(c, rem, [=] __device__(u64 t) {
            tp[t] = op[t] + pb;
            np[t] = cp[op[t] + pb];
        });
    }
    std::vector<u32> tail = read_vector(c, dtail.p, rem), tcnt = read_vector(c, dtcnt.p, rem);
    std::vector<u64> toff(rem);
    u64 k = 0;
    for (u32 t = 0; t < rem; ++t) {
        toff[t] = k;
        k += tcnt[t];
    }
    DevBuf<u64> dtoff(rem, s);
    CUDA_CHECK(cudaMemcpyAsync(dtoff.p, toff.data(), sizeof(u64) * rem, cudaMemcpyHostToDevice, s));
    DevBuf<u64> spill(k + 1, s);
    DevBuf<u32> dev_of(k + 1, s);
    if (c.trace) std::fprintf(stderr, "[hbp trace] spill group %d: %u tail packs, %llu samples\n", gi, rem,
                              static_cast<unsigned long long>(k));
    LAUNCH(k_gather_spill, rem, 256, 0, s, T.members.p, T.moff.p, T.cnt.p, dtail.p, rem, dtoff.p, spill.p);
    sort_entries(c, corpus, spill.p, k, false, cap);
    const u32 spill_pbase = static_cast<u32>(T.n_packs);
    if (N > 32 * kSpillSlots || k >= 65536)
        LAUNCH(k_spill_serial, 1, 32, 0, s, spill.p, k, N, cap, dtail.p, rem, spill_pbase, T.n_members, gi,
               ibase + nfull, T.members.p, T.moff.p, T.cnt.p, T.cap.p, T.total.p, T.att.p, dev_of.p, slots.p,
               igroup.p);
    else if (N <= 32)
        LAUNCH(k_spill<1>, 1, 32, 0, s, spill.p, k, N, cap, dtail.p, rem, spill_pbase, T.n_members, gi, ibase + nfull,
               T.members.p, T.moff.p, T.cnt.p, T.cap.p, T.total.p, T.att.p, dev_of.p, slots.p, igroup.p);
    else
    LAUNCH(k_spill<kSpillSlots>, 1, 32, 0, s, spill.p, k, N, cap, dtail.p, rem, spill_pbase, T.n_members, gi, ibase + nfull,
           T.members.p, T.moff.p, T.cnt.p, T.cap.p, T.total.p, T.att.p, dev_of.p, slots.p, igroup.p);
    CUDA_CHECK(cudaStreamSynchronize(s));  // host vectors above go out of scope
    T.n_packs += N;
    T.n_members += k;
    return nfull + 1;
}

void emit_plan(Ctx& c, PackTable& T, DevBuf<u32>& slots, DevBuf<int32_t>& igroup, u64 I, u32 N, uint64_t seed,
               DevicePlan& out, bool shuffle = true) {
    cudaStream_t s = c.stream;
    out.n_iterations = static_cast<int64_t>(I);
    out.n_devices = static_cast<int64_t>(I * N);
    out.iter_group.alloc(I + 1, s);
    out.iter_dev_offsets.alloc(I + 1, s);
    out.dev_index.alloc(I * N + 1, s);
    out.dev_pack_offsets.alloc(I * N + 1, s);
    if (I == 0) {
        CUDA_CHECK(cudaMemsetAsync(out.iter_dev_offsets.p, 0, sizeof(int64_t), s));
        CUDA_CHECK(cudaMemsetAsync(out.dev_pack_offsets.p, 0, sizeof(int64_t), s));
        out.n_packs = 0;
        out.n_members = 0;
        out.pack_member_offsets.alloc(1, s);
        CUDA_CHECK(cudaMemsetAsync(out.pack_member_offsets.p, 0, sizeof(int64_t), s));
        return;
    }
    DevBuf<u32> src(I, s);
    if (shuffle) {
        fy_source_positions(c, derive_seed(seed, "plan-shuffle"), static_cast<i64>(I), src.p);  // balance.cpp:255-256
    } else {
        LAUNCH(k_iota, G(I), kB, 0, s, src.p, I);
    }
    LAUNCH(k_out_iterations, G(I), kB, 0, s, src.p, I, N, igroup.p, out.iter_group.p, out.iter_dev_offsets.p,
           out.dev_index.p);
    {
        const u32* sp = src.p;
        const u32* sl = slots.p;
        int64_t* dpo = out.dev_pack_offsets.p;
        const i64 D = static_cast<i64>(I * N);
        const u32 NN = N;
        scan_exclusive<int64_t>(
            D + 1,
            [=] __device__(i64 x) -> int64_t {
                if (x >= D) return 0;
                return sl[static_cast<u64>(sp[x / NN]) * NN + (x % NN)] != kNone ? 1 : 0;
            },
            [=] __device__(i64 x, int64_t v) { dpo[x] = v; }, s, c.scan, "scan.plan2");
    }
    const u64 P = static_cast<u64>(read_vector(c, out.dev_pack_offsets.p + I * N, 1)[0]);
    out.n_packs = static_cast<int64_t>(P);
    out.pack_capacity.alloc(P + 1, s);
    out.pack_total.alloc(P + 1, s);
    out.pack_attention.alloc(P + 1, s);
    out.pack_member_offsets.alloc(P + 1, s);
    DevBuf<u32> pglobal(P + 1, s);
    DevBuf<u64> pcnt(P + 1, s);
    LAUNCH(k_out_packs, G(I * N), kB, 0, s, src.p, I, N, slots.p, out.dev_pack_offsets.p, T.cnt.p, T.cap.p,
           T.total.p, T.att.p, out.pack_capacity.p, out.pack_total.p, out.pack_attention.p, pglobal.p, pcnt.p);
    {
        const u64* pc = pcnt.p;
        int64_t* mo = out.pack_member_offsets.p;
        const i64 PP = static_cast<i64>(P);
        scan_exclusive<int64_t>(
            PP + 1, [=] __device__(i64 q) -> int64_t { return q < PP ? static_cast<int64_t>(pc[q]) : 0; },
            [=] __device__(i64 q, int64_t v) { mo[q] = v; }, s, c.scan, "scan.plan3");
    }
    const u64 M = static_cast<u64>(read_vector(c, out.pack_member_offsets.p + P, 1)[0]);
    out.n_members = static_cast<int64_t>(M);
    out.member_index.alloc(M + 1, s);
    LAUNCH(k_out_members, grid_for(P * 8, kB, 148u * 64u), kB, 0, s, pglobal.p, P, out.pack_member_offsets.p,
           T.moff.p, T.cnt.p, T.members.p, out.member_index.p);
}

}  // namespace

int64_t DeviceCorpus::length_of(Ctx& c, i64 i) const {
    if (lengths_host) return lengths_host[i];
    return read_vector(c, lengths_dev + i, 1)[0];
}

void ingest(Ctx& c, const hbp_samples* in, DeviceCorpus& corpus) {
    if (in->n < 0) fail_validation("negative sample count");
    if (in->n > 0x7fffffffLL) fail_validation("corpus too large for the engine (more than 2^31-1 samples)");
    corpus.n = in->n;
    if (in->memory == HBP_MEM_HOST) corpus.lengths_host = in->lengths;
    else corpus.lengths_dev = in->lengths;
    if (in->n == 0) return;
    DevBuf<int64_t> dids;
    const IngestFlags f = upload_and_scan(c, in, corpus, 0x7fffffffLL, dids);
    corpus.first_bad_len = f.first_bad_len;
    corpus.first_huge = f.first_over;
    if (!corpus.ids_ascending) {
        const int64_t* ids_dev = in->memory == HBP_MEM_HOST ? dids.p : in->ids;
        corpus.first_dup = rank_ids(c, ids_dev, corpus);
    }
}

void validate_corpus(Ctx& c, const hbp_samples* in, const DeviceCorpus& corpus, const std::string& source) {
    (void)in;
    if (corpus.n == 0) fail_validation("empty corpus: " + source);
    if (corpus.first_bad_len != ~0ull && corpus.first_bad_len <= corpus.first_dup) {
        const i64 i = static_cast<i64>(corpus.first_bad_len);
        fail_validation("sample " + std::to_string(corpus.id_of(i)) + " has non-positive length " +
                        std::to_string(corpus.length_of(c, i)));
    }
    if (corpus.first_dup != ~0ull)
        fail_validation("duplicate sample id " + std::to_string(corpus.id_of(static_cast<i64>(corpus.first_dup))));
}

namespace {

// Partitions the corpus by group (stable) and returns entries + offsets.
void partition(Ctx& c, DeviceCorpus& corpus, const std::vector<hbp_group_config>& groups, int64_t l_max,
               DevBuf<u64>& entries, std::vector<u64>& goff) {
    cudaStream_t s = c.stream;
    const u64 n = static_cast<u64>(corpus.n);
    const int ng = static_cast<int>(groups.size());
    std::vector<int64_t> gl(ng);
    for (int g = 0; g < ng; ++g) gl[g] = groups[g].length;
    DevBuf<int64_t> dgl(ng, s);
    CUDA_CHECK(cudaMemcpyAsync(dgl.p, gl.data(), sizeof(int64_t) * ng, cudaMemcpyHostToDevice, s));
    DevBuf<u32> key(n, s), val(n, s), tk(n, s), tv(n, s);
    DevBuf<unsigned long long> counts(65, s);  // per group, then [64] the first sample beyond l_max
    counts.zero();
    const unsigned long long none = ~0ull;
    CUDA_CHECK(cudaMemcpyAsync(counts.p + 64, &none, sizeof(none), cudaMemcpyHostToDevice, s));
    // len32 saturates at 2^31-1; longer samples are tracked in first_huge
    const u32 lm = l_max > 0x7fffffffLL ? 0x7fffffffu : static_cast<u32>(l_max);
    LAUNCH(k_group_keys, G(n), kB, 0, s, corpus.len32.p, n, dgl.p, ng, lm, key.p, val.p, counts.p);
    if (ng > 1) radix_sort_pairs(c, key.p, val.p, static_cast<i64>(n), bits_for(ng - 1), false, tk.p, tv.p);
    entries.alloc(n, s);
    LAUNCH(k_entries_from_idx, G(n), kB, 0, s, corpus.len32.p, val.p, n, entries.p);
    const auto cnt = read_vector(c, counts.p, 65);
    u64 first = cnt[64];
    if (corpus.first_huge < first) first = corpus.first_huge;
    if (first != ~0ull)
        fail_validation("sample " + std::to_string(corpus.id_of(static_cast<i64>(first))) +
                        " exceeds the largest packing length " + std::to_string(l_max));
    goff.assign(ng + 1, 0);
    for (int g = 0; g < ng; ++g) goff[g + 1] = goff[g] + cnt[g];
}

}  // namespace

void group_data_device(Ctx& c, DeviceCorpus& corpus, const std::vector<hbp_group_config>& groups, int64_t l_max,
                       std::vector<int64_t>& offsets, std::vector<int32_t>& members) {
    validate_groups(groups, l_max);
    if (groups.size() > 64) fail_validation("the GPU engine supports at most 64 packing groups");
    DevBuf<u64> entries;
    std::vector<u64> goff;
    if (corpus.n > 0) {
        partition(c, corpus, groups, l_max, entries, goff);  // also group_data's l_max check
    } else {
        goff.assign(groups.size() + 1, 0);
    }
    offsets.assign(goff.begin(), goff.end());
    members.resize(static_cast<size_t>(corpus.n));
    if (corpus.n > 0) {
        DevBuf<int32_t> idx(static_cast<size_t>(corpus.n), c.stream);
        const u64* ep = entries.p;
        int32_t* ip = idx.p;
        for_each_index(c, static_cast<u64>(corpus.n), [=] __device__(u64 i) { ip[i] = static_cast<int32_t>(entry_idx(ep[i])); });
        CUDA_CHECK(cudaMemcpyAsync(members.data(), idx.p, sizeof(int32_t) * corpus.n, cudaMemcpyDeviceToHost, c.stream));
        CUDA_CHECK(cudaStreamSynchronize(c.stream));
    }
}

void build_plan_device(Ctx& c, DeviceCorpus& corpus, const PlanArgs& a, DevicePlan& out) {
    cudaStream_t s = c.stream;
    validate_groups(a.groups, a.l_max);
    if (a.device_count < 1) fail_validation("device count must be >= 1");
    if (a.groups.size() > 64) fail_validation("the GPU engine supports at most 64 packing groups");
    out.device_count = a.device_count;
    out.seed = a.seed;
    out.groups = a.groups;
    out.l_best = a.l_best;
    out.l_max = a.l_max;

    const u64 n = static_cast<u64>(corpus.n);
    const u32 N = static_cast<u32>(a.device_count);
    const int ng = static_cast<int>(a.groups.size());
    DevBuf<u64> entries;
    std::vector<u64> goff;
    partition(c, corpus, a.groups, a.l_max, entries, goff);  // also group_data's l_max check
    trace_mark(c, "group_data");

    // Pools, concatenated: Pin holds pool g at off[g] in input order (the
    // partition's output as is); Ps holds the same pools sorted for greedy
    // fill (length desc, key asc), in DEScending group order, so the fill
    // items of group gi -- pools gi-1 .. 0, nearest (longest) first,
    // balance.cpp:235-243 -- are the contiguous tail of Ps from soff[gi-1].
    // Each pool is sorted once; after a fill, one scan compacts the pools it
    // drew from in both layouts (order preserved), so sorted stays sorted.
    std::vector<u64> psize(ng), off(ng + 1, 0), soff(ng, 0);
    for (int g = 0; g < ng; ++g) psize[g] = goff[g + 1] - goff[g];
    DevBuf<u64> Pin = std::move(entries), Pin2, Ps, Ps2;
    auto refresh_offsets = [&]() {
        off[0] = 0;
        for (int g = 0; g < ng; ++g) off[g + 1] = off[g] + psize[g];
        u64 o = 0;
        for (int g = ng - 1; g >= 0; --g) {
            soff[g] = o;
            o += psize[g];
        }
    };
    refresh_offsets();
    const bool any_fill = a.greedy_fill && ng > 1;

    PackTable T;
    const u64 cap_packs = n + static_cast<u64>(ng) * N + 1;
    T.members.alloc(2 * n + 1, s);
    T.moff.alloc(cap_packs, s);
    T.cnt.alloc(cap_packs, s);
    T.cap.alloc(cap_packs, s);
    T.total.alloc(cap_packs, s);
    T.att.alloc(cap_packs, s);
    const u64 max_iters = n / N + ng + 2;
    DevBuf<u32> slots(max_iters * N, s);
    DevBuf<int32_t> igroup(max_iters, s);
    u64 I = 0;
    DevBuf<u8> consumed;
    bool sorted_ready = false;

    for (int gi = ng - 1; gi >= 0; --gi) {
        if (psize[gi] == 0) continue;
        const u32 cap = static_cast<u32>(a.groups[gi].length);
        // greedy fill from pools gi-1 .. 0: the items and their runs depend
        // only on the pools, so they are prepared on the side stream while
        // this group packs on the main stream (the first time with the sorts)
        u64 n_fill = 0;
        if (any_fill && gi > 0) {
            for (int j = 0; j < gi; ++j) n_fill += psize[j];
        }
        DevBuf<u32> fill_bin, fill_slot, run_item, run_len, n_runs;
        FitRuns fruns;
        if (n_fill > 0 && !sorted_ready) Ps.alloc(n + 1, s);
        const u64* fill_items = n_fill > 0 ? Ps.p + soff[gi - 1] : nullptr;
        SideJoin fork_guard(c);  // after the buffers the side stream uses: joined before they go
        if (n_fill > 0) {
            run_item.alloc(n_fill, s);
            run_len.alloc(n_fill, s);
            n_runs.alloc(4, s);
            fruns = FitRuns{run_item.p, run_len.p, n_runs.p};
            side_fork(c);
            fork_guard.armed = true;
            {
                SideScope side(c);
                if (!sorted_ready) {
                    for (int j = gi - 1; j >= 0; --j) {
                        if (!psize[j]) continue;
                        CUDA_CHECK(cudaMemcpyAsync(Ps.p + soff[j], Pin.p + off[j], sizeof(u64) * psize[j],
                                                   cudaMemcpyDeviceToDevice, c.stream));
                        sort_entries(c, corpus, Ps.p + soff[j], psize[j], corpus.key32.p == nullptr,
                                     static_cast<u32>(a.groups[j].length));
                    }
                }
                prepare_runs(c, fill_items, static_cast<i64>(n_fill), corpus.key32.p,
                             static_cast<u64>(corpus.neg_ids), fruns);
            }
            sorted_ready = true;
        }
        PackedGroup pg;
        pack_pool(c, corpus, Pin.p + off[gi], psize[gi], cap, a.strategy,
                  derive_seed(a.seed, "pack", static_cast<uint64_t>(gi)), pg);
        fork_guard.join();
        trace_mark(c, "fill.sort");
        if (n_fill > 0 && pg.P() == 0) n_fill = 0;  // nothing to fill
        if (n_fill > 0) {
            const u64 P = pg.P();
            fill_bin.alloc(n_fill, s);
            fill_slot.alloc(n_fill, s);
            first_fit_runs(c, fill_items, static_cast<i64>(n_fill), pg.leaves.p, static_cast<i64>(P),
                           static_cast<i64>(P), cap, FitMode::Fill, fill_bin.p, fill_slot.p, corpus.key32.p,
                           static_cast<u64>(corpus.neg_ids), &fruns);
            trace_mark(c, "fill.engine");
            if (!consumed.p) {
                consumed.alloc(n, s);
                consumed.zero();
            }
            LAUNCH(k_mark_consumed, G(n_fill), kB, 0, s, fill_items, fill_bin.p, n_fill, consumed.p);
        }
        trace_mark(c, "fill.expand+compact");
        const u64 pbase = T.n_packs;
        const u64 P = layout_group(c, pg, fill_items, n_fill, fill_bin.p, fill_slot.p, cap, T);
        trace_mark(c, "layout");
        I += batch_group(c, corpus, T, pbase, P, N, cap, gi, a.balance_batching, a.seed, I, slots, igroup);
        trace_mark(c, "batching");
        if (n_fill > 0) {
            // the pools gi-1 .. 0 lose the samples this fill took: one scan
            // compacts both layouts (keep counts of Pin in the low, of Ps in
            // the high half; Ps only while a later group still fills from it)
            // and records the running count at the end of each Pin pool (the
            // new sizes are the differences; one read)
            std::vector<u64> h_end(gi);
            for (int j = 0; j < gi; ++j) h_end[j] = psize[j] ? off[j + 1] - 1 : ~0ull;  // empty: never matched
            DevBuf<u64> dend(gi, s), dincl(gi, s);
            CUDA_CHECK(cudaMemcpyAsync(dend.p, h_end.data(), sizeof(u64) * gi, cudaMemcpyHostToDevice, s));
            if (!Pin2.p) Pin2.alloc(n + 1, s);
            const bool keep_sorted = gi > 1;  // a later group still fills from the sorted pools
            if (keep_sorted && !Ps2.p) Ps2.alloc(n + 1, s);
            const u64* pin = Pin.p;
            const u64* ps = Ps.p + soff[gi - 1];
            u64* pin2 = Pin2.p;
            u64* ps2 = keep_sorted ? Ps2.p + soff[gi - 1] : nullptr;
            const u8* cons = consumed.p;
            const u64* ends = dend.p;
            u64* incl = dincl.p;
            const int nseg = gi;
if (keep_sorted) {
                scan_exclusive_v<u64>(
                    static_cast<i64>(n_fill),
                    [=] __device__(i64 i) -> u64 {
                        return (cons[entry_idx(pin[i])] ? 0ull : 1ull) | (!cons[entry_idx(ps[i])] ? (1ull << 32) : 0ull);
                    },
                    [=] __device__(i64 i, u64 v, u64 x) {
                        const bool k1 = (x & 1ull) != 0;
                        if (k1) pin2[static_cast<u32>(v)] = pin[i];
                        if (x >> 32) ps2[v >> 32] = ps[i];
                        for (int j = 0; j < nseg; ++j)
                            if (static_cast<u64>(i) == ends[j]) incl[j] = static_cast<u32>(v) + (k1 ? 1u : 0u);
                    },
                    s, c.scan, "scan.plan4");
            } else {  // the last fill: only the input-order pools are used again
                scan_exclusive_v<u32>(
                    static_cast<i64>(n_fill), [=] __device__(i64 i) -> u32 { return cons[entry_idx(pin[i])] ? 0u : 1u; },
                    [=] __device__(i64 i, u32 v, u32 x) {
                        const bool k1 = x != 0;
                        if (k1) pin2[v] = pin[i];
                        for (int j = 0; j < nseg; ++j)
                            if (static_cast<u64>(i) == ends[j]) incl[j] = v + (k1 ? 1u : 0u);
                    },
                    s, c.scan, "scan.plan4");
            }
            const std::vector<u64> h_incl = read_vector(c, dincl.p, gi);  // (also orders the host copy above)
            std::vector<u64> kept(gi, 0);
            u64 run = 0;
            for (int j = 0; j < gi; ++j)
                if (psize[j]) {
                    kept[j] = h_incl[j] - run;
                    run = h_incl[j];
                }
            std::swap(Pin, Pin2);
            if (keep_sorted) std::swap(Ps, Ps2);
            for (int j = 0; j < gi; ++j) psize[j] = kept[j];
            // the groups >= gi are done: keep their sizes out of the offsets
            const u64 base_s = soff[gi - 1];
            for (int g = gi; g < ng; ++g) psize[g] = 0;
            refresh_offsets();
            // Ps2 (now Ps) holds the compacted tail at the old tail start
            for (int j = 0; j < gi; ++j) soff[j] += base_s;
        } else {
            psize[gi] = 0;
        }
    }
    emit_plan(c, T, slots, igroup, I, N, a.seed, out);
    trace_mark(c, "emit");
    CUDA_CHECK(cudaStreamSynchronize(s));
    if (std::getenv("HBP_COUNT_SYNCS"))
        std::fprintf(stderr, "[hbp] build_plan: %lld host round trips so far on this context\n",
                     static_cast<long long>(c.syncs));
}

void pack_device(Ctx& c, DeviceCorpus& corpus, int64_t capacity, const hbp_strategy& st, uint64_t seed,
                 DevicePlan& out) {
    cudaStream_t s = c.stream;
    const u64 n = static_cast<u64>(corpus.n);
    // pack() checks, packing.cpp:211-225: strategy, capacity, then the first
    // sample that is too long or non-positive
    validate_strategy(st);
    if (capacity < 1) fail_validation("pack capacity must be >= 1");
    {
        u64 first_over = ~0ull;
        if (n > 0) {
            DevBuf<unsigned long long> over(1, s);
            const unsigned long long none = ~0ull;
            CUDA_CHECK(cudaMemcpyAsync(over.p, &none, sizeof(none), cudaMemcpyHostToDevice, s));
            const u32* lp = corpus.len32.p;
            unsigned long long* op = over.p;
            const u32 lim = capacity > 0x7fffffffLL ? 0x7fffffffu : static_cast<u32>(capacity);
            for_each_index(c, n, [=] __device__(u64 i) {
                if (lp[i] > lim) atomicMin(op, static_cast<unsigned long long>(i));
            });
            first_over = read_scalar(c, over.p);
            if (corpus.first_huge < first_over) first_over = corpus.first_huge;
        }
        const u64 first_bad = corpus.first_bad_len;
        if (first_over != ~0ull && first_over <= first_bad) {
            const i64 i = static_cast<i64>(first_over);
            fail_validation("sample " + std::to_string(corpus.id_of(i)) + " length " +
                            std::to_string(corpus.length_of(c, i)) + " exceeds pack capacity " +
                            std::to_string(capacity));
        }
        if (first_bad != ~0ull)
            fail_validation("sample " + std::to_string(corpus.id_of(static_cast<i64>(first_bad))) +
                            " has non-positive length");
    }
    if (capacity > 0x7fffffffLL) fail_validation("pack capacity exceeds the engine limit (2^31-1)");
    const u32 cap = static_cast<u32>(capacity);
    DevBuf<u64> entries(n + 1, s);
    DevBuf<u32> iota(n + 1, s);
    LAUNCH(k_iota, G(n), kB, 0, s, iota.p, n);
    LAUNCH(k_entries_from_idx, G(n), kB, 0, s, corpus.len32.p, iota.p, n, entries.p);
    PackedGroup pg;
    pack_pool(c, corpus, entries.p, n, cap, st, seed, pg);
    PackTable T;
    T.members.alloc(n + 1, s);
    T.moff.alloc(n + 1, s);
    T.cnt.alloc(n + 1, s);
    T.cap.alloc(n + 1, s);
    T.total.alloc(n + 1, s);
    T.att.alloc(n + 1, s);
    const u64 P = layout_group(c, pg, nullptr, 0, nullptr, nullptr, cap, T);
    // a pack list: packs in order, no iterations
    out.n_iterations = 0;
    out.n_devices = 0;
    out.n_packs = static_cast<int64_t>(P);
    out.n_members = static_cast<int64_t>(T.n_members);
    out.iter_group.alloc(1, s);
    out.iter_dev_offsets.alloc(1, s);
    out.dev_index.alloc(1, s);
    out.dev_pack_offsets.alloc(1, s);
    CUDA_CHECK(cudaMemsetAsync(out.iter_dev_offsets.p, 0, sizeof(int64_t), s));
    CUDA_CHECK(cudaMemsetAsync(out.dev_pack_offsets.p, 0, sizeof(int64_t), s));
    out.pack_capacity.alloc(P + 1, s);
    out.pack_total.alloc(P + 1, s);
    out.pack_attention.alloc(P + 1, s);
    out.pack_member_offsets.alloc(P + 1, s);
    out.member_index.alloc(T.n_members + 1, s);
    DevBuf<u32> pglobal(P + 1, s);
    LAUNCH(k_iota, G(P), kB, 0, s, pglobal.p, P);
    const u32* cntp = T.cnt.p;
    const u32* capp = T.cap.p;
    const u32* totp = T.total.p;
    const u64* attp = T.att.p;
    int64_t* oc = out.pack_capacity.p;
    int64_t* ot = out.pack_total.p;
    int64_t* oa = out.pack_attention.p;
    int64_t* om = out.pack_member_offsets.p;
    const i64 PP = static_cast<i64>(P);
    scan_exclusive<int64_t>(
        PP + 1, [=] __device__(i64 q) -> int64_t { return q < PP ? static_cast<int64_t>(cntp[q]) : 0; },
        [=] __device__(i64 q, int64_t v) {
            om[q] = v;
            if (q < PP) {
                oc[q] = capp[q];
                ot[q] = totp[q];
                oa[q] = static_cast<int64_t>(attp[q]);
            }
        },
        s, c.scan, "scan.plan5");
    if (P > 0)
        LAUNCH(k_out_members, grid_for(P * 8, kB, 148u * 64u), kB, 0, s, pglobal.p, P, out.pack_member_offsets.p,
               T.moff.p, T.cnt.p, T.members.p, out.member_index.p);
    CUDA_CHECK(cudaStreamSynchronize(s));
}

void plan_to_host(Ctx& c, DevicePlan& p) {
    if (p.on_host) return;
    const size_t I = static_cast<size_t>(p.n_iterations), D = static_cast<size_t>(p.n_devices),
                 P = static_cast<size_t>(p.n_packs), M = static_cast<size_t>(p.n_members);
    const size_t bytes = 8 * ((I + 1) + (I + 1) + (D + 1) + (D + 1) + 4 * (P + 1) + (P + 1) + (M + 1) / 2 + I / 8 + 10);
    if (!p.host.p) p.host = c.host_pool.acquire(bytes);
    char* cur = static_cast<char*>(p.host.p);
    auto cp = [&](auto*& h, auto& d, size_t n) {
        using T = std::remove_pointer_t<std::remove_reference_t<decltype(h)>>;
        h = reinterpret_cast<T*>(cur);
        cur += (sizeof(T) * n + 7) / 8 * 8;
        if (n) CUDA_CHECK(cudaMemcpyAsync(h, d.p, sizeof(T) * n, cudaMemcpyDeviceToHost, c.stream));
    };
    cp(p.h_iter_group, p.iter_group, I);
    cp(p.h_iter_dev_offsets, p.iter_dev_offsets, I + 1);
    cp(p.h_dev_index, p.dev_index, D);
    cp(p.h_dev_pack_offsets, p.dev_pack_offsets, D + 1);
    cp(p.h_pack_capacity, p.pack_capacity, P);
    cp(p.h_pack_total, p.pack_total, P);
    cp(p.h_pack_attention, p.pack_attention, P);
    cp(p.h_pack_member_offsets, p.pack_member_offsets, P + 1);
    cp(p.h_member_index, p.member_index, M);
    if (p.iter_phase.p) cp(p.h_iter_phase, p.iter_phase, I);
    else p.h_iter_phase = nullptr;
    CUDA_CHECK(cudaStreamSynchronize(c.stream));
    p.on_host = true;
}

// ---------------------------------------------------------------------------
// stand-alone stages over host pack lists (C++ / Python drop-in calls)
// ---------------------------------------------------------------------------

// leaves (max(0, capacity - total) << 32 | members) of host-listed packs
__global__ void k_fill_leaves(const int64_t* __restrict__ cap, const int64_t* __restrict__ off,
                              const int64_t* __restrict__ lens, u64 P, u64* __restrict__ leaves, u32* __restrict__ base) {
    for (u64 p = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; p < P;
         p += static_cast<u64>(gridDim.x) * blockDim.x) {
        int64_t tot = 0;
        for (int64_t k = off[p]; k < off[p + 1]; ++k) tot += lens[k];
        const int64_t r = cap[p] - tot;
        const u32 res = r <= 0 ? 0u : (r > 0x7fffffffLL ? 0x7fffffffu : static_cast<u32>(r));
        base[p] = static_cast<u32>(off[p + 1] - off[p]);
        leaves[p] = (static_cast<u64>(res) << 32) | base[p];
    }
}

// picks of one pool: count per pack, and the pool sample each placed item is
__global__ void k_fill_count(const u64* __restrict__ items, const u32* __restrict__ bin, u64 m, u32* __restrict__ cnt) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < m;
         i += static_cast<u64>(gridDim.x) * blockDim.x)
        if (bin[i] != kNone) atomicAdd(&cnt[bin[i]], 1u);
}

// pick k of pack p sits at added[off[p] + slot - base[p]] (slots count up
// from the pack's own members in pick order); its pool sample leaves the pool
__global__ void k_fill_place(const u64* __restrict__ items, const u32* __restrict__ bin, const u32* __restrict__ slot,
                             u64 m, const u32* __restrict__ base, const u64* __restrict__ off, int64_t* __restrict__ added,
                             u8* __restrict__ keep) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < m;
         i += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u32 b = bin[i];
        if (b == kNone) continue;
        const u32 pi = entry_idx(items[i]);
        added[off[b] + slot[i] - base[b]] = static_cast<int64_t>(pi);
        keep[pi] = 0;
    }
}

void greedy_fill_device(Ctx& c, i64 n_packs, const int64_t* pack_cap, const int64_t* pack_off, const int64_t* lens,
                        int n_pools, const int64_t* pool_off, const int64_t* pool_ids, const int64_t* pool_lens,
                        std::vector<int64_t>& added_off, std::vector<int64_t>& added, std::vector<uint8_t>& keep) {
    cudaStream_t s = c.stream;
    const i64 M = n_pools > 0 ? pool_off[n_pools] : 0;
    added_off.assign(static_cast<size_t>(n_packs) + 1, 0);
    added.clear();
    keep.assign(static_cast<size_t>(M), 1);
    if (n_packs == 0 || M == 0) return;
    // pool samples as one corpus: ids give the tie-break ranks
    hbp_samples in{pool_ids, pool_lens, M, HBP_MEM_HOST, "pools"};
    DeviceCorpus corpus;
    ingest(c, &in, corpus);
    // the packs' leaves, built on the device from the host pack list
    const u64 P = static_cast<u64>(n_packs);
    const u64 NM = static_cast<u64>(pack_off[n_packs]);
    DevBuf<int64_t> dcap(P, s), doff(P + 1, s), dlens(NM + 1, s);
    CUDA_CHECK(cudaMemcpyAsync(dcap.p, pack_cap, sizeof(int64_t) * P, cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaMemcpyAsync(doff.p, pack_off, sizeof(int64_t) * (P + 1), cudaMemcpyHostToDevice, s));
    if (NM) CUDA_CHECK(cudaMemcpyAsync(dlens.p, lens, sizeof(int64_t) * NM, cudaMemcpyHostToDevice, s));
    DevBuf<u64> dleaves(P, s);
    DevBuf<u32> base(P, s), cnt(P + 1, s);
    cnt.zero();
    LAUNCH(k_fill_leaves, G(P), kB, 0, s, dcap.p, doff.p, dlens.p, P, dleaves.p, base.p);
    // every pool's items (sorted) and their (pack, slot), nearest pool first;
    // pool-by-pool equals pack-by-pack (each pool is only consumed from)
    DevBuf<u64> items(static_cast<u64>(M), s);
    DevBuf<u32> bin(static_cast<u64>(M), s), slot(static_cast<u64>(M), s);
    DevBuf<u32> mx(1, s);
    for (int j = n_pools - 1; j >= 0; --j) {
        const u64 a = static_cast<u64>(pool_off[j]), m = static_cast<u64>(pool_off[j + 1] - pool_off[j]);
        if (m == 0) continue;
        u64* it = items.p + a;
        const u32* len32 = corpus.len32.p;
        u32* mxp = mx.p;
        mx.zero();
        for_each_index(c, m, [=] __device__(u64 i) {
            const u32 l = len32[a + i];
            it[i] = (static_cast<u64>(l) << 32) | static_cast<u64>(a + i);
            atomicMax(mxp, l);
        });
        const u32 maxlen = std::max<u32>(1u, read_scalar(c, mx.p));
        sort_entries(c, corpus, it, m, corpus.key32.p == nullptr, maxlen);
        first_fit_runs(c, it, static_cast<i64>(m), dleaves.p, n_packs, n_packs, 1u, FitMode::Fill, bin.p + a,
                       slot.p + a, corpus.key32.p, static_cast<u64>(corpus.neg_ids));
        LAUNCH(k_fill_count, G(m), kB, 0, s, it, bin.p + a, m, cnt.p);
    }
    // picks per pack -> offsets, then every pick at its place
    DevBuf<u64> off(P + 1, s);
    {
        const u32* cp = cnt.p;
        u64* op = off.p;
        const i64 NP = static_cast<i64>(P);
        scan_exclusive<u64>(
            NP + 1, [=] __device__(i64 i) { return i < NP ? static_cast<u64>(cp[i]) : 0ull; },
            [=] __device__(i64 i, u64 v) { op[i] = v; }, s, c.scan, "scan.fill_picks");
    }
    const u64 total = read_vector(c, off.p + P, 1)[0];
    DevBuf<int64_t> dadded(total + 1, s);
    DevBuf<u8> dkeep(static_cast<u64>(M), s);
    CUDA_CHECK(cudaMemsetAsync(dkeep.p, 1, static_cast<size_t>(M), s));
    LAUNCH(k_fill_place, G(static_cast<u64>(M)), kB, 0, s, items.p, bin.p, slot.p, static_cast<u64>(M), base.p, off.p,
           dadded.p, dkeep.p);
    const auto ho = read_vector(c, off.p, P + 1);
    for (u64 p = 0; p <= P; ++p) added_off[p] = static_cast<int64_t>(ho[p]);
    added.resize(total);
    if (total) CUDA_CHECK(cudaMemcpyAsync(added.data(), dadded.p, sizeof(int64_t) * total, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaMemcpyAsync(keep.data(), dkeep.p, static_cast<size_t>(M), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
}

void batching_device(Ctx& c, int64_t capacity, i64 n_packs, const int64_t* pack_cap, const int64_t* pack_off,
                     const int64_t* ids, const int64_t* lens, int32_t N, int32_t gi, bool random, uint64_t seed,
                     DevicePlan& out) {
    cudaStream_t s = c.stream;
    if (N < 1) fail_validation("device count must be >= 1");
    out.device_count = N;
    out.seed = seed;
    const i64 M = n_packs > 0 ? pack_off[n_packs] : 0;
    if (n_packs == 0) {
        PackTable T;
        DevBuf<u32> slots(1, s);
        DevBuf<int32_t> ig(1, s);
        emit_plan(c, T, slots, ig, 0, static_cast<u32>(N), seed, out, false);
        return;
    }
    hbp_samples in{ids, lens, M, HBP_MEM_HOST, "packs"};
    DeviceCorpus corpus;
    if (M > 0) ingest(c, &in, corpus);
    const u64 P = static_cast<u64>(n_packs);
    PackTable T;
    T.members.alloc(2 * static_cast<u64>(M) + 1, s);
    T.moff.alloc(P + N + 1, s);
    T.cnt.alloc(P + N + 1, s);
    T.cap.alloc(P + N + 1, s);
    T.total.alloc(P + N + 1, s);
    T.att.alloc(P + N + 1, s);
    std::vector<u64> hm(static_cast<size_t>(M)), moff(P);
    std::vector<u32> cnt(P), cap(P), tot(P);
    std::vector<u64> att(P);
    for (u64 p = 0; p < P; ++p) {
        moff[p] = static_cast<u64>(pack_off[p]);
        cnt[p] = static_cast<u32>(pack_off[p + 1] - pack_off[p]);
        cap[p] = static_cast<u32>(std::min<int64_t>(pack_cap[p], 0x7fffffff));
        int64_t t = 0, at = 0;
        for (int64_t k = pack_off[p]; k < pack_off[p + 1]; ++k) {
            t += lens[k];
            at += lens[k] * lens[k];
            hm[static_cast<size_t>(k)] = make_entry(static_cast<u32>(std::min<int64_t>(lens[k], 0x7fffffff)),
                                                    static_cast<u32>(k));
        }
        tot[p] = static_cast<u32>(t);
        att[p] = static_cast<u64>(at);
    }
    auto up = [&](auto* d, const auto& h) {
        if (!h.empty()) CUDA_CHECK(cudaMemcpyAsync(d, h.data(), sizeof(h[0]) * h.size(), cudaMemcpyHostToDevice, s));
    };
    up(T.members.p, hm);
    up(T.moff.p, moff);
    up(T.cnt.p, cnt);
    up(T.cap.p, cap);
    up(T.total.p, tot);
    up(T.att.p, att);
    T.n_packs = P;
    T.n_members = static_cast<u64>(M);
    const u64 max_iters = P / N + 2;
    DevBuf<u32> slots(max_iters * N, s);
    DevBuf<int32_t> igroup(max_iters, s);
    const u64 I = batch_group(c, corpus, T, 0, P, static_cast<u32>(N),
                              static_cast<u32>(std::min<int64_t>(capacity, 0x7fffffff)), gi, !random, seed, 0, slots,
                              igroup);
    emit_plan(c, T, slots, igroup, I, static_cast<u32>(N), seed, out, false);
    CUDA_CHECK(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------------------
// padded batching baselines (packing.cpp:265-317) and build_batching_plan
// (balance.cpp:260-298)
// ---------------------------------------------------------------------------

namespace {

__global__ void k_iota_entries(const u32* __restrict__ len32, u64 n, u64* __restrict__ e) {
    GRID_STRIDE(i, n) e[i] = make_entry(len32[i], static_cast<u32>(i));
}

__global__ void k_max_u32(const u32* __restrict__ v, u64 n, unsigned int* __restrict__ out) {
    u32 m = 0;
    GRID_STRIDE(i, n) m = max(m, v[i]);
    m = warp_max(m);
    if ((threadIdx.x & 31u) == 0) atomicMax(out, m);
}

// Batch starting at position i (budgeted_batches, packing.cpp:267-289): the
// first sample always, then the next while (count + 1) * max <= budget. In
// length-descending order the max is the first sample's length.
__global__ void k_batch_next(const u64* __restrict__ order, u64 n, u64 budget, bool sorted, u32* __restrict__ nxt) {
    GRID_STRIDE(i, n) {
        const u64 l0 = entry_len(order[i]);
        u64 j;
        if (sorted) {
            const u64 k = budget / l0;  // >= 1: budget >= every length
            j = i + k < n ? i + k : n;
        } else {
            u64 cnt = 1, mx = l0;
            j = i + 1;
            while (j < n) {
                const u64 l = entry_len(order[j]);
                const u64 nm = l > mx ? l : mx;
                if ((cnt + 1) * nm > budget) break;
                ++cnt;
                mx = nm;
                ++j;
            }
        }
        nxt[i] = static_cast<u32>(j);
    }
}

__global__ void k_batch_max(const u64* __restrict__ order, const u32* __restrict__ bstart, u64 nb, u64 n,
                            u32* __restrict__ bmax) {
    GRID_STRIDE(b, nb) {
        const u64 a = bstart[b], e = b + 1 < nb ? bstart[b + 1] : n;
        u32 m = 0;
        for (u64 k = a; k < e; ++k) m = max(m, entry_len(order[k]));
        bmax[b] = m;
    }
}

// One single-sample pack per row, padded to the batch max; device g of the
// plan holds batch g (balance.cpp:279-293).
__global__ void k_batching_packs(const u64* __restrict__ order, const u32* __restrict__ bidx,
                                 const u32* __restrict__ bmax, u64 n, int64_t* __restrict__ cap,
                                 int64_t* __restrict__ total, int64_t* __restrict__ att,
                                 int64_t* __restrict__ moff, int32_t* __restrict__ member) {
    GRID_STRIDE(p, n) {
        const u64 e = order[p];
        const int64_t l = entry_len(e);
        cap[p] = bmax[bidx[p]];
        total[p] = l;
        att[p] = l * l;
        moff[p] = static_cast<int64_t>(p);
        member[p] = static_cast<int32_t>(entry_idx(e));
        if (p + 1 == n) moff[n] = static_cast<int64_t>(n);
    }
}

__global__ void k_batching_devices(const u32* __restrict__ bstart, u64 nb, u64 n, u64 I, u32 N,
                                   int32_t* __restrict__ igroup, int64_t* __restrict__ idoff,
                                   int32_t* __restrict__ dindex, int64_t* __restrict__ dpoff) {
    GRID_STRIDE(g, I * N) {
        dpoff[g] = g < nb ? static_cast<int64_t>(bstart[g]) : static_cast<int64_t>(n);
        dindex[g] = static_cast<int32_t>(g % N);
        if (g % N == 0) {
            igroup[g / N] = 0;
            idoff[g / N] = static_cast<int64_t>(g);
        }
        if (g + 1 == I * N) {
            dpoff[I * N] = static_cast<int64_t>(n);
            idoff[I] = static_cast<int64_t>(I * N);
        }
    }
}

}  // namespace

void padded_batches_device(Ctx& c, const DeviceCorpus& corpus, int64_t budget, bool sorted, uint64_t seed,
                           PaddedBatches& out) {
    cudaStream_t s = c.stream;
    const u64 n = static_cast<u64>(corpus.n);
    // samples.max_length() vs the budget (packing.cpp:296-301, 309-314)
    int64_t longest = 0;
    if (n > 0) {
        DevBuf<unsigned int> mx(1, s);
        mx.zero();
        LAUNCH(k_max_u32, grid_for(n, 256, 148u * 8u), 256, 0, s, corpus.len32.p, n, mx.p);
        longest = read_scalar(c, mx.p);
        if (corpus.first_huge != ~0ull)  // lengths past 2^31 - 1 (len32 saturates): the exact maximum on the host
            for (u64 i = 0; i < n; ++i) longest = std::max<int64_t>(longest, corpus.length_of(c, static_cast<i64>(i)));
    }
    if (budget < longest)
        fail_validation("token budget " + std::to_string(budget) + " is below the longest sample (" +
                        std::to_string(longest) + ")");
    out.n = n;
    out.order.alloc(n + 1, s);
    out.n_batches = 0;
    if (n == 0) return;
    LAUNCH(k_iota_entries, G(n), kB, 0, s, corpus.len32.p, n, out.order.p);
    if (sorted) {
        sort_entries(c, corpus, out.order.p, n, corpus.key32.p == nullptr, static_cast<u32>(longest));
    } else {  // Rng(derive_seed(seed, "random-batching")).shuffle
        DevBuf<u32> src(n, s);
        DevBuf<u64> tmp(n, s);
        fy_source_positions(c, derive_seed(seed, "random-batching"), static_cast<i64>(n), src.p);
        gather_u64(c, out.order.p, src.p, tmp.p, static_cast<i64>(n));
        CUDA_CHECK(cudaMemcpyAsync(out.order.p, tmp.p, sizeof(u64) * n, cudaMemcpyDeviceToDevice, s));
    }
    DevBuf<u32> nxt(n, s), flags(chain_flag_words(n), s), tlast(chain_flag_words(n) / 64 + 1, s);
    LAUNCH(k_batch_next, G(n), kB, 0, s, out.order.p, n, static_cast<u64>(budget), sorted, nxt.p);
    chain_starts(c, nxt.p, n, flags.p, tlast.p);
    // batch starts (compacted) and every position's batch
    out.bstart.alloc(n + 1, s);
    out.bidx.alloc(n, s);
    DevBuf<u32> nb(1, s);
    {
        const u32* fl = flags.p;
        u32* bs = out.bstart.p;
        u32* bi = out.bidx.p;
        u32* nbp = nb.p;
        const i64 nn = static_cast<i64>(n);
        scan_exclusive_v<u32>(
            nn, [=] __device__(i64 i) { return (fl[i >> 5] >> (i & 31)) & 1u; },
            [=] __device__(i64 i, u32 v, u32 f) {
                if (f) bs[v] = static_cast<u32>(i);
                bi[i] = v + f - 1;
                if (i == nn - 1) *nbp = v + f;
            },
            s, c.scan, "scan.plan6");
    }
    out.n_batches = read_scalar(c, nb.p);
    out.bmax.alloc(out.n_batches + 1, s);
    LAUNCH(k_batch_max, G(out.n_batches), kB, 0, s, out.order.p, out.bstart.p, out.n_batches, n, out.bmax.p);
}

void batching_plan_device(Ctx& c, const DeviceCorpus& corpus, const hbp_group_config& group, int32_t device_count,
                          bool sorted, uint64_t seed, DevicePlan& out) {
    if (device_count < 1) fail_validation("device count must be >= 1");
    cudaStream_t s = c.stream;
    PaddedBatches pb;
    padded_batches_device(c, corpus, group.length, sorted, seed, pb);
    const u64 n = pb.n, B = pb.n_batches, N = static_cast<u64>(device_count);
    const u64 I = (B + N - 1) / N;
    out.device_count = device_count;
    out.seed = seed;
    out.groups = {group};
    out.l_best = out.l_max = group.length;  // HierarchicalGroups::single
    out.n_iterations = static_cast<int64_t>(I);
    out.n_devices = static_cast<int64_t>(I * N);
    out.n_packs = static_cast<int64_t>(n);
    out.n_members = static_cast<int64_t>(n);
    out.iter_group.alloc(I + 1, s);
    out.iter_dev_offsets.alloc(I + 1, s);
    out.dev_index.alloc(I * N + 1, s);
    out.dev_pack_offsets.alloc(I * N + 1, s);
    out.pack_capacity.alloc(n + 1, s);
    out.pack_total.alloc(n + 1, s);
    out.pack_attention.alloc(n + 1, s);
    out.pack_member_offsets.alloc(n + 1, s);
    out.member_index.alloc(n + 1, s);
    if (I == 0) {
        const int64_t zero = 0;
        CUDA_CHECK(cudaMemcpyAsync(out.iter_dev_offsets.p, &zero, sizeof(zero), cudaMemcpyHostToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(out.pack_member_offsets.p, &zero, sizeof(zero), cudaMemcpyHostToDevice, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        return;
    }
    LAUNCH(k_batching_devices, G(I * N), kB, 0, s, pb.bstart.p, B, n, I, static_cast<u32>(N), out.iter_group.p,
           out.iter_dev_offsets.p, out.dev_index.p, out.dev_pack_offsets.p);
    LAUNCH(k_batching_packs, G(n), kB, 0, s, pb.order.p, pb.bidx.p, pb.bmax.p, n, out.pack_capacity.p,
           out.pack_total.p, out.pack_attention.p, out.pack_member_offsets.p, out.member_index.p);
    CUDA_CHECK(cudaStreamSynchronize(s));
}

}  // namespace hbp_b200
