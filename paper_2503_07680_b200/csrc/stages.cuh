// stages.cuh — device data layouts shared between stages and the stage
// entry points (nextfit.cu, firstfit.cu, batching.cu, metrics.cu).
//
// Sample entries travel as one u64: (length << 32) | sample_index, so a
// shuffle or compaction moves length and identity together (one 8-byte
// gather instead of two dependent 4-byte ones). Sample ids only matter for
// tie-breaks; the engine orders by input index, which equals id order when
// the ids are ascending in input order (checked at ingest) and is replaced
// by the id rank otherwise.
#pragma once

#include <vector>

#include "engine.cuh"

namespace hbp_b200 {

__host__ __device__ __forceinline__ u64 make_entry(u32 len, u32 idx) { return (static_cast<u64>(len) << 32) | idx; }
__host__ __device__ __forceinline__ u32 entry_len(u64 e) { return static_cast<u32>(e >> 32); }
__host__ __device__ __forceinline__ u32 entry_idx(u64 e) { return static_cast<u32>(e); }

// Append-only pack list in device memory (frozen ISF packs).
struct PackSink {
    u64* members;     // entries
    u64* pack_off;    // first member of each pack
    u32* pack_total;
    u64* n_members;   // device counters
    u64* n_packs;
};

// nextfit.cu: next-fit over F, freeze packs with total >= tmin into sink
// (after the n_members / n_packs it already holds; both updated), the rest
// (in pack order) into newpool. Returns the new pool size.
// Starts of the chain 0 -> nxt[0] -> ... (nxt monotone, nxt[s] > s) as bits:
// chain_flag_words(m) u32 words (tiles of 2048 positions); tlast[tile] =
// 1 + the tile's last start (0: none), chain_flag_words(m) / 64 entries.
u64 chain_flag_words(u64 m);
void chain_starts(Ctx& c, const u32* nxt, u64 m, u32* flags, u32* tlast);

// shuffle.cu: every ISF round of a pool of up to 64K samples in one launch
// (one cluster: the shuffle, then the next-fit round tile by tile); the
// remainder back in A, cur / n_members / n_packs updated (one read). False
// (nothing done) for larger pools.
bool isf_small(Ctx& c, const std::vector<uint64_t>& seeds, u64* A, u64& cur, u32 cap, u64 tmin, PackSink sink,
               u64& n_members, u64& n_packs);

i64 nextfit_freeze(Ctx& c, const u64* F, i64 m, u32 cap, u64 tmin, PackSink sink, u64* newpool, u64& n_members,
                   u64& n_packs, const u64* P_in = nullptr);

// ---- first-fit by runs (firstfit.cu) -------------------------------------
//
// Items sorted by (length desc, id asc) are grouped into runs of equal
// length. A run of c items of size s goes, in bin order, to every bin with
// residual >= s (floor(r / s) items each) until the run is used up; what is
// left either opens new bins of floor(cap / s) items (FFD, packing.cpp:
// 86-103 over sort_decreasing) or stays unassigned (greedy fill,
// balance.cpp:62-101: every pack repeatedly takes the largest fitting
// sample, lowest id first -- the same assignment processed length by
// length). One warp walks the runs over a 32-ary max-residual tree.
struct FitRecords {
    // item range [item, item + count) -> bins bin + k / per_bin, slots
    // slot0 + k % per_bin
    u32* item;
    u32* count;
    u32* bin;
    u32* per_bin;
    u32* slot0;
};

struct FitResult {
    i64 bins = 0;     // bins after the run (existing + opened)
    i64 records = 0;
};

enum class FitMode { Ffd, Fill };

// `leaves` (capacity max_bins) holds (residual << 32 | count) per bin; the
// first `bins0` are live. items: sorted entries. Writes item -> (bin, slot),
// kNone for items left unassigned (fill mode).
// Fill mode with sample ids <= -2 (neg_keys > 0: the items whose tie-break
// key -- key32[idx], or idx when key32 is null -- is below neg_keys): the
// reference's probe {residual, id = -1} (balance.cpp:82-83) makes such a
// sample ineligible when its length equals the residual exactly. Runs then
// split at the id class and the negative part of each length is "strict":
// a bin with residual r takes floor((r - 1) / s) of its items, and the
// non-negative part after it the usual floor(r' / s) -- the reference's
// pack-by-pack picks, run by run (flag: bit 31 of run_len).
// The runs of equal length of sorted items (first item, length | strict
// bit 31, and their count in n_runs[0]): computed by first_fit_runs, or
// ahead of it (prepare_runs, no host sync) -- e.g. on the side stream while
// the bins are still being built. Buffers sized by the caller (n items).
struct FitRuns {
    u32* run_item = nullptr;
    u32* run_len = nullptr;
    u32* n_runs = nullptr;  // device scalar (4 words: the tree engines reuse it)
};
void prepare_runs(Ctx& c, const u64* items, i64 n_items, const u32* key32, u64 neg_keys, FitRuns r);

FitResult first_fit_runs(Ctx& c, const u64* items, i64 n_items, u64* leaves, i64 bins0, i64 max_bins, u32 cap,
                         FitMode mode, u32* item_bin, u32* item_slot, const u32* key32 = nullptr, u64 neg_keys = 0,
                         const FitRuns* pre = nullptr);

// scanfit.cu: best fit (worst = false, packing.cpp:105-127) or the
// emptiest-pack rule of SPFHP (worst = true, packing.cpp:129-162) of the
// items in the given order into fresh bins; same outputs as first_fit_runs.
FitResult scan_fit(Ctx& c, const u64* items, i64 n, u64* leaves, i64 max_bins, u32 cap, bool worst, u32* item_bin,
                   u32* item_slot);

// chain.cu: first fit as a pipeline of bins. Bin b sees the items no bin
// before it took, in order, and takes each one that fits, so bins form a
// systolic chain: warp j owns 32 * m consecutive bins and passes, per run,
// the count its bins left to warp j + 1. Runs [run_begin, run_end).
struct ChainRuns {
    const u32* run_item;
    const u32* run_len;
    u32 n_items, n_runs, run_begin, run_end;
};
// Bins [0, live) hold `leaves`; FFD: bins [live, n_bins) start empty
// (residual cap). Bins are covered by as many resident-chain passes as
// needed (the first sized by first_pass_bins when non-zero). `used` = 1 + the
// highest bin holding items. `take` (n_items, zeroed; pre-placed items marked
// as heads with take 1 and their bin/slot) is scratch for the head expansion.
bool chain_fit(Ctx& c, const ChainRuns& runs, u64* leaves, u32 live, u32 n_bins, u32 cap, bool ffd, u32* item_bin,
               u32* item_slot, u32* take, u32 first_pass_bins, u32& used, bool expand = true);
// Heads (item_bin / item_slot / take at each take's first item) -> every item.
void expand_heads(Ctx& c, u64 n, u32* item_bin, u32* item_slot, const u32* take);

// item -> (bin, slot) for every item covered by a record; others get kNone.
void expand_fit_records(Ctx& c, FitRecords rec, i64 n_records, i64 n_items, u32* item_bin, u32* item_slot);

}  // namespace hbp_b200
