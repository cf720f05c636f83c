// radix.cuh — stable LSD radix sort entry point (radix.cu).
#pragma once

#include "engine.cuh"

namespace hbp_b200 {

// Sorts (keys, vals) stably by the low `bits` bits of keys, in place.
// tmp_* may be null (allocated internally) or n-element scratch.
void radix_sort_pairs(Ctx& c, u32* keys, u32* vals, i64 n, int bits, bool descending, u32* tmp_keys = nullptr,
                      u32* tmp_vals = nullptr);

// Entries (len << 32 | idx) sorted by (length desc, key asc) in one launch
// when n is small (one CTA): by key (key32[idx], or idx when null) over
// key_bits first when key_bits > 0, then by length over len_bits. Returns
// false (nothing done) when n is too large.
bool sort_entries_small(Ctx& c, u64* e, i64 n, const u32* key32, int key_bits, int len_bits);

}  // namespace hbp_b200
