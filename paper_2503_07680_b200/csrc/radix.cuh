// radix.cuh — stable LSD radix sort entry point (radix.cu).
#pragma once

#include "engine.cuh"

namespace hbp_b200 {

// Sorts (keys, vals) stably by the low `bits` bits of keys, in place.
// tmp_* may be null (allocated internally) or n-element scratch.
void radix_sort_pairs(Ctx& c, u32* keys, u32* vals, i64 n, int bits, bool descending, u32* tmp_keys = nullptr,
                      u32* tmp_vals = nullptr);

}  // namespace hbp_b200
