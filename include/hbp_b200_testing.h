/*
 * hbp_b200_testing.h — stage-level entry points exported for parity tests.
 *
 * Each exposes one engine stage on its own so tests can check it against
 * the oracle in isolation (the full path is in hbp_b200.h). All buffers are
 * host memory; every call runs the CUDA stage on the context's device.
 */
#ifndef HBP_B200_TESTING_H
#define HBP_B200_TESTING_H

#include <stdint.h>

#include "hbp_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Rng(seed).shuffle over m elements (rng.hpp:61-68): out_src[p] is the
 * original position of the element that lands at p. */
int hbp_test_shuffle_positions(hbp_ctx* ctx, uint64_t seed, int64_t m, uint32_t* out_src);

/* Exclusive prefix sum of n uint32 values into uint64 (decoupled look-back). */
int hbp_test_scan_u32(hbp_ctx* ctx, const uint32_t* in, int64_t n, uint64_t* out);

/* Stable LSD radix sort of (key, value) pairs by key, ascending or
 * descending, over the low `bits` bits of the key. */
int hbp_test_radix_sort(hbp_ctx* ctx, uint32_t* keys, uint32_t* values, int64_t n, int32_t bits,
                        int32_t descending);

/* Every later Fisher-Yates on this context treats the first draw of step
 * `step` as rejected (0: none), exercising the repair of a rejected draw
 * (probability < m / 2^64 in real runs). */
int hbp_test_set_force_reject(hbp_ctx* ctx, uint64_t step);

/* The candidates rank `rank` of `world` evaluates in hbp_sweep_sharded
 * (ascending global indices; out_idx holds n_candidates entries). Host only. */
int hbp_test_sweep_shard(const hbp_group_config* cand_groups, const int64_t* cand_offsets, int64_t n_candidates,
                         int32_t rank, int32_t world, int64_t* out_idx, int64_t* out_n);

#ifdef __cplusplus
}
#endif

#endif /* HBP_B200_TESTING_H */
