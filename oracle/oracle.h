/*
 * oracle.h — TEST INFRASTRUCTURE ONLY. Never linked or called by the product.
 *
 * One C ABI implemented twice:
 *   - oracle/hbp_oracle.c : a plain-C sequential restatement of the
 *     reference planner (/root/reference/proj/src), built into
 *     oracle/liboracle_hbp.so;
 *   - oracle/ref_shim.cpp : a thin shim over the reference sources compiled
 *     in place (namespace renamed hbp -> hbp_ref), built into
 *     oracle/_ref/libhbp_ref.so when /root/reference is present.
 * Tests load either library with ctypes and call the same functions, so the
 * restatement is pinned against the real reference, and the CUDA engine is
 * checked against both. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load these libraries.
 *
 * All functions return 0 / 2 (ValidationError) / 3 (InfeasibleError) /
 * 4 (IoError) and copy the exception text into err[errlen].
 */
#ifndef HBP_ORACLE_H
#define HBP_ORACLE_H

#include <stdint.h>

#include "../include/hbp_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* A flat plan / pack list / pool list with explicit sample ids, malloc'd by
 * the library. Pack lists and pools have no iterations or devices. */
typedef struct oracle_plan {
    int32_t device_count;
    uint64_t seed;
    int64_t n_iterations;
    int64_t n_devices;
    int64_t n_packs;
    int64_t n_members;
    int32_t* iter_group;
    int64_t* iter_dev_offsets;
    int32_t* dev_index;
    int64_t* dev_pack_offsets;
    int64_t* pack_capacity;
    int64_t* pack_total;
    int64_t* pack_attention;
    int64_t* pack_member_offsets;
    int64_t* member_id;
    int64_t* member_length;
} oracle_plan;

void oracle_plan_free(oracle_plan* p);
/* 1 for the restatement, 2 for the compiled reference. */
int oracle_kind(void);

/* synth_lengths as bound in bindings/py_hbp.cpp:80-97 (long_dist "" ->
 * short_dist), generator ingest.cpp:279-329. lengths[count]; ids 0..n-1. */
int oracle_synth_lengths(int64_t count, const char* short_dist,
                         double long_fraction, const char* long_dist,
                         int64_t max_length, uint64_t seed, int64_t* lengths,
                         char* err, int errlen);
/* Rng(seed).shuffle (rng.hpp:61-68) of 0..m-1: out[p] = original position. */
int oracle_shuffle_positions(uint64_t seed, int64_t m, uint32_t* out);
/* types.cpp:8-24 */
int oracle_validate(const int64_t* ids, const int64_t* lengths, int64_t n,
                    char* err, int errlen);
/* types.cpp:52-72 */
int oracle_fingerprint(const int64_t* ids, const int64_t* lengths, int64_t n,
                       uint64_t* hash, int64_t* count, int64_t* tokens);
/* balance.cpp:25-44: one "pack" per group (capacity = group length). */
int oracle_group_data(const int64_t* ids, const int64_t* lengths, int64_t n,
                      const hbp_groups* groups, oracle_plan** out, char* err,
                      int errlen);
/* packing.cpp:210-261 */
int oracle_pack(const int64_t* ids, const int64_t* lengths, int64_t n,
                int64_t capacity, const hbp_strategy* strategy, uint64_t seed,
                oracle_plan** out, char* err, int errlen);
/* balance.cpp:46-101; pools as one "pack" per pool. */
int oracle_greedy_fill(const oracle_plan* packs, const oracle_plan* pools,
                       oracle_plan** out_packs, oracle_plan** out_pools,
                       char* err, int errlen);
/* balance.cpp:180-205 */
int oracle_balance_batching(const oracle_plan* packs, int32_t device_count,
                            int32_t group_index, int32_t sp_comm,
                            int32_t random_batching, uint64_t seed,
                            oracle_plan** out, char* err, int errlen);
/* balance.cpp:207-258 */
int oracle_build_plan(const int64_t* ids, const int64_t* lengths, int64_t n,
                      const hbp_groups* groups, const hbp_plan_options* options,
                      oracle_plan** out, char* err, int errlen);
/* metrics.cpp:107-144 */
int oracle_report(const hbp_plan_view* plan, hbp_metrics* out, double* dbr,
                  double* abr, char* err, int errlen);
/* sim.cpp:9-60 (no fingerprint) */
int oracle_simulate(const hbp_plan_view* plan,
                    const hbp_hardware_profile* profile, hbp_sim_totals* out,
                    double* iteration_seconds, double* device_compute,
                    double* device_comm, double* device_idle, char* err,
                    int errlen);
/* costmodel.cpp:37-53 */
int oracle_memory_used(int64_t length, int32_t sp, int32_t ckpt,
                       const hbp_hardware_profile* profile, int64_t* out,
                       char* err, int errlen);
/* costmodel.cpp:55-104 over explicit packs */
int oracle_iter_time(const int64_t* capacity, const int64_t* total,
                     const int64_t* attention, int64_t n_packs, int32_t sp,
                     int32_t ckpt, const hbp_hardware_profile* profile,
                     double* out, char* err, int errlen);
/* costmodel.cpp:110-138, 144-265: profile_time / profile_memory /
 * derive_ckpt of an analytic or table profiler. */
int oracle_profile_time(const hbp_profiler* profiler, int64_t length,
                        int32_t sp, int32_t ckpt, double* out, char* err,
                        int errlen);
int oracle_profile_memory(const hbp_profiler* profiler, int64_t length,
                          int32_t sp, int32_t ckpt, int64_t* out, char* err,
                          int errlen);
int oracle_derive_ckpt(const hbp_profiler* profiler, int64_t length,
                       int32_t sp, int32_t* out, char* err, int errlen);
/* costmodel.cpp:271-292 */
int oracle_greedy_profile_ckpt(const hbp_profiler* profiler, int64_t length,
                               int32_t sp, int32_t ckpt_min, int32_t ckpt_max,
                               int32_t* out, char* err, int errlen);
/* costmodel.cpp:294-325 */
int oracle_find_best_sp_ckpt(const hbp_profiler* profiler, int64_t length,
                             const int32_t* sp, int32_t n_sp, int32_t* out_sp,
                             int32_t* out_ckpt, double* out_seconds,
                             char* err, int errlen);
/* autoselect.cpp:76-168 */
int oracle_select_groups(const int64_t* lengths, int32_t n_lengths,
                         const hbp_profiler* profiler, const int32_t* sp,
                         int32_t n_sp, hbp_group_config* out_groups,
                         int32_t* out_count, int64_t* out_l_best,
                         int64_t* out_l_max, char* err, int errlen);
/* simulate(build_plan(...)).total_seconds per
 * candidate, +inf on InfeasibleError, argmin lowest index. */
int oracle_sweep(const int64_t* ids, const int64_t* lengths, int64_t n,
                 const hbp_group_config* cand_groups,
                 const int64_t* cand_offsets, const int64_t* cand_l_best,
                 int64_t n_candidates, const hbp_plan_options* options,
                 const hbp_hardware_profile* profile, double* out_seconds,
                 int64_t* out_best, char* err, int errlen);

#ifdef __cplusplus
}
#endif

#endif /* HBP_ORACLE_H */
