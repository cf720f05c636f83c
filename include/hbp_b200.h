/*
 * hbp_b200.h — C-ABI of the B200 batch-construction engine for Hierarchical
 * Balance Packing (arXiv 2503.07680).
 *
 * Plain pointers and sizes only: no C++ or torch types cross this boundary.
 * Every entry point replaces one reference C++ entry point of
 * /root/reference/proj (cited per function, path:line relative to proj/).
 * The C++ drop-in headers under include/hbp/ and the Python module wrap
 * these calls; INTEGRATION.md shows the bindings a maintainer would add.
 *
 * Status codes mirror the reference CLI exit codes (tools/hbp_main.cpp:38-40):
 *   0 ok, 2 ValidationError, 3 InfeasibleError, 4 IoError; 5 is a CUDA or
 *   internal failure (never silently recovered; there is no CPU path).
 * The message of the last failure on a context is hbp_last_error(ctx); the
 * text is the exact message the reference would throw.
 *
 * Threading: one hbp_ctx owns one CUDA stream and its scratch; contexts are
 * independent, a single context must not be used from two threads at once
 * (the reference is single-threaded and reentrant).
 */
#ifndef HBP_B200_H
#define HBP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HBP_B200_ABI_VERSION 1

enum hbp_status {
    HBP_OK = 0,
    HBP_ERR_VALIDATION = 2,
    HBP_ERR_INFEASIBLE = 3,
    HBP_ERR_IO = 4,
    HBP_ERR_CUDA = 5,
    /* a JSON key or type error the reference raises as nlohmann::json::exception
       (plan_from_json, io.cpp:112-160); the message is the library's what() */
    HBP_ERR_JSON = 6
};

/* Same order as hbp::StrategyKind (include/hbp/packing.hpp:17). */
enum hbp_strategy_kind {
    HBP_STRATEGY_RANDOM = 0,
    HBP_STRATEGY_ISF = 1,
    HBP_STRATEGY_FFS = 2,
    HBP_STRATEGY_FFD = 3,
    HBP_STRATEGY_BFS = 4,
    HBP_STRATEGY_SPFHP = 5
};

/* Where a caller-provided buffer lives. */
enum hbp_memory { HBP_MEM_HOST = 0, HBP_MEM_DEVICE = 1 };

/* hbp::GroupConfig (autoselect.hpp:13-18) flattened with its RuntimeConfig
 * (costmodel.hpp:20-25). */
typedef struct hbp_group_config {
    int64_t length;
    int32_t sp;
    int32_t ckpt;
} hbp_group_config;

/* hbp::HierarchicalGroups (autoselect.hpp:20-27). */
typedef struct hbp_groups {
    const hbp_group_config* groups;
    int32_t count;
    int64_t l_best;
    int64_t l_max;
} hbp_groups;

/* hbp::PackingStrategy (packing.hpp:22-30). */
typedef struct hbp_strategy {
    int32_t kind;             /* hbp_strategy_kind */
    int32_t isf_iterations;   /* reference default 8 */
    double isf_fill_threshold; /* reference default 0.98 */
} hbp_strategy;

/* hbp::PlanOptions (balance.hpp:64-70). */
typedef struct hbp_plan_options {
    hbp_strategy strategy;
    int32_t device_count;
    int32_t balance_batching; /* 0 -> random pack batching */
    int32_t greedy_fill;
    uint64_t seed;
} hbp_plan_options;

/* hbp::HardwareProfile (costmodel.hpp:31-47). */
typedef struct hbp_hardware_profile {
    double per_token_linear_cost;
    double per_token2_attention_cost;
    double sp_comm_cost;
    double gc_recompute_factor;
    double fixed_iteration_cost;
    int32_t layer_count;
    int64_t base_memory;
    double per_token_activation_memory;
    double gc_memory_saving_per_layer;
    int64_t reference_length;
    int64_t device_memory;
} hbp_hardware_profile;

/* The reference's HardwareProfile{} defaults (costmodel.hpp:32-43). */
void hbp_hardware_profile_defaults(hbp_hardware_profile* out);

/* Input corpus: reference SampleSet (types.hpp:24-46) as two parallel
 * arrays. ids == NULL means ids 0..n-1 in order (what the Python
 * SampleSet(lengths) constructor builds, bindings/py_hbp.cpp:25-35).
 * `memory` says where ids/lengths live. */
typedef struct hbp_samples {
    const int64_t* ids;
    const int64_t* lengths;
    int64_t n;
    int32_t memory;     /* hbp_memory */
    const char* source; /* SampleSet::source, used in "empty corpus: <source>"; may be NULL */
} hbp_samples;

/*
 * Flat plan: CSR of iterations -> device batches -> packs -> members.
 * Mirrors hbp::Plan / Iteration / DeviceBatch / Pack (balance.hpp:18-37,
 * metrics.hpp:16-35). member_index[] indexes the input sample arrays; it may
 * be NULL in plans handed to hbp_report / hbp_simulate, which only read pack
 * totals. All arrays are host memory.
 */
typedef struct hbp_plan_view {
    int32_t device_count;
    uint64_t seed;
    hbp_groups groups;
    int64_t n_iterations;
    int64_t n_devices;
    int64_t n_packs;
    int64_t n_members;
    const int32_t* iter_group;          /* [n_iterations] */
    const int64_t* iter_dev_offsets;    /* [n_iterations + 1] */
    const int32_t* dev_index;           /* [n_devices] */
    const int64_t* dev_pack_offsets;    /* [n_devices + 1] */
    const int64_t* pack_capacity;       /* [n_packs] */
    const int64_t* pack_total;          /* [n_packs] */
    const int64_t* pack_attention;      /* [n_packs] */
    const int64_t* pack_member_offsets; /* [n_packs + 1] */
    const int32_t* member_index;        /* [n_members] */
    const int8_t* iter_phase;           /* [n_iterations]: 1 = warmup (curriculum_order); NULL: all hybrid */
} hbp_plan_view;

/* hbp::MetricsReport headline numbers (metrics.hpp:67-74). */
typedef struct hbp_metrics {
    double dbr;
    double pr;
    double abr;
    double cr;
    double ave_t;
} hbp_metrics;

/* hbp::SimReport scalars (sim.hpp:38-47). */
typedef struct hbp_sim_totals {
    double total_seconds;
    double gpu_days;
    int32_t switch_count;
    int32_t device_count;
    hbp_metrics metrics;
} hbp_sim_totals;

/* One measured profile row, hbp::ProfileRow (costmodel.hpp:114-121). */
typedef struct hbp_profile_row {
    int64_t length;
    int32_t sp;
    int32_t ckpt;
    int64_t memory_bytes;
    double seconds;
    int32_t oom;
} hbp_profile_row;

enum hbp_profiler_kind { HBP_PROFILER_ANALYTIC = 0, HBP_PROFILER_TABLE = 1 };

/* AnalyticProfiler (costmodel.hpp:96-111) or TableProfiler (:123-147). */
typedef struct hbp_profiler {
    int32_t kind;
    hbp_hardware_profile profile; /* analytic */
    int32_t ckpt_min;             /* analytic, default 0 */
    int32_t ckpt_max;             /* analytic, -1 -> layer_count */
    const hbp_profile_row* rows;  /* table */
    int64_t n_rows;
    int64_t device_memory;        /* table, default 80 GiB */
} hbp_profiler;

/* ---- context ---------------------------------------------------------- */

typedef struct hbp_ctx hbp_ctx;
typedef struct hbp_plan hbp_plan; /* device-resident plan (opaque) */

int hbp_ctx_create(int device, hbp_ctx** out);
void hbp_ctx_destroy(hbp_ctx* ctx);
const char* hbp_last_error(const hbp_ctx* ctx);
/* Blocks until all work queued on the context's stream has finished. */
int hbp_ctx_synchronize(hbp_ctx* ctx);
/* The cudaStream_t the context launches on, as an opaque pointer. */
void* hbp_ctx_stream(hbp_ctx* ctx);
/* Kernel launches issued on this context since creation (for the bench). */
int64_t hbp_ctx_launch_count(const hbp_ctx* ctx);
/* Kernel profiling: while on, every engine launch is bracketed by CUDA
 * events on the context stream and tagged with its kernel family and
 * algorithmic bytes. hbp_ctx_stage_stats(index) reports per family the
 * summed device time, launch count and algorithmic bytes; it returns
 * HBP_ERR_VALIDATION past the last family. */
int hbp_ctx_set_profiling(hbp_ctx* ctx, int32_t on);
int hbp_ctx_stage_stats(hbp_ctx* ctx, int32_t index, char* name, int32_t name_len, double* ms, int64_t* launches,
                        double* bytes);

/* ---- L1: synthetic corpora (input generation, host threads) -------------- */

/* synth_lengths as bound by the reference Python module
 * (bindings/py_hbp.cpp:80-97; generator src/ingest.cpp:279-329): long_dist
 * NULL or "" reuses short_dist. Bit-identical to the reference on the same
 * libm. out_lengths[count]; ids are 0..count-1. */
int hbp_synth_lengths(int64_t count, const char* short_dist, double long_fraction, const char* long_dist,
                      int64_t max_length, uint64_t seed, int64_t* out_lengths, char* err, int errlen);

/* ---- L1: corpus files ----------------------------------------------------- */

enum hbp_corpus_format { HBP_CORPUS_JSONL = 0, HBP_CORPUS_CSV = 1, HBP_CORPUS_RAW = 2 };

/* load_lengths(istream, format, source) (include/hbp/ingest.hpp:23-24,
 * src/ingest.cpp:57-160) over the bytes of a corpus file already read into
 * host memory (the reference reads an istream), parsed on the GPU.
 * Errors are the reference's: the first malformed line in file order
 * ("line N: not an integer length: '...'", "... trailing garbage ...",
 * "... length must be >= 1, got V", "... too few columns",
 * "... invalid JSON: <nlohmann parse_error text>", "... expected object
 * with integer \"length\"", the CSV header message, "empty corpus:
 * <source>"), then SampleSet::validate (duplicate explicit JSONL ids).
 * Ids are the record index unless a JSONL record has an integer "id".
 * out_ids (may be NULL) and out_lengths (`out_memory`) hold `capacity`
 * entries: (bytes + 1) / 2 always suffices. *out_count = n. */
int hbp_load_lengths(hbp_ctx* ctx, const char* text, int64_t bytes, int32_t format, const char* source,
                     int64_t* out_ids, int64_t* out_lengths, int64_t capacity, int32_t out_memory,
                     int64_t* out_count);

/* ---- L0: validation ---------------------------------------------------- */

/* SampleSet::validate (src/types.cpp:8-24): non-empty, length >= 1, unique
 * ids; the first offending sample in input order is reported. */
int hbp_validate(hbp_ctx* ctx, const hbp_samples* samples);

/* ---- L2: hot path ------------------------------------------------------ */

/* group_data (include/hbp/balance.hpp:42-43, src/balance.cpp:25-44).
 * Writes group_offsets[groups->count + 1] and member_index[n]: the samples
 * of group g, in input order, are member_index[group_offsets[g] ..
 * group_offsets[g+1]). Host output buffers. */
int hbp_group_data(hbp_ctx* ctx, const hbp_samples* samples,
                   const hbp_groups* groups, int64_t* group_offsets,
                   int32_t* member_index);

/* pack (include/hbp/packing.hpp:46-47, src/packing.cpp:210-261). The result
 * is a plan with no iterations: n_packs packs, capacity == `capacity`. */
int hbp_pack(hbp_ctx* ctx, const hbp_samples* samples, int64_t capacity,
             const hbp_strategy* strategy, uint64_t seed, hbp_plan** out);

/* A host pack list: pack p holds samples [pack_offsets[p], pack_offsets[p+1])
 * of ids/lengths, with its own capacity. */
typedef struct hbp_packs_in {
    int64_t n_packs;
    const int64_t* pack_offsets; /* [n_packs + 1] */
    const int64_t* pack_capacity; /* [n_packs] */
    const int64_t* ids;
    const int64_t* lengths;
} hbp_packs_in;

/* greedy_fill (include/hbp/balance.hpp:48, src/balance.cpp:46-101). Pools
 * are n_pools sample lists (pool_offsets[n_pools + 1]) ordered smallest
 * group first, as in the reference. Outputs: out_added_offsets[n_packs + 1]
 * and out_added[] (capacity: total pool samples) list, per pack and in pick
 * order, the flattened pool index of every sample it takes;
 * out_pool_keep[total pool samples] is 1 for samples left in their pool. */
int hbp_greedy_fill(hbp_ctx* ctx, const hbp_packs_in* packs, int32_t n_pools, const int64_t* pool_offsets,
                    const int64_t* pool_ids, const int64_t* pool_lengths, int64_t* out_added_offsets,
                    int64_t* out_added, uint8_t* out_pool_keep);

/* balance_batching / random_pack_batching (include/hbp/balance.hpp:55-62,
 * src/balance.cpp:105-205) over a host pack list of common `capacity`
 * (PackList::capacity). The result is a plan without the plan shuffle; its
 * member_index[] indexes packs->ids / packs->lengths. */
int hbp_balance_batching(hbp_ctx* ctx, const hbp_packs_in* packs, int64_t capacity, int32_t device_count,
                         int32_t group_index, int32_t random_batching, uint64_t seed, hbp_plan** out);

/* build_plan (include/hbp/balance.hpp:75-76, src/balance.cpp:207-258). */
int hbp_build_plan(hbp_ctx* ctx, const hbp_samples* samples,
                   const hbp_groups* groups, const hbp_plan_options* options,
                   hbp_plan** out);

/* Host view of a plan produced by hbp_pack / hbp_build_plan. The first call
 * copies the plan to host; the view stays valid until hbp_plan_free. */
int hbp_plan_view_get(hbp_ctx* ctx, hbp_plan* plan, hbp_plan_view* out);

/* Report / simulate sharded by data-parallel column.
 * Per-iteration DEVICE buffers (n_iterations entries each) the caller
 * allocates and all-reduces between the calls:
 *   phase 0 on columns [col0, col1): tmax, amax, busy (all-reduce MAX),
 *           tokens, pad_gap, pad_cap (SUM), sim_err (one int64, MIN);
 *   phase 1: tgap, agap (SUM);
 *   finish:  metrics and simulate totals, bit-identical to hbp_report_plan /
 *            hbp_simulate_plan on the whole plan (gaps are integers).
 * profile NULL: report only (busy and sim_err may be NULL). */
typedef struct hbp_eval_columns_bufs {
    int64_t* tmax;
    int64_t* amax;
    int64_t* tokens;
    int64_t* pad_gap;
    int64_t* pad_cap;
    double* busy;
    int64_t* tgap;
    int64_t* agap;
    int64_t* sim_err;
} hbp_eval_columns_bufs;

int hbp_eval_columns(hbp_ctx* ctx, hbp_plan* plan, int32_t phase, int32_t col0, int32_t col1,
                     const hbp_hardware_profile* profile, const hbp_eval_columns_bufs* bufs);
int hbp_eval_columns_finish(hbp_ctx* ctx, hbp_plan* plan, const hbp_hardware_profile* profile,
                            const hbp_eval_columns_bufs* bufs, hbp_metrics* out, hbp_sim_totals* sim);

/* Padded-batching baselines. */
enum { HBP_BATCHING_SORTED = 0, HBP_BATCHING_RANDOM = 1 };

/* hbp::sorted_batching / random_batching (src/packing.cpp:265-317): samples
 * in (length desc, id asc) order, or shuffled by
 * Rng(derive_seed(seed, "random-batching")), cut greedily into batches while
 * count * max_length <= token_budget. Outputs: order[n] (input indices in
 * batching order), batch_offsets[n + 1] (first order position of each batch,
 * then n), batch_max[n] (each batch's longest sample), *n_batches. Host
 * memory. Throws "token budget B is below the longest sample (L)". */
int hbp_padded_batching(hbp_ctx* ctx, const hbp_samples* samples, int64_t token_budget, int32_t mode,
                        uint64_t seed, int32_t* order, int64_t* batch_offsets, int64_t* batch_max,
                        int64_t* n_batches);

/* hbp::build_batching_plan (src/balance.cpp:260-298): the padded batches of
 * `mode` with token budget group.length, device_count per iteration, each
 * sample its own pack padded to its batch's longest; the plan's groups are
 * HierarchicalGroups::single(group). */
int hbp_build_batching_plan(hbp_ctx* ctx, const hbp_samples* samples, hbp_group_config group,
                            int32_t device_count, int32_t mode, uint64_t seed, hbp_plan** out);

/* hbp::curriculum_order (src/schedule.cpp:10-63) of a device plan: a new
 * plan whose first warmup_iterations iterations (phase warmup) are drawn,
 * seeded by derive_seed(seed, "curriculum"), from groups below
 * short_group_cutoff, the rest a seeded shuffle of what is left. Errors:
 * "warmup_iterations must be >= 0", "short_group_cutoff must select ...",
 * "curriculum needs W short-group iterations but the plan has only S". */
int hbp_curriculum_order(hbp_ctx* ctx, hbp_plan* plan, int32_t warmup_iterations, int32_t short_group_cutoff,
                         hbp_plan** out);

/* hbp::assign_runtime (src/schedule.cpp:65-77): per-iteration sp / ckpt of
 * its group (host arrays [n_iterations]) and the number of changes between
 * consecutive iterations. */
int hbp_assign_runtime(hbp_ctx* ctx, hbp_plan* plan, int32_t* sp, int32_t* ckpt, int64_t* switch_count);

/* hbp::write_schedule_csv (src/schedule.cpp:79-89): "iteration,group,sp,
 * ckpt,phase" rows; same buffer convention as hbp_plan_to_json. */
int hbp_schedule_csv(hbp_ctx* ctx, hbp_plan* plan, char* out, int64_t capacity, int64_t* out_len);

/* plan_from_json (include/hbp/io.hpp:26, src/io.cpp:112-160) on the GPU:
 * the manifest text (host memory) -> a device plan whose member_index
 * indexes the manifest's own samples in member order (hbp_plan_members).
 * Reads the canonical layout plan_to_json / write_plan produce, verified
 * byte for byte by re-serialising; text that is not JSON fails with the
 * reference's "bad plan manifest: <nlohmann message>", valid JSON in another
 * layout with a validation error saying so. Semantic errors are the
 * reference's ("plan manifest: unsupported version V", the groups' own,
 * "... iteration group index out of range", "... pack exceeds its
 * capacity"), first in its order. */
int hbp_plan_from_json(hbp_ctx* ctx, const char* text, int64_t bytes, hbp_plan** out, int64_t* out_n_members);
/* A device plan from a host view (all arrays host memory, member_index
 * required, iter_phase may be NULL): for plans built on the host side of a
 * caller (e.g. the C++ façade's hbp::Plan) that then use hbp_plan_to_json,
 * hbp_report_plan, hbp_simulate_plan, ... */
int hbp_plan_upload(hbp_ctx* ctx, const hbp_plan_view* view, hbp_plan** out);
/* ids[n_members], lengths[n_members] (host) of a plan read by
 * hbp_plan_from_json: sample k of the plan view is (ids[k], lengths[k]). */
int hbp_plan_members(hbp_ctx* ctx, hbp_plan* plan, int64_t* ids, int64_t* lengths);

/* Plan manifest (replaces hbp::plan_to_json, src/io.cpp:85-110): the
 * byte-identical nlohmann dump(2) text of the plan, built on the GPU.
 * `samples` is the corpus the plan was built from (ids / lengths of the
 * members; host or device memory). With out == NULL only *out_len (bytes,
 * including the final newline, no NUL) is set; otherwise out must hold
 * capacity >= *out_len bytes (HBP_ERR_VALIDATION if not). */
int hbp_plan_to_json(hbp_ctx* ctx, hbp_plan* plan, const hbp_samples* samples, char* out, int64_t capacity,
                     int64_t* out_len);
void hbp_plan_free(hbp_plan* plan);

/* report (include/hbp/metrics.hpp:78, src/metrics.cpp:107-144).
 * per_iteration_dbr / _abr may be NULL; otherwise [n_iterations]. */
int hbp_report(hbp_ctx* ctx, const hbp_plan_view* plan, hbp_metrics* out,
               double* per_iteration_dbr, double* per_iteration_abr);
/* Run-level totals for cr / ave_t over device batches (include/hbp/metrics.hpp:
 * cr, ave_t; src/metrics.cpp:71-105): iteration i holds device batches
 * [iter_dev_offsets[i], iter_dev_offsets[i + 1]) of `tokens` /
 * `comm_tokens` (host arrays). out[0] = Σ tokens, out[1] = Σ comm tokens,
 * out[2] = the most devices of any iteration. */
int hbp_run_totals(hbp_ctx* ctx, const int64_t* tokens, const int64_t* comm_tokens, const int64_t* iter_dev_offsets,
                   int64_t n_iterations, int64_t* out);
int hbp_report_plan(hbp_ctx* ctx, hbp_plan* plan, hbp_metrics* out,
                    double* per_iteration_dbr, double* per_iteration_abr);

/* simulate (include/hbp/sim.hpp:52-53, src/sim.cpp:9-60) minus the corpus
 * fingerprint, which is plan-invariant and host-side (types.cpp:52-72).
 * iteration_seconds [n_iterations] and device_* [n_devices] may be NULL. */
int hbp_simulate(hbp_ctx* ctx, const hbp_plan_view* plan,
                 const hbp_hardware_profile* profile, hbp_sim_totals* out,
                 double* iteration_seconds, double* device_compute,
                 double* device_comm, double* device_idle);
int hbp_simulate_plan(hbp_ctx* ctx, hbp_plan* plan,
                      const hbp_hardware_profile* profile, hbp_sim_totals* out,
                      double* iteration_seconds);

/* ---- cost model / auto-selection ---------------------------------------- */

/* memory_used (costmodel.hpp:50-51, src/costmodel.cpp:37-53). */
int hbp_memory_used(hbp_ctx* ctx, int64_t length, int32_t sp, int32_t ckpt,
                    const hbp_hardware_profile* profile, int64_t* out);

/* Profiler::profile_time / profile_memory / derive_ckpt of an analytic or
 * table profiler (costmodel.hpp:85-93; AnalyticProfiler costmodel.cpp:123-138,
 * TableProfiler :223-265). Constructor checks (AnalyticProfiler probe bounds,
 * TableProfiler duplicate rows) run first, as in the reference. */
int hbp_profiler_time(hbp_ctx* ctx, const hbp_profiler* profiler, int64_t length, int32_t sp, int32_t ckpt,
                      double* out);
int hbp_profiler_memory(hbp_ctx* ctx, const hbp_profiler* profiler, int64_t length, int32_t sp, int32_t ckpt,
                        int64_t* out);
int hbp_profiler_derive_ckpt(hbp_ctx* ctx, const hbp_profiler* profiler, int64_t length, int32_t sp, int32_t* out);

/* greedy_profile_ckpt (costmodel.hpp:158-159, src/costmodel.cpp:271-292). */
int hbp_greedy_profile_ckpt(hbp_ctx* ctx, const hbp_profiler* profiler,
                            int64_t length, int32_t sp, int32_t ckpt_min,
                            int32_t ckpt_max, int32_t* out);

/* find_best_sp_ckpt (costmodel.hpp:169-170, src/costmodel.cpp:294-325). */
int hbp_find_best_sp_ckpt(hbp_ctx* ctx, const hbp_profiler* profiler,
                          int64_t length, const int32_t* sp_candidates,
                          int32_t n_sp, int32_t* out_sp, int32_t* out_ckpt,
                          double* out_seconds);

/* select_groups (autoselect.hpp:36-38, src/autoselect.cpp:76-168).
 * out_groups must hold at least 4 entries. */
int hbp_select_groups(hbp_ctx* ctx, const int64_t* candidate_lengths,
                      int32_t n_lengths, const hbp_profiler* profiler,
                      const int32_t* sp_candidates, int32_t n_sp,
                      hbp_group_config* out_groups, int32_t* out_count,
                      int64_t* out_l_best, int64_t* out_l_max);

/* Candidate sweep (built from the reference's own
 * build_plan + simulate): for candidate c, groups
 * cand_groups[cand_offsets[c] .. cand_offsets[c+1]) with l_best
 * cand_l_best[c]; out_seconds[c] = simulate(build_plan(samples, groups_c,
 * options), profile).total_seconds, +inf when the candidate raises
 * InfeasibleError. *out_best = argmin (lowest index on ties, -1 if none is
 * feasible). Candidates sharing a length set share one packing. */
int hbp_sweep(hbp_ctx* ctx, const hbp_samples* samples,
              const hbp_group_config* cand_groups, const int64_t* cand_offsets,
              const int64_t* cand_l_best, int64_t n_candidates,
              const hbp_plan_options* options,
              const hbp_hardware_profile* profile, double* out_seconds,
              int64_t* out_best);

/* ---- Multi-GPU -------------------------------------------
 * One process per GPU. The reference has no counterpart (single process; its
 * "devices" are vector entries, balance.hpp:18-22); these entry points run the
 * two parts of the path that shard with their one exchange each as NCCL
 * collectives on the context's stream. NCCL is loaded at run time
 * (libnccl.so.2 already in the process, else the system's).
 *
 * Rank 0 calls hbp_comm_unique_id and sends the HBP_COMM_ID_BYTES bytes to
 * every rank out of band (e.g. torch.distributed); every rank then calls
 * hbp_comm_create with the same id, its rank and the world size
 * (collective: blocks until all ranks joined). */
#define HBP_COMM_ID_BYTES 128
typedef struct hbp_comm hbp_comm;
int hbp_comm_unique_id(hbp_ctx* ctx, unsigned char* out_id);
int hbp_comm_create(hbp_ctx* ctx, const unsigned char* id, int32_t rank, int32_t world, hbp_comm** out);
void hbp_comm_destroy(hbp_comm* comm);

/* hbp_sweep across the communicator's ranks (BASELINE C3 / C5): whole length
 * sets are dealt round-robin in decreasing estimated cost, every rank runs the
 * single-GPU sweep on its share, then ncclAllReduce(MIN) of the per-candidate
 * seconds and ncclAllGather of every rank's first error and (best seconds,
 * best index). Every rank returns the full out_seconds[n_candidates], the
 * global argmin (lowest index on ties) and the error the sequential sweep
 * raises (the first in index order). *out_local: candidates this rank
 * evaluated (may be NULL). Collective. */
int hbp_sweep_sharded(hbp_ctx* ctx, hbp_comm* comm, const hbp_samples* samples,
                      const hbp_group_config* cand_groups, const int64_t* cand_offsets,
                      const int64_t* cand_l_best, int64_t n_candidates,
                      const hbp_plan_options* options, const hbp_hardware_profile* profile,
                      double* out_seconds, int64_t* out_best, int64_t* out_local);

/* report (+ simulate when profile != NULL) of a plan every rank holds, each
 * rank evaluating its DP columns [r N / W, (r + 1) N / W): hbp_eval_columns
 * phase 0, ncclAllReduce MAX / SUM / MIN, phase 1, ncclAllReduce SUM, finish.
 * Bit-identical on every rank to hbp_report_plan / hbp_simulate_plan
 * (metrics.cpp:107-144, sim.cpp:9-60). Collective. */
int hbp_eval_sharded(hbp_ctx* ctx, hbp_comm* comm, hbp_plan* plan, const hbp_hardware_profile* profile,
                     hbp_metrics* out, hbp_sim_totals* sim);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* HBP_B200_H */
