// autoselect.cuh — device profilers, Alg. 1/3/4 problem records (autoselect.cu)
// and the host side that formats the reference's exception text from the
// recorded failure events (autoselect_host.cu).
#pragma once

#include <string>
#include <vector>

#include "engine.cuh"

namespace hbp_b200 {

// failure codes (each maps to one reference message)
enum AsCode : int {
    AS_OK = 0,
    AS_V_SP = 1,          // "sp must be >= 1"                              costmodel.cpp:39
    AS_V_CKPT = 2,        // "ckpt must lie in [0, layer_count]"            costmodel.cpp:41
    AS_V_GREEDY = 3,      // "greedy_profile_ckpt: ckpt_min must be < ckpt_max"  :274
    AS_I_SLOPE = 4,       // "GC does not reduce memory under this profile (slope %f bytes/layer)" :282
    AS_I_NOROW = 5,       // "no profile row for length L, sp S"            :225
    AS_I_OOMROW = 6,      // "profiled configuration is out of memory at length L, sp S"  :229
    AS_I_NOROW_CKPT = 7,  // "no profile row for length L, sp S, ckpt C"    :234
    AS_I_NOFIT = 8,       // "sp=S does not fit device memory even at ckpt C"  :305
    AS_I_MEM = 9,         // iter_time memory check                         :74-81
};
enum AsStatus : int { AS_S_NONE = 10, AS_S_LARGEST = 11, AS_S_STAGE2 = 12, AS_S_MID = 13 };

struct AsErr {
    int code;
    int64_t length;
    int32_t sp;
    int32_t ckpt;
    int64_t used;
    double slope;
};

// Device profiler (analytic or table) -- rows live in device memory.
struct DevProfiler {
    int32_t kind;
    hbp_hardware_profile profile;
    int32_t ckpt_min, ckpt_max;  // analytic probe bounds (resolved)
    const hbp_profile_row* rows;
    int64_t n_rows;
    int64_t device_memory;
};

// One select_groups call; all pointers are device memory.
struct AsProblem {
    const DevProfiler* profiler;
    const int64_t* lengths;
    int32_t n_lengths;
    const int32_t* sps;
    int32_t n_sp;
    // per length
    uint8_t* length_ok;
    int32_t* best_sp;
    int32_t* best_ckpt;
    double* best_sec;
    AsErr* fails;  // [n_lengths * n_sp]
    // result
    int32_t status;
    AsErr stage2;
    hbp_group_config out[4];
    int32_t n_out;
    int64_t l_best, l_max;
};

enum AsOp : int { AS_Q_GREEDY = 1, AS_Q_DERIVE = 2, AS_Q_MEMORY = 3, AS_Q_TIME = 4, AS_Q_BEST = 5 };

struct AsQuery {
    int32_t op;
    int64_t length;
    int32_t sp, ckpt, ckpt_min, ckpt_max;
    const int32_t* sps;  // AS_Q_BEST
    int32_t n_sp;
    AsErr* fails;        // AS_Q_BEST: [n_sp]
    // outputs
    AsErr err;
    int32_t ok;
    int32_t out_ckpt, out_sp;
    int64_t out_mem;
    double out_sec;
};

void run_select_problems(Ctx& c, AsProblem* d_probs, int n);
void run_queries(Ctx& c, const DevProfiler* d_prof, AsQuery* d_q, int n);

// host side (autoselect_host.cu)
std::string as_message(const AsErr& e);
bool as_is_validation(int code);

// Resolves and validates a C-ABI profiler (AnalyticProfiler constructor /
// TableProfiler constructor checks) and uploads it; keeps device storage.
struct DeviceProfilerHolder {
    DevBuf<hbp_profile_row> rows;
    DevBuf<DevProfiler> dev;
    DevProfiler host{};
};
void upload_profiler(Ctx& c, const hbp_profiler* in, DeviceProfilerHolder& out);

struct SelectResult {
    std::vector<hbp_group_config> groups;
    int64_t l_best = 0, l_max = 0;
};
// select_groups for one or many problems sharing a profiler; throws the
// reference's error for problem 0 when it fails (batch: per-problem status).
SelectResult select_groups_device(Ctx& c, const hbp_profiler* prof, const std::vector<int64_t>& lengths,
                                  const std::vector<int32_t>& sps);

}  // namespace hbp_b200
