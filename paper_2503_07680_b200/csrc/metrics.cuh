// metrics.cuh — report / simulate over a flat device plan (metrics.cu).
#pragma once

#include <vector>

#include "engine.cuh"

namespace hbp_b200 {

struct PlanArrays {
    const int32_t* iter_group;
    const int64_t* iter_dev_offsets;
    const int64_t* dev_pack_offsets;
    const int64_t* pack_capacity;
    const int64_t* pack_total;
    const int64_t* pack_attention;
    i64 I;  // iterations
    i64 D;  // devices
};

struct EvalOut {
    hbp_metrics m{};
    double total_seconds = 0.0;
    int32_t switch_count = 0;
};

// profile == nullptr: report() only. Output arrays are device pointers or null.
void eval_plan(Ctx& c, const PlanArrays& p, int32_t device_count, const std::vector<hbp_group_config>& groups,
               const hbp_hardware_profile* profile, EvalOut& out, double* d_dbr, double* d_abr, double* d_secs,
               double* d_dcomp, double* d_dcomm, double* d_didle);

// Sharded by DP column; phase 0 / 1 on device columns
// [c0, c1) of every iteration, finish on the all-reduced buffers.
void eval_columns(Ctx& c, const PlanArrays& p, const std::vector<hbp_group_config>& groups,
                  const hbp_hardware_profile* profile, int phase, int32_t c0, int32_t c1,
                  const hbp_eval_columns_bufs& b);
void eval_columns_finish(Ctx& c, const PlanArrays& p, int32_t device_count,
                         const std::vector<hbp_group_config>& groups, const hbp_hardware_profile* profile,
                         const hbp_eval_columns_bufs& b, EvalOut& out);

}  // namespace hbp_b200
