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

}  // namespace hbp_b200
