// plan_handle.hpp — a host hbp::Plan on the device and back (façade-internal).
#pragma once

#include <vector>

#include "hbp/balance.hpp"
#include "hbp_b200.h"

namespace hbp::detail {

// The plan as a device plan (hbp_plan_upload); member k of the device plan
// is sample (ids[k], lens[k]), in the plan's own member order.
struct UploadedPlan {
    hbp_plan* h = nullptr;
    std::vector<int64_t> ids, lens;
    UploadedPlan() = default;
    UploadedPlan(const UploadedPlan&) = delete;
    UploadedPlan& operator=(const UploadedPlan&) = delete;
    UploadedPlan(UploadedPlan&& o) noexcept : h(o.h), ids(std::move(o.ids)), lens(std::move(o.lens)) { o.h = nullptr; }
    ~UploadedPlan() { hbp_plan_free(h); }
};

UploadedPlan upload_plan(const Plan& plan);

// The owning Plan of a device plan whose member_index indexes ids / lens.
Plan plan_of_handle(hbp_plan* h, const std::vector<int64_t>& ids, const std::vector<int64_t>& lens);

}  // namespace hbp::detail
