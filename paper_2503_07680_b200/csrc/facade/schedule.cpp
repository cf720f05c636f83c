// schedule.cpp — façade for include/hbp/schedule.hpp: the host plan goes to
// the device (hbp_plan_upload), the engine reorders / assigns / formats it
// (src/schedule.cpp:10-89 semantics, csrc/schedule.cu).
#include <ostream>
#include <string>

#include "engine_ctx.hpp"
#include "hbp/schedule.hpp"
#include "plan_handle.hpp"

namespace hbp {

Plan curriculum_order(const Plan& plan, const CurriculumSpec& spec) {
    const detail::UploadedPlan u = detail::upload_plan(plan);
    hbp_plan* out = nullptr;
    detail::check(hbp_curriculum_order(detail::ctx(), u.h, spec.warmup_iterations, spec.short_group_cutoff, &out));
    struct Free {
        hbp_plan* p;
        ~Free() { hbp_plan_free(p); }
    } f{out};
    return detail::plan_of_handle(out, u.ids, u.lens);
}

RuntimeAssignment assign_runtime(const Plan& plan) {
    const detail::UploadedPlan u = detail::upload_plan(plan);
    const size_t n = plan.iterations.size();
    std::vector<int32_t> sp(n + 1), ck(n + 1);
    int64_t switches = 0;
    detail::check(hbp_assign_runtime(detail::ctx(), u.h, sp.data(), ck.data(), &switches));
    RuntimeAssignment r;
    for (size_t i = 0; i < n; ++i) r.per_iteration.push_back(RuntimeConfig{sp[i], ck[i]});
    r.switch_count = static_cast<int>(switches);
    return r;
}

void write_schedule_csv(const Plan& plan, std::ostream& out) {
    const detail::UploadedPlan u = detail::upload_plan(plan);
    int64_t n = 0;
    detail::check(hbp_schedule_csv(detail::ctx(), u.h, nullptr, 0, &n));
    std::string text(static_cast<size_t>(n), '\0');
    detail::check(hbp_schedule_csv(detail::ctx(), u.h, text.data(), n, &n));
    out << text;
}

}  // namespace hbp
