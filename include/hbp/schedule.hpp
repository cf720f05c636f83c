// hbp/schedule.hpp — curriculum ordering, runtime assignment and the
// schedule CSV (drop-in for the plan part of reference
// include/hbp/schedule.hpp:13-37), run on the GPU engine
// (hbp_curriculum_order, hbp_assign_runtime, hbp_schedule_csv). The loss
// normalizers of that header are not part of the B200 engine.
#ifndef HBP_SCHEDULE_HPP
#define HBP_SCHEDULE_HPP

#include <iosfwd>
#include <vector>

#include "hbp/balance.hpp"
#include "hbp/costmodel.hpp"

namespace hbp {

struct CurriculumSpec {
    int warmup_iterations = 500;
    // Group indices below the cutoff count as "short".
    int short_group_cutoff = 1;
};

// The first warmup_iterations steps drawn (seeded) from short groups only,
// the rest a seeded shuffle of what is left; a permutation of the input
// iterations. ValidationError with both counts when too few are short.
Plan curriculum_order(const Plan& plan, const CurriculumSpec& spec);

struct RuntimeAssignment {
    std::vector<RuntimeConfig> per_iteration;
    int switch_count = 0;  // consecutive-iteration config changes
};

RuntimeAssignment assign_runtime(const Plan& plan);

// iteration,group,sp,ckpt,phase
void write_schedule_csv(const Plan& plan, std::ostream& out);

}  // namespace hbp

#endif  // HBP_SCHEDULE_HPP
