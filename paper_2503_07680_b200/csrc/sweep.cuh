// sweep.cuh — the candidate sweep's internal entry points (sweep.cu), shared
// with the multi-GPU sweep over NCCL (comm.cu).
#pragma once

#include <string>
#include <vector>

#include "../../include/hbp_b200.h"
#include "pipeline.cuh"

namespace hbp_b200 {

struct SweepErr {
    int code = HBP_OK;
    std::string msg;
};

// ingest + SampleSet::validate of the sweep's corpus (every rank the same)
void sweep_ingest(hbp_ctx& c, const hbp_samples* samples, DeviceCorpus& corpus);

// Evaluates the candidates `idx` (ascending global indices): secs[k] /
// errs[k] for each k evaluated, exactly as the sequential sweep would (a
// block of one length set stops at its first error).
void sweep_evaluate(hbp_ctx& c, const DeviceCorpus& corpus, const hbp_group_config* cand_groups,
                    const int64_t* cand_offsets, const int64_t* cand_l_best, const std::vector<int64_t>& idx,
                    const hbp_plan_options* options, const hbp_hardware_profile* profile, std::vector<double>& secs,
                    std::vector<SweepErr>& errs);

// The candidates rank `rank` of `world` evaluates: whole length sets dealt
// round-robin in decreasing estimated cost (paper_2503_07680_b200/sweep.py
// shard() is the same rule).
std::vector<int64_t> sweep_shard(const hbp_group_config* cand_groups, const int64_t* cand_offsets,
                                 int64_t n_candidates, int rank, int world);

}  // namespace hbp_b200
