// hbp/packing.hpp — packing strategies behind one interface (drop-in for
// reference include/hbp/packing.hpp). pack() runs on the GPU (hbp_pack):
// ISF, random, FFD and FFS through the engine's kernels; BFS and SPFHP are
// not in the engine yet and raise ValidationError naming the strategy.
#ifndef HBP_PACKING_HPP
#define HBP_PACKING_HPP

#include <cstdint>
#include <string>
#include <vector>

#include "hbp/metrics.hpp"
#include "hbp/types.hpp"

namespace hbp {

enum class StrategyKind { Random, Isf, Ffs, Ffd, Bfs, Spfhp };

StrategyKind parse_strategy(const std::string& name);
std::string strategy_name(StrategyKind kind);

struct PackingStrategy {
    StrategyKind kind = StrategyKind::Isf;
    int isf_iterations = 8;            // ISF rounds
    double isf_fill_threshold = 0.98;  // freeze packs filled to this ratio
    void validate() const;
};

struct PackList {
    std::vector<Pack> packs;
    Tokens capacity = 0;
    std::vector<Sample> leftover;
    Tokens total_tokens() const;
};

PackList pack(const SampleSet& samples, Tokens capacity, const PackingStrategy& strategy, std::uint64_t seed);

struct PaddedBatch {
    std::vector<Sample> samples;
    Tokens max_length = 0;
    Tokens padded_tokens = 0;
};

std::vector<PaddedBatch> sorted_batching(const SampleSet& samples, Tokens token_budget);
std::vector<PaddedBatch> random_batching(const SampleSet& samples, Tokens token_budget, std::uint64_t seed);

}  // namespace hbp

#endif  // HBP_PACKING_HPP
