// hbp/io.hpp — the plan manifest (drop-in for the plan part of reference
// include/hbp/io.hpp:22-28). Text is written and read on the GPU
// (hbp_plan_to_json / hbp_plan_from_json); the groups / metrics / sim-report
// manifests are not part of the B200 engine.
#ifndef HBP_IO_HPP
#define HBP_IO_HPP

#include <filesystem>
#include <string>

#include "hbp/balance.hpp"

namespace hbp {

// Versioned JSON of the plan (nlohmann dump(2) layout, byte-identical to the
// reference); save / load / save round-trips bit-exactly. The reader takes
// the layout plan_to_json writes.
std::string plan_to_json(const Plan& plan);
Plan plan_from_json(const std::string& text);
void write_plan(const Plan& plan, const std::filesystem::path& path);
Plan read_plan(const std::filesystem::path& path);

}  // namespace hbp

#endif  // HBP_IO_HPP
