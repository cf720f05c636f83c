// manifest_host.hpp — host side of the general plan manifest reader
// (plan_json.cu, corpus_host.cpp): plain types, no CUDA.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/hbp_b200.h"

namespace hbp_b200 {

struct ManifestHeader {
    int32_t device_count = 0;
    uint64_t seed = 0;
    std::vector<hbp_group_config> groups;
    int64_t l_best = 0, l_max = 0;
};

// code 0: none; HBP_ERR_VALIDATION: the reference's ValidationError text;
// HBP_ERR_JSON: an nlohmann type / key error (json::exception::what())
struct ManifestError {
    int code;
    std::string msg;
};

// the header of a manifest whose iterations value is [] (io.cpp:121-124)
ManifestError manifest_header(const std::string& doc, ManifestHeader& h);
// the first error plan_from_json raises on `text`, or {0, ""}
ManifestError manifest_error(const std::string& text);

}  // namespace hbp_b200
