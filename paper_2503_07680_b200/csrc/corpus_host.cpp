// corpus_host.cpp — the text of nlohmann's parse_error for one JSONL line
// (ingest.cpp:67-72 reports e.what()). Called only after the GPU parser
// (corpus.cu) found that line invalid; the reference's message is the
// library's own, so the same library formats it.
#include <string>

#include <nlohmann/json.hpp>

namespace hbp_b200 {

std::string json_parse_error_text(const std::string& line) {
    try {
        const auto doc = nlohmann::json::parse(line);
        (void)doc;
    } catch (const nlohmann::json::parse_error& e) {
        return e.what();
    }
    return std::string();
}

}  // namespace hbp_b200

// ---- plan manifest: the small header, and error texts ----------------------
//
// plan_from_json (src/io.cpp:112-160) reads the manifest through nlohmann's
// DOM. The GPU reader (plan_json.cu) tokenises and validates the whole text
// and reads the iterations on the device; the host sees only the header
// (device_count, groups, seed, version: a few hundred bytes, the iterations
// value replaced by []) and, when the device flags an error, the text once
// more to report the error the reference raises first in its own order.
#include "manifest_host.hpp"

namespace hbp_b200 {

namespace {

using nlohmann::json;

// the checks of io.cpp:44-55 and :29-42 (groups validate: autoselect.cpp:18-33),
// device_count, seed; then, with `iterations`, the per-iteration reads of
// io.cpp:126-157 (values discarded): the first failure as the reference
// reports it
ManifestError walk(const json& obj, ManifestHeader* h, bool iterations) {
    ManifestError none{0, std::string()};
    try {
        if (!obj.is_object() || !obj.contains("version"))
            return {2, "plan manifest: missing version field"};
        const int v = obj["version"].get<int>();
        if (v != 1) return {2, "plan manifest: unsupported version " + std::to_string(v)};
        const json& gobj = obj.at("groups");
        std::vector<hbp_group_config> groups;
        for (const auto& g : gobj.at("groups")) {
            hbp_group_config gc{};
            gc.length = g.at("length").get<int64_t>();
            gc.sp = g.at("sp").get<int>();
            gc.ckpt = g.at("ckpt").get<int>();
            groups.push_back(gc);
        }
        const int64_t l_best = gobj.at("l_best").get<int64_t>();
        const int64_t l_max = gobj.at("l_max").get<int64_t>();
        if (groups.empty()) return {2, "no packing groups"};
        int64_t prev = 0;
        for (const auto& g : groups) {
            if (g.length <= prev) return {2, "group lengths must be strictly increasing"};
            if (g.sp < 1 || g.ckpt < 0) return {2, "invalid group runtime config"};
            prev = g.length;
        }
        if (groups.back().length != l_max) return {2, "last group must carry l_max"};
        const int device_count = obj.at("device_count").get<int>();
        const uint64_t seed = obj.at("seed").get<uint64_t>();
        if (h) {
            h->groups = groups;
            h->l_best = l_best;
            h->l_max = l_max;
            h->device_count = device_count;
            h->seed = seed;
        }
        if (!iterations) return none;
        for (const auto& it : obj.at("iterations")) {
            const int gi = it.at("group").get<int>();
            if (gi < 0 || gi >= static_cast<int>(groups.size()))
                return {2, "plan manifest: iteration group index out of range"};
            (void)it.at("phase").get<std::string>();
            for (const auto& dev : it.at("devices")) {
                for (const auto& pack : dev) {
                    const int64_t cap = pack.at("capacity").get<int64_t>();
                    int64_t total = 0;
                    for (const auto& s : pack.at("samples")) {
                        (void)s.at(0).get<int64_t>();
                        total += s.at(1).get<int64_t>();
                    }
                    if (total > cap) return {2, "plan manifest: pack exceeds its capacity"};
                }
            }
        }
    } catch (const json::exception& e) {
        return {6, e.what()};
    }
    return none;
}

}  // namespace

ManifestError manifest_header(const std::string& doc, ManifestHeader& h) {
    json obj;
    try {
        obj = json::parse(doc);
    } catch (const json::parse_error& e) {
        return {2, std::string("bad plan manifest: ") + e.what()};
    }
    return walk(obj, &h, false);
}

ManifestError manifest_error(const std::string& text) {
    json obj;
    try {
        obj = json::parse(text);
    } catch (const json::parse_error& e) {
        return {2, std::string("bad plan manifest: ") + e.what()};
    }
    return walk(obj, nullptr, true);
}

}  // namespace hbp_b200
