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
