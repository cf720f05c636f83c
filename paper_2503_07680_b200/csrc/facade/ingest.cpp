// ingest.cpp — façade for corpus files (parsed on the GPU by
// hbp_load_lengths) and synthetic corpora (hbp_synth_lengths).
#include <cstdio>
#include <fstream>
#include <iterator>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "engine_ctx.hpp"
#include "hbp/ingest.hpp"
#include "hbp_b200.h"

namespace hbp {

CorpusFormat parse_corpus_format(const std::string& name) {  // ingest.cpp:140-145
    if (name == "jsonl") return CorpusFormat::Jsonl;
    if (name == "csv") return CorpusFormat::Csv;
    if (name == "raw-lengths" || name == "raw") return CorpusFormat::RawLengths;
    throw ValidationError("unknown corpus format: " + name);
}

SampleSet load_lengths(std::istream& in, CorpusFormat format, const std::string& source_name) {
    const std::string text{std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};
    const int32_t f = format == CorpusFormat::Jsonl ? HBP_CORPUS_JSONL
                      : format == CorpusFormat::Csv ? HBP_CORPUS_CSV : HBP_CORPUS_RAW;
    const int64_t cap = static_cast<int64_t>(text.size() / 2 + 1);
    // up to (bytes + 1) / 2 records; left uninitialised, the engine writes the first n
    std::unique_ptr<int64_t[]> ids(new int64_t[static_cast<size_t>(cap)]);
    std::unique_ptr<int64_t[]> lengths(new int64_t[static_cast<size_t>(cap)]);
    int64_t n = 0;
    detail::check(hbp_load_lengths(detail::ctx(), text.data(), static_cast<int64_t>(text.size()), f,
                                   source_name.c_str(), ids.get(), lengths.get(), cap, HBP_MEM_HOST, &n));
    SampleSet set;
    set.source = source_name;
    set.samples.resize(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) set.samples[static_cast<size_t>(i)] = Sample{ids[i], lengths[i]};
    return set;
}

SampleSet load_lengths(const std::filesystem::path& path, CorpusFormat format) {  // ingest.cpp:162-168
    std::ifstream in(path);
    if (!in) throw IoError("cannot open corpus file: " + path.string());
    return load_lengths(in, format, path.string());
}

void write_jsonl(const SampleSet& set, std::ostream& out) {  // ingest.cpp:170-174
    for (const auto& s : set.samples) out << "{\"id\":" << s.id << ",\"length\":" << s.length << "}\n";
}

void write_jsonl(const SampleSet& set, const std::filesystem::path& path) {
    std::ofstream out(path);
    if (!out) throw IoError("cannot write corpus file: " + path.string());
    write_jsonl(set, out);
}

void LengthDistribution::validate() const {
    switch (family) {
        case Family::Constant:
            if (a < 1.0) throw ValidationError("constant length must be >= 1");
            break;
        case Family::Uniform:
            if (a < 1.0 || b < a) throw ValidationError("uniform bounds must satisfy 1 <= low <= high");
            break;
        case Family::Normal:
            if (b < 0.0) throw ValidationError("normal stddev must be >= 0");
            break;
        case Family::LogNormal:
            if (b < 0.0) throw ValidationError("lognormal sigma must be >= 0");
            break;
    }
}

LengthDistribution parse_distribution(const std::string& text) {
    std::vector<std::string> parts;
    std::string part;
    std::stringstream ss(text);
    while (std::getline(ss, part, ':')) parts.push_back(part);
    if (parts.empty()) throw ValidationError("empty distribution spec");
    auto num = [&](std::size_t i) {
        try {
            return std::stod(parts.at(i));
        } catch (const std::exception&) {
            throw ValidationError("bad distribution parameter in '" + text + "'");
        }
    };
    LengthDistribution d;
    std::size_t want = 3;
    if (parts[0] == "constant") {
        d.family = LengthDistribution::Family::Constant;
        want = 2;
    } else if (parts[0] == "uniform") {
        d.family = LengthDistribution::Family::Uniform;
    } else if (parts[0] == "normal") {
        d.family = LengthDistribution::Family::Normal;
    } else if (parts[0] == "lognormal") {
        d.family = LengthDistribution::Family::LogNormal;
    } else {
        throw ValidationError("unknown distribution family: " + parts[0]);
    }
    if (parts.size() != want) {
        static const char* msg[] = {"constant needs 1 parameter", "uniform needs 2 parameters",
                                    "normal needs 2 parameters", "lognormal needs 2 parameters"};
        throw ValidationError(msg[static_cast<int>(d.family)]);
    }
    d.a = num(1);
    if (want == 3) d.b = num(2);
    d.validate();
    return d;
}

std::string format_distribution(const LengthDistribution& d) {
    std::ostringstream os;
    static const char* fam[] = {"constant", "uniform", "normal", "lognormal"};
    os << fam[static_cast<int>(d.family)] << ":" << d.a;
    if (d.family != LengthDistribution::Family::Constant) os << ":" << d.b;
    return os.str();
}

void SynthSpec::validate() const {
    if (count < 1) throw ValidationError("synth count must be >= 1");
    if (long_fraction < 0.0 || long_fraction > 1.0) throw ValidationError("long_fraction must lie in [0, 1]");
    if (max_length < 1) throw ValidationError("max_length must be >= 1");
    short_dist.validate();
    long_dist.validate();
}

namespace {
// lossless text form of a distribution for the C-ABI
std::string exact(const LengthDistribution& d) {
    static const char* fam[] = {"constant", "uniform", "normal", "lognormal"};
    char buf[128];
    if (d.family == LengthDistribution::Family::Constant)
        std::snprintf(buf, sizeof buf, "%s:%.17g", fam[0], d.a);
    else
        std::snprintf(buf, sizeof buf, "%s:%.17g:%.17g", fam[static_cast<int>(d.family)], d.a, d.b);
    return buf;
}
}  // namespace

SampleSet synth_lengths(const SynthSpec& spec) {
    spec.validate();
    std::vector<int64_t> lengths(static_cast<size_t>(spec.count));
    char err[256] = {0};
    const std::string s = exact(spec.short_dist), l = exact(spec.long_dist);
    if (hbp_synth_lengths(spec.count, s.c_str(), spec.long_fraction, l.c_str(), spec.max_length, spec.seed,
                          lengths.data(), err, sizeof err) != HBP_OK)
        throw ValidationError(err);
    SampleSet set;
    set.source = "synth(seed=" + std::to_string(spec.seed) + ")";
    set.samples.resize(lengths.size());
    for (size_t i = 0; i < lengths.size(); ++i) set.samples[i] = Sample{static_cast<SampleId>(i), lengths[i]};
    return set;
}

SynthSpec parse_synth_spec(const std::string& text, std::uint64_t seed) {
    SynthSpec spec;
    spec.seed = seed;
    std::string item;
    std::stringstream ss(text);
    bool count = false, shrt = false, mx = false;
    while (std::getline(ss, item, ',')) {
        const auto eq = item.find('=');
        if (eq == std::string::npos) throw ValidationError("bad synth spec item (want key=value): " + item);
        const std::string key = item.substr(0, eq), value = item.substr(eq + 1);
        try {
            if (key == "count") {
                spec.count = std::stoll(value);
                count = true;
            } else if (key == "long_fraction" || key == "long_frac") {
                spec.long_fraction = std::stod(value);
            } else if (key == "short") {
                spec.short_dist = parse_distribution(value);
                shrt = true;
            } else if (key == "long") {
                spec.long_dist = parse_distribution(value);
            } else if (key == "max" || key == "max_length") {
                spec.max_length = std::stoll(value);
                mx = true;
            } else {
                throw ValidationError("unknown synth spec key: " + key);
            }
        } catch (const ValidationError&) {
            throw;
        } catch (const std::exception&) {
            throw ValidationError("bad synth spec value for " + key + ": " + value);
        }
    }
    if (!count || !shrt || !mx) throw ValidationError("synth spec needs at least count=, short= and max=");
    spec.validate();
    return spec;
}

}  // namespace hbp
