// costmodel.cpp — façade for the cost model, profilers and auto-selection.
//
// AnalyticProfiler / TableProfiler queries, Alg. 3/4 and Alg. 1 run on the
// GPU through the C-ABI. A Profiler subclass written by a user (the
// reference's sanctioned extension point, e.g. a "GC off" profiler) cannot
// be called from device code, so for those the search runs here against
// the virtual interface, following the reference algorithm step by step
// (costmodel.cpp:271-325, autoselect.cpp:35-168).
#include <algorithm>
#include <cctype>
#include <cmath>
#include <fstream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "../costmodel.cuh"
#include "engine_ctx.hpp"
#include "hbp/autoselect.hpp"
#include "hbp/costmodel.hpp"
#include "hbp_b200.h"

namespace hbp {

using detail::check;
using detail::ctx;

hbp_hardware_profile to_flat(const HardwareProfile& p) {
    return hbp_hardware_profile{p.per_token_linear_cost, p.per_token2_attention_cost, p.sp_comm_cost,
                                p.gc_recompute_factor, p.fixed_iteration_cost, p.layer_count, p.base_memory,
                                p.per_token_activation_memory, p.gc_memory_saving_per_layer, p.reference_length,
                                p.device_memory};
}

void HardwareProfile::validate() const {
    const int code = hbp_b200::cm_profile_check(to_flat(*this));
    if (code) throw ValidationError(hbp_b200::cm_profile_message(code));
}

std::int64_t memory_used(Tokens l, RuntimeConfig config, const HardwareProfile& profile) {
    const hbp_hardware_profile p = to_flat(profile);
    int64_t out = 0;
    check(hbp_memory_used(ctx(), l, config.sp, config.ckpt, &p, &out));
    return out;
}

DeviceWork device_work(std::span<const Pack> packs) {
    DeviceWork w;
    for (const auto& p : packs) {
        w.padded_tokens += p.capacity;
        w.real_tokens += p.total;
        const Tokens pad = p.capacity - p.total;
        w.attention += p.attention + pad * pad;  // the padded tail counts as one segment
        w.max_capacity = std::max(w.max_capacity, p.capacity);
    }
    return w;
}

// One device's busy time: the same expression code the GPU simulate uses
// (costmodel.cuh), compiled without FMA contraction.
double iter_time(const DeviceWork& work, RuntimeConfig config, const HardwareProfile& profile) {
    profile.validate();
    if (work.padded_tokens == 0) return 0.0;
    if (config.sp < 1) throw ValidationError("sp must be >= 1");
    if (config.ckpt < 0 || config.ckpt > profile.layer_count) throw ValidationError("ckpt must lie in [0, layer_count]");
    const hbp_hardware_profile p = to_flat(profile);
    const int64_t used = hbp_b200::cm_memory_used(work.max_capacity, config.sp, config.ckpt, p);
    if (used > profile.device_memory)
        throw InfeasibleError("configuration sp=" + std::to_string(config.sp) + " ckpt=" + std::to_string(config.ckpt) +
                              " at length " + std::to_string(work.max_capacity) + " requires " + std::to_string(used) +
                              " bytes, " + std::to_string(profile.device_memory) + " available");
    return hbp_b200::cm_iter_time(work.padded_tokens, work.attention, config.sp, config.ckpt, p);
}

double iter_time(std::span<const Pack> device_packs, RuntimeConfig config, const HardwareProfile& profile) {
    return iter_time(device_work(device_packs), config, profile);
}

// ---------------------------------------------------------------------------
// profilers
// ---------------------------------------------------------------------------

namespace {

struct FlatProfiler {
    hbp_profiler p{};
    std::vector<hbp_profile_row> rows;
};

std::optional<FlatProfiler> flat_profiler(const Profiler& prof) {
    FlatProfiler f;
    if (const auto* a = dynamic_cast<const AnalyticProfiler*>(&prof)) {
        f.p.kind = HBP_PROFILER_ANALYTIC;
        f.p.profile = to_flat(a->profile());
        f.p.ckpt_min = a->ckpt_min();
        f.p.ckpt_max = a->ckpt_max();
        f.p.device_memory = a->profile().device_memory;
        return f;
    }
    if (const auto* t = dynamic_cast<const TableProfiler*>(&prof)) {
        f.p.kind = HBP_PROFILER_TABLE;
        hbp_hardware_profile_defaults(&f.p.profile);
        for (const auto& r : t->rows())
            f.rows.push_back(hbp_profile_row{r.length, r.sp, r.ckpt, r.memory_bytes, r.seconds, r.oom ? 1 : 0});
        f.p.rows = f.rows.data();
        f.p.n_rows = static_cast<int64_t>(f.rows.size());
        f.p.device_memory = t->device_memory();
        return f;
    }
    return std::nullopt;
}

}  // namespace

AnalyticProfiler::AnalyticProfiler(HardwareProfile profile, int ckpt_min, int ckpt_max)
    : profile_(profile), ckpt_min_(ckpt_min), ckpt_max_(ckpt_max < 0 ? profile.layer_count : ckpt_max) {
    profile_.validate();
    if (ckpt_min_ < 0 || ckpt_min_ >= ckpt_max_ || ckpt_max_ > profile_.layer_count)
        throw ValidationError("ckpt probe bounds must satisfy 0 <= ckpt_min < ckpt_max <= layer_count");
}

double AnalyticProfiler::profile_time(Tokens l, RuntimeConfig config) const {
    auto f = flat_profiler(*this);
    double out = 0.0;
    check(hbp_profiler_time(ctx(), &f->p, l, config.sp, config.ckpt, &out));
    return out;
}

std::int64_t AnalyticProfiler::profile_memory(Tokens l, RuntimeConfig config) const {
    auto f = flat_profiler(*this);
    int64_t out = 0;
    check(hbp_profiler_memory(ctx(), &f->p, l, config.sp, config.ckpt, &out));
    return out;
}

int AnalyticProfiler::derive_ckpt(Tokens l, int sp) const {
    auto f = flat_profiler(*this);
    int32_t out = 0;
    check(hbp_profiler_derive_ckpt(ctx(), &f->p, l, sp, &out));
    return out;
}

TableProfiler::TableProfiler(std::vector<ProfileRow> rows, std::int64_t device_memory)
    : rows_(std::move(rows)), device_memory_(device_memory) {
    for (std::size_t i = 0; i < rows_.size(); ++i)
        if (!by_length_sp_.emplace(std::make_pair(rows_[i].length, rows_[i].sp), i).second)
            throw ValidationError("duplicate profile row for length " + std::to_string(rows_[i].length) + ", sp " +
                                  std::to_string(rows_[i].sp));
}

TableProfiler TableProfiler::from_csv(std::istream& in, const std::string& name, std::int64_t device_memory) {
    std::vector<ProfileRow> rows;
    std::string line;
    std::size_t line_no = 0;
    bool header_seen = false;
    auto trim = [](const std::string& c) {
        const auto b = c.find_first_not_of(" \t\r");
        if (b == std::string::npos) return std::string();
        return c.substr(b, c.find_last_not_of(" \t\r") - b + 1);
    };
    while (std::getline(in, line)) {
        ++line_no;
        if (line.find_first_not_of(" \t\r") == std::string::npos || line[0] == '#') continue;
        std::vector<std::string> cells;
        std::stringstream ss(line);
        std::string cell;
        while (std::getline(ss, cell, ',')) cells.push_back(trim(cell));
        if (!header_seen && !cells.empty() && cells[0] == "length") {
            header_seen = true;
            continue;
        }
        if (cells.size() < 5)
            throw ValidationError(name + " line " + std::to_string(line_no) +
                                  ": want length,sp,ckpt,memory_bytes,iter_seconds");
        ProfileRow r;
        try {
            r.length = std::stoll(cells[0]);
            r.sp = std::stoi(cells[1]);
            r.ckpt = std::stoi(cells[2]);
            if (cells[3] == "oom") {
                r.oom = true;
            } else {
                r.memory_bytes = std::stoll(cells[3]);
                r.seconds = std::stod(cells[4]);
            }
        } catch (const std::exception&) {
            throw ValidationError(name + " line " + std::to_string(line_no) + ": malformed profile row");
        }
        rows.push_back(r);
    }
    if (rows.empty()) throw ValidationError("profile table is empty: " + name);
    return TableProfiler(std::move(rows), device_memory);
}

TableProfiler TableProfiler::from_csv_file(const std::filesystem::path& path, std::int64_t device_memory) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open profile table: " + path.string());
    return from_csv(in, path.string(), device_memory);
}

const ProfileRow* TableProfiler::find(Tokens l, int sp) const {
    const auto it = by_length_sp_.find(std::make_pair(l, sp));
    return it == by_length_sp_.end() ? nullptr : &rows_[it->second];
}

double TableProfiler::profile_time(Tokens l, RuntimeConfig config) const {
    auto f = flat_profiler(*this);
    double out = 0.0;
    check(hbp_profiler_time(ctx(), &f->p, l, config.sp, config.ckpt, &out));
    return out;
}

std::int64_t TableProfiler::profile_memory(Tokens l, RuntimeConfig config) const {
    auto f = flat_profiler(*this);
    int64_t out = 0;
    check(hbp_profiler_memory(ctx(), &f->p, l, config.sp, config.ckpt, &out));
    return out;
}

int TableProfiler::derive_ckpt(Tokens l, int sp) const {
    auto f = flat_profiler(*this);
    int32_t out = 0;
    check(hbp_profiler_derive_ckpt(ctx(), &f->p, l, sp, &out));
    return out;
}

// ---------------------------------------------------------------------------
// Alg. 4 / Alg. 3
// ---------------------------------------------------------------------------

int greedy_profile_ckpt(const Profiler& profiler, Tokens l, int sp, int ckpt_min, int ckpt_max) {
    if (auto f = flat_profiler(profiler)) {
        int32_t out = 0;
        check(hbp_greedy_profile_ckpt(ctx(), &f->p, l, sp, ckpt_min, ckpt_max, &out));
        return out;
    }
    if (ckpt_min >= ckpt_max) throw ValidationError("greedy_profile_ckpt: ckpt_min must be < ckpt_max");
    const double m1r = static_cast<double>(profiler.profile_memory(l, RuntimeConfig{sp, ckpt_min}));
    const double m2r = static_cast<double>(profiler.profile_memory(l, RuntimeConfig{sp, ckpt_max}));
    const double slope = (m2r - m1r) / static_cast<double>(ckpt_max - ckpt_min);
    if (slope <= 0.0)
        throw InfeasibleError("GC does not reduce memory under this profile (slope " + std::to_string(slope) +
                              " bytes/layer)");
    const int rounded = static_cast<int>(std::ceil(static_cast<double>(ckpt_max) - m2r / slope));
    return std::clamp(rounded, 0, ckpt_max);
}

SpCkptChoice find_best_sp_ckpt(const Profiler& profiler, Tokens l, std::span<const int> sp_candidates) {
    if (sp_candidates.empty()) throw ValidationError("find_best_sp_ckpt: no sp candidates");
    if (auto f = flat_profiler(profiler)) {
        std::vector<int32_t> sps(sp_candidates.begin(), sp_candidates.end());
        int32_t sp = 0, ck = 0;
        double sec = 0.0;
        check(hbp_find_best_sp_ckpt(ctx(), &f->p, l, sps.data(), static_cast<int32_t>(sps.size()), &sp, &ck, &sec));
        return SpCkptChoice{RuntimeConfig{sp, ck}, sec};
    }
    std::optional<SpCkptChoice> best;
    std::string failures;
    for (const int sp : sp_candidates) {
        try {
            RuntimeConfig c{sp, profiler.derive_ckpt(l, sp)};
            if (profiler.profile_memory(l, c) < 0)
                throw InfeasibleError("sp=" + std::to_string(sp) + " does not fit device memory even at ckpt " +
                                      std::to_string(c.ckpt));
            const double s = profiler.profile_time(l, c);
            if (!best || s < best->seconds) best = SpCkptChoice{c, s};
        } catch (const Error& e) {
            if (!failures.empty()) failures += "; ";
            failures += "sp=" + std::to_string(sp) + ": " + e.what();
        }
    }
    if (!best) throw InfeasibleError("no feasible (sp, ckpt) for length " + std::to_string(l) + ": " + failures);
    return *best;
}

double profiling_overhead(std::size_t length_count, std::size_t sp_count, std::size_t memory_probe_count,
                          int profile_iter, double iteration_time) {
    if (length_count < 1 || sp_count < 1 || memory_probe_count < 1 || profile_iter < 1)
        throw ValidationError("profiling_overhead: all counts must be >= 1");
    const double probes = static_cast<double>(length_count) * static_cast<double>(sp_count) *
                              static_cast<double>(profile_iter) +
                          static_cast<double>(memory_probe_count) * static_cast<double>(profile_iter);
    return probes * iteration_time;
}

// Flat JSON object of numbers, e.g. data/profiles/analytic_default.json.
HardwareProfile load_analytic_profile(std::istream& in, const std::string& name) {
    std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    std::map<std::string, std::string> kv;
    size_t i = text.find('{');
    auto bad = [&](const std::string& why) { return ValidationError("bad analytic profile " + name + ": " + why); };
    if (i == std::string::npos) throw bad("expected an object");
    ++i;
    while (true) {
        while (i < text.size() && std::isspace(static_cast<unsigned char>(text[i]))) ++i;
        if (i < text.size() && text[i] == '}') break;
        if (i >= text.size() || text[i] != '"') throw bad("expected a key");
        const size_t e = text.find('"', i + 1);
        if (e == std::string::npos) throw bad("unterminated key");
        const std::string key = text.substr(i + 1, e - i - 1);
        i = text.find(':', e);
        if (i == std::string::npos) throw bad("expected ':'");
        ++i;
        size_t j = i;
        while (j < text.size() && text[j] != ',' && text[j] != '}') ++j;
        std::string val = text.substr(i, j - i);
        val.erase(0, val.find_first_not_of(" \t\r\n"));
        val.erase(val.find_last_not_of(" \t\r\n") + 1);
        kv[key] = val;
        i = j;
        if (i < text.size() && text[i] == ',') ++i;
    }
    HardwareProfile p = HardwareProfile::defaults();
    auto num = [&](const char* k, auto& out) {
        auto it = kv.find(k);
        if (it == kv.end()) return;
        try {
            out = static_cast<std::remove_reference_t<decltype(out)>>(std::stod(it->second));
        } catch (const std::exception&) {
            throw bad(std::string("field ") + k);
        }
    };
    num("per_token_linear_cost", p.per_token_linear_cost);
    num("per_token2_attention_cost", p.per_token2_attention_cost);
    num("sp_comm_cost", p.sp_comm_cost);
    num("gc_recompute_factor", p.gc_recompute_factor);
    num("fixed_iteration_cost", p.fixed_iteration_cost);
    num("layer_count", p.layer_count);
    if (kv.count("base_memory")) p.base_memory = std::stoll(kv["base_memory"]);
    num("per_token_activation_memory", p.per_token_activation_memory);
    num("gc_memory_saving_per_layer", p.gc_memory_saving_per_layer);
    if (kv.count("device_memory")) p.device_memory = std::stoll(kv["device_memory"]);
    if (kv.count("reference_length")) p.reference_length = std::stoll(kv["reference_length"]);
    p.validate();
    return p;
}

HardwareProfile load_analytic_profile_file(const std::filesystem::path& path) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open analytic profile: " + path.string());
    return load_analytic_profile(in, path.string());
}

// ---------------------------------------------------------------------------
// autoselect.hpp
// ---------------------------------------------------------------------------

HierarchicalGroups HierarchicalGroups::single(GroupConfig g) {
    HierarchicalGroups h;
    h.groups.push_back(g);
    h.l_best = g.length;
    h.l_max = g.length;
    h.validate();
    return h;
}

void HierarchicalGroups::validate() const {
    if (groups.empty()) throw ValidationError("no packing groups");
    Tokens prev = 0;
    for (const auto& g : groups) {
        if (g.length <= prev) throw ValidationError("group lengths must be strictly increasing");
        if (g.config.sp < 1 || g.config.ckpt < 0) throw ValidationError("invalid group runtime config");
        prev = g.length;
    }
    if (groups.back().length != l_max) throw ValidationError("last group must carry l_max");
}

namespace {
bool pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }
}  // namespace

HierarchicalGroups select_groups(std::span<const Tokens> candidate_lengths, const Profiler& profiler,
                                 std::span<const int> sp_candidates) {
    if (auto f = flat_profiler(profiler)) {
        std::vector<int64_t> ls(candidate_lengths.begin(), candidate_lengths.end());
        std::vector<int32_t> sps(sp_candidates.begin(), sp_candidates.end());
        hbp_group_config out[4];
        int32_t n = 0;
        int64_t lb = 0, lm = 0;
        check(hbp_select_groups(ctx(), ls.data(), static_cast<int32_t>(ls.size()), &f->p, sps.data(),
                                static_cast<int32_t>(sps.size()), out, &n, &lb, &lm));
        HierarchicalGroups h;
        for (int i = 0; i < n; ++i) h.groups.push_back(GroupConfig{out[i].length, RuntimeConfig{out[i].sp, out[i].ckpt}});
        h.l_best = lb;
        h.l_max = lm;
        return h;
    }
    // user-defined profiler: the reference algorithm against its virtuals
    if (candidate_lengths.empty()) throw ValidationError("select_groups: no candidate lengths");
    std::vector<Tokens> lengths(candidate_lengths.begin(), candidate_lengths.end());
    for (size_t i = 1; i < lengths.size(); ++i)
        if (lengths[i] <= lengths[i - 1]) throw ValidationError("candidate lengths must be strictly ascending");
    for (const int sp : sp_candidates)
        if (!pow2(sp)) throw ValidationError("sp candidates must be powers of two, got " + std::to_string(sp));
    struct Row {
        Tokens length;
        SpCkptChoice choice;
    };
    std::vector<Row> ok;
    std::string failures;
    for (const Tokens l : lengths) {
        try {
            ok.push_back(Row{l, find_best_sp_ckpt(profiler, l, sp_candidates)});
        } catch (const Error& e) {
            if (!failures.empty()) failures += "; ";
            failures += e.what();
        }
    }
    if (ok.empty()) throw InfeasibleError("no candidate length is feasible: " + failures);
    if (ok.back().length != lengths.back())
        throw InfeasibleError("largest candidate length " + std::to_string(lengths.back()) + " is infeasible: " + failures);
    size_t bi = 0;
    for (size_t i = 1; i < ok.size(); ++i)
        if (ok[i].choice.seconds < ok[bi].choice.seconds) bi = i;
    const Tokens l_best = ok[bi].length, l_max = ok.back().length;
    const RuntimeConfig s_best = ok[bi].choice.config, s_max = ok.back().choice.config;
    const Tokens l1 = l_best / s_best.sp, l2 = l_max / s_max.sp;
    std::vector<GroupConfig> raw;
    raw.push_back(GroupConfig{l1, RuntimeConfig{1, profiler.derive_ckpt(l1, 1)}});
    raw.push_back(GroupConfig{l_best, s_best});
    if (l2 > l_best) {
        const double target = static_cast<double>(l2) / static_cast<double>(l1);
        int bsp = -1, bck = 0;
        double bgap = 0.0;
        for (const int sp : sp_candidates) {
            if (!pow2(sp)) continue;
            int ck = 0;
            try {
                ck = profiler.derive_ckpt(l2, sp);
                if (profiler.profile_memory(l2, RuntimeConfig{sp, ck}) < 0) continue;
            } catch (const Error&) {
                continue;
            }
            const double gap = std::abs(std::log2(static_cast<double>(sp)) - std::log2(target));
            if (bsp < 0 || gap < bgap || (gap == bgap && sp < bsp)) {
                bsp = sp;
                bgap = gap;
                bck = ck;
            }
        }
        if (bsp < 0) throw InfeasibleError("no feasible sp for mid-level group of length " + std::to_string(l2));
        raw.push_back(GroupConfig{l2, RuntimeConfig{bsp, bck}});
    }
    raw.push_back(GroupConfig{l_max, s_max});
    std::map<Tokens, GroupConfig> dedup;
    for (const auto& g : raw) {
        auto it = dedup.find(g.length);
        if (it == dedup.end()) dedup.emplace(g.length, g);
        else if (g.config.sp < it->second.config.sp) it->second = g;
    }
    HierarchicalGroups out;
    for (const auto& [len, g] : dedup) out.groups.push_back(g);
    out.l_best = l_best;
    out.l_max = l_max;
    out.validate();
    return out;
}

}  // namespace hbp
