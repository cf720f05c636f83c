// core.cpp — the C++ drop-in façade over the B200 engine (types, metrics,
// packing, balance, sim). Every plan-level operation crosses the C-ABI
// (include/hbp_b200.h) into the CUDA engine; the façade converts between the
// reference's nested value types (include/hbp/*.hpp) and the flat CSR the
// engine works on. Scalar helpers over a few host values (dbr over one
// iteration, pr over one batch, ...) and the plan-invariant corpus
// fingerprint are evaluated in place, as the reference does.
#include <algorithm>
#include <array>
#include <cstring>
#include <string>
#include <vector>

#include "engine_ctx.hpp"
#include "hbp/balance.hpp"
#include "hbp/metrics.hpp"
#include "hbp/packing.hpp"
#include "hbp/rng.hpp"
#include "hbp/sim.hpp"
#include "hbp/types.hpp"
#include "hbp_b200.h"

namespace hbp {

using detail::check;
using detail::ctx;

namespace {

struct SoA {
    std::vector<int64_t> ids, lengths;
    hbp_samples view(const std::string& source) const {
        return hbp_samples{ids.data(), lengths.data(), static_cast<int64_t>(lengths.size()), HBP_MEM_HOST,
                           source.c_str()};
    }
};

SoA soa(const std::vector<Sample>& v) {
    SoA s;
    s.ids.reserve(v.size());
    s.lengths.reserve(v.size());
    for (const auto& x : v) {
        s.ids.push_back(x.id);
        s.lengths.push_back(x.length);
    }
    return s;
}

std::vector<hbp_group_config> flat_groups(const HierarchicalGroups& g) {
    std::vector<hbp_group_config> out;
    for (const auto& x : g.groups) out.push_back(hbp_group_config{x.length, x.config.sp, x.config.ckpt});
    return out;
}

hbp_strategy flat_strategy(const PackingStrategy& s) {
    return hbp_strategy{static_cast<int32_t>(s.kind), s.isf_iterations, s.isf_fill_threshold};
}

// owns a device plan handle
struct PlanHandle {
    hbp_plan* p = nullptr;
    ~PlanHandle() { hbp_plan_free(p); }
    hbp_plan_view view() {
        hbp_plan_view v{};
        check(hbp_plan_view_get(ctx(), p, &v));
        return v;
    }
};

Pack pack_from_view(const hbp_plan_view& v, int64_t q, const std::vector<Sample>& src) {
    Pack p = Pack::make(v.pack_capacity[q]);
    for (int64_t k = v.pack_member_offsets[q]; k < v.pack_member_offsets[q + 1]; ++k) p.add(src[v.member_index[k]]);
    return p;
}

std::vector<Iteration> iterations_from_view(const hbp_plan_view& v, const std::vector<Sample>& src,
                                            const HierarchicalGroups* groups, bool sp_comm_fixed) {
    std::vector<Iteration> out(static_cast<size_t>(v.n_iterations));
    for (int64_t i = 0; i < v.n_iterations; ++i) {
        Iteration& it = out[static_cast<size_t>(i)];
        it.group_index = v.iter_group[i];
        it.phase = (v.iter_phase && v.iter_phase[i]) ? Phase::Warmup : Phase::Hybrid;
        const bool sp = groups ? groups->groups.at(static_cast<size_t>(it.group_index)).config.sp > 1 : sp_comm_fixed;
        for (int64_t d = v.iter_dev_offsets[i]; d < v.iter_dev_offsets[i + 1]; ++d) {
            std::vector<Pack> packs;
            for (int64_t q = v.dev_pack_offsets[d]; q < v.dev_pack_offsets[d + 1]; ++q)
                packs.push_back(pack_from_view(v, q, src));
            it.devices.push_back(DeviceBatch::build(v.dev_index[d], std::move(packs), sp));
        }
    }
    return out;
}

// Plan -> flat arrays (no members) for hbp_report / hbp_simulate.
struct FlatPlan {
    std::vector<int32_t> iter_group, dev_index;
    std::vector<int64_t> iter_dev_offsets{0}, dev_pack_offsets{0}, cap, tot, att, member_off{0};
    std::vector<hbp_group_config> groups;
    hbp_plan_view v{};
    explicit FlatPlan(const Plan& plan) {
        groups = flat_groups(plan.groups);
        for (const auto& it : plan.iterations) {
            iter_group.push_back(it.group_index);
            for (const auto& d : it.devices) {
                dev_index.push_back(d.device_index);
                for (const auto& p : d.packs) {
                    cap.push_back(p.capacity);
                    tot.push_back(p.total);
                    att.push_back(p.attention);
                    member_off.push_back(member_off.back() + static_cast<int64_t>(p.samples.size()));
                }
                dev_pack_offsets.push_back(static_cast<int64_t>(cap.size()));
            }
            iter_dev_offsets.push_back(static_cast<int64_t>(dev_index.size()));
        }
        v.device_count = plan.device_count;
        v.seed = plan.seed;
        v.groups = hbp_groups{groups.data(), static_cast<int32_t>(groups.size()), plan.groups.l_best, plan.groups.l_max};
        v.n_iterations = static_cast<int64_t>(iter_group.size());
        v.n_devices = static_cast<int64_t>(dev_index.size());
        v.n_packs = static_cast<int64_t>(cap.size());
        v.n_members = member_off.back();
        v.iter_group = iter_group.data();
        v.iter_dev_offsets = iter_dev_offsets.data();
        v.dev_index = dev_index.data();
        v.dev_pack_offsets = dev_pack_offsets.data();
        v.pack_capacity = cap.data();
        v.pack_total = tot.data();
        v.pack_attention = att.data();
        v.pack_member_offsets = member_off.data();
        v.member_index = nullptr;
    }
};

// packs -> hbp_packs_in
struct FlatPacks {
    std::vector<int64_t> off{0}, cap, ids, lens;
    hbp_packs_in in{};
    explicit FlatPacks(const std::vector<Pack>& packs) {
        for (const auto& p : packs) {
            cap.push_back(p.capacity);
            for (const auto& s : p.samples) {
                ids.push_back(s.id);
                lens.push_back(s.length);
            }
            off.push_back(static_cast<int64_t>(ids.size()));
        }
        in = hbp_packs_in{static_cast<int64_t>(packs.size()), off.data(), cap.data(), ids.data(), lens.data()};
    }
};

}  // namespace

// ---------------------------------------------------------------------------
// types.hpp
// ---------------------------------------------------------------------------

void SampleSet::validate() const {
    const SoA s = soa(samples);
    const hbp_samples v = s.view(source);
    check(hbp_validate(ctx(), &v));
}

SampleSet apply_length_cap(const SampleSet& set, Tokens max_length, OverlongPolicy policy) {
    SampleSet out;
    out.source = set.source;
    out.samples.reserve(set.samples.size());
    for (const auto& s : set.samples) {
        if (s.length <= max_length) {
            out.samples.push_back(s);
        } else if (policy == OverlongPolicy::Error) {
            throw ValidationError("sample " + std::to_string(s.id) + " length " + std::to_string(s.length) +
                                  " exceeds max packing length " + std::to_string(max_length));
        } else if (policy == OverlongPolicy::TruncateToMax) {
            out.samples.push_back(Sample{s.id, max_length});
        }
    }
    return out;
}

CorpusFingerprint fingerprint(const std::vector<Sample>& samples) {
    std::vector<Sample> by_id = samples;
    std::sort(by_id.begin(), by_id.end(), [](const Sample& a, const Sample& b) { return a.id < b.id; });
    CorpusFingerprint fp;
    fp.sample_count = static_cast<int64_t>(by_id.size());
    uint64_t h = 0xcbf29ce484222325ULL;  // FNV-1a over (id, length) little-endian bytes
    for (const auto& s : by_id) {
        for (const uint64_t v : {static_cast<uint64_t>(s.id), static_cast<uint64_t>(s.length)})
            for (int b = 0; b < 8; ++b) {
                h ^= (v >> (8 * b)) & 0xffu;
                h *= 0x100000001b3ULL;
            }
        fp.total_tokens += s.length;
    }
    fp.id_hash = h;
    return fp;
}

// ---------------------------------------------------------------------------
// metrics.hpp
// ---------------------------------------------------------------------------

DeviceBatch DeviceBatch::build(int device_index, std::vector<Pack> packs, bool sp_comm) {
    DeviceBatch b;
    b.device_index = device_index;
    b.packs = std::move(packs);
    for (const auto& p : b.packs) {
        b.tokens += p.total;
        b.attention += p.attention;
    }
    b.comm_tokens = sp_comm ? b.tokens : 0;
    return b;
}

double dbr(std::span<const DeviceBatch> iteration) {
    if (iteration.empty()) throw ValidationError("dbr: no devices");
    Tokens top = 0;
    for (const auto& d : iteration) top = std::max(top, d.tokens);
    if (top == 0) throw ValidationError("dbr undefined: all devices carry zero tokens");
    double gap = 0.0;
    for (const auto& d : iteration) gap += static_cast<double>(top - d.tokens);
    return gap / (static_cast<double>(top) * static_cast<double>(iteration.size()));
}

double pr(std::span<const Tokens> lengths, Tokens t_max) {
    if (lengths.empty()) throw ValidationError("pr: empty batch");
    if (t_max <= 0) throw ValidationError("pr: t_max must be positive");
    double gap = 0.0;
    for (const Tokens t : lengths) {
        if (t > t_max)
            throw ValidationError("pr: length " + std::to_string(t) + " exceeds t_max " + std::to_string(t_max));
        gap += static_cast<double>(t_max - t);
    }
    return gap / (static_cast<double>(t_max) * static_cast<double>(lengths.size()));
}

double pack_pr(std::span<const Pack> packs) {
    double gap = 0.0, cap = 0.0;
    for (const auto& p : packs) {
        if (p.total > p.capacity) throw ValidationError("pr: pack total exceeds capacity");
        gap += static_cast<double>(p.capacity - p.total);
        cap += static_cast<double>(p.capacity);
    }
    if (cap == 0.0) throw ValidationError("pr: zero total capacity");
    return gap / cap;
}

double abr(std::span<const DeviceBatch> iteration) {
    if (iteration.empty()) throw ValidationError("abr: no devices");
    int64_t top = 0;
    for (const auto& d : iteration) top = std::max(top, d.attention);
    if (top == 0) throw ValidationError("abr undefined: all devices carry zero attention");
    double gap = 0.0;
    for (const auto& d : iteration) gap += static_cast<double>(top - d.attention);
    return gap / (static_cast<double>(top) * static_cast<double>(iteration.size()));
}

namespace {
// Σ tokens, Σ comm tokens, widest iteration of a run -- on the engine
// (hbp_run_totals); the ratios are formed here as the reference forms them
std::array<int64_t, 3> run_totals(std::span<const std::vector<DeviceBatch>> iterations) {
    std::vector<int64_t> tok, comm, off{0};
    for (const auto& it : iterations) {
        for (const auto& d : it) {
            tok.push_back(d.tokens);
            comm.push_back(d.comm_tokens);
        }
        off.push_back(static_cast<int64_t>(tok.size()));
    }
    std::array<int64_t, 3> out{0, 0, 0};
    check(hbp_run_totals(ctx(), tok.data(), comm.data(), off.data(), static_cast<int64_t>(iterations.size()),
                         out.data()));
    return out;
}
}  // namespace

double cr(std::span<const std::vector<DeviceBatch>> iterations) {
    const auto t = run_totals(iterations);
    if (t[0] == 0) throw ValidationError("cr: no tokens in run");
    return static_cast<double>(t[1]) / static_cast<double>(t[0]);
}

double ave_t(std::span<const std::vector<DeviceBatch>> iterations) {
    if (iterations.empty()) throw ValidationError("ave_t: no iterations");
    const auto t = run_totals(iterations);
    if (t[2] == 0) throw ValidationError("ave_t: no devices");
    return static_cast<double>(t[0]) / (static_cast<double>(iterations.size()) * static_cast<double>(t[2]));
}

MetricsReport report(const Plan& plan) {
    if (plan.iterations.empty()) throw ValidationError("metrics report: empty plan");
    FlatPlan f(plan);
    hbp_metrics m{};
    std::vector<double> d(plan.iterations.size()), a(plan.iterations.size());
    check(hbp_report(ctx(), &f.v, &m, d.data(), a.data()));
    MetricsReport r;
    r.dbr = m.dbr;
    r.pr = m.pr;
    r.abr = m.abr;
    r.cr = m.cr;
    r.ave_t = m.ave_t;
    r.per_iteration.resize(d.size());
    for (size_t i = 0; i < d.size(); ++i) r.per_iteration[i] = IterationTrace{d[i], a[i]};
    return r;
}

// ---------------------------------------------------------------------------
// packing.hpp
// ---------------------------------------------------------------------------

StrategyKind parse_strategy(const std::string& name) {
    static const std::pair<const char*, StrategyKind> names[] = {
        {"random", StrategyKind::Random}, {"isf", StrategyKind::Isf}, {"ffs", StrategyKind::Ffs},
        {"ffd", StrategyKind::Ffd},       {"bfs", StrategyKind::Bfs}, {"spfhp", StrategyKind::Spfhp}};
    for (const auto& [n, k] : names)
        if (name == n) return k;
    throw ValidationError("unknown packing strategy: " + name);
}

std::string strategy_name(StrategyKind kind) {
    switch (kind) {
        case StrategyKind::Random: return "random";
        case StrategyKind::Isf: return "isf";
        case StrategyKind::Ffs: return "ffs";
        case StrategyKind::Ffd: return "ffd";
        case StrategyKind::Bfs: return "bfs";
        case StrategyKind::Spfhp: return "spfhp";
    }
    return "?";
}

void PackingStrategy::validate() const {
    if (kind != StrategyKind::Isf) return;
    if (isf_iterations < 1) throw ValidationError("isf_iterations must be >= 1");
    if (isf_fill_threshold <= 0.0 || isf_fill_threshold > 1.0)
        throw ValidationError("isf fill threshold must lie in (0, 1]");
}

Tokens PackList::total_tokens() const {
    Tokens t = 0;
    for (const auto& p : packs) t += p.total;
    for (const auto& s : leftover) t += s.length;
    return t;
}

PackList pack(const SampleSet& samples, Tokens capacity, const PackingStrategy& strategy, std::uint64_t seed) {
    const SoA s = soa(samples.samples);
    const hbp_samples v = s.view(samples.source);
    const hbp_strategy st = flat_strategy(strategy);
    PlanHandle h;
    check(hbp_pack(ctx(), &v, capacity, &st, seed, &h.p));
    const hbp_plan_view pv = h.view();
    PackList out;
    out.capacity = capacity;
    out.packs.reserve(static_cast<size_t>(pv.n_packs));
    for (int64_t q = 0; q < pv.n_packs; ++q) out.packs.push_back(pack_from_view(pv, q, samples.samples));
    return out;
}

namespace {
// hbp_padded_batching (GPU) -> PaddedBatch lists
std::vector<PaddedBatch> padded(const SampleSet& samples, Tokens token_budget, int32_t mode, std::uint64_t seed) {
    const SoA s = soa(samples.samples);
    const hbp_samples v = s.view(samples.source);
    const size_t n = samples.samples.size();
    std::vector<int32_t> order(n ? n : 1);
    std::vector<int64_t> off(n + 1), mx(n ? n : 1);
    int64_t nb = 0;
    check(hbp_padded_batching(ctx(), &v, token_budget, mode, seed, order.data(), off.data(), mx.data(), &nb));
    std::vector<PaddedBatch> out(static_cast<size_t>(nb));
    for (int64_t b = 0; b < nb; ++b) {
        auto& pb = out[static_cast<size_t>(b)];
        for (int64_t k = off[b]; k < off[b + 1]; ++k) pb.samples.push_back(samples.samples[order[k]]);
        pb.max_length = mx[b];
        pb.padded_tokens = static_cast<Tokens>(pb.samples.size()) * pb.max_length;
    }
    return out;
}
}  // namespace

std::vector<PaddedBatch> sorted_batching(const SampleSet& samples, Tokens token_budget) {
    return padded(samples, token_budget, HBP_BATCHING_SORTED, 0);
}

std::vector<PaddedBatch> random_batching(const SampleSet& samples, Tokens token_budget, std::uint64_t seed) {
    return padded(samples, token_budget, HBP_BATCHING_RANDOM, seed);
}

// ---------------------------------------------------------------------------
// balance.hpp
// ---------------------------------------------------------------------------

CorpusFingerprint Plan::corpus() const { return fingerprint(all_samples()); }

std::vector<Sample> Plan::all_samples() const {
    std::vector<Sample> out;
    for (const auto& it : iterations)
        for (const auto& d : it.devices)
            for (const auto& p : d.packs) out.insert(out.end(), p.samples.begin(), p.samples.end());
    return out;
}

std::vector<SampleSet> group_data(const SampleSet& samples, const HierarchicalGroups& groups) {
    const SoA s = soa(samples.samples);
    const hbp_samples v = s.view(samples.source);
    auto g = flat_groups(groups);
    const hbp_groups hg{g.data(), static_cast<int32_t>(g.size()), groups.l_best, groups.l_max};
    std::vector<int64_t> off(g.size() + 1);
    std::vector<int32_t> mem(samples.samples.size() + 1);
    check(hbp_group_data(ctx(), &v, &hg, off.data(), mem.data()));
    std::vector<SampleSet> parts(g.size());
    for (size_t i = 0; i < parts.size(); ++i) {
        parts[i].source = samples.source + "#group" + std::to_string(i);
        for (int64_t k = off[i]; k < off[i + 1]; ++k) parts[i].samples.push_back(samples.samples[mem[k]]);
    }
    return parts;
}

void greedy_fill(PackList& packs, std::vector<SampleSet>& smaller_pools) {
    FlatPacks fp(packs.packs);
    std::vector<int64_t> pool_off{0}, pool_ids, pool_lens;
    for (const auto& p : smaller_pools) {
        for (const auto& s : p.samples) {
            pool_ids.push_back(s.id);
            pool_lens.push_back(s.length);
        }
        pool_off.push_back(static_cast<int64_t>(pool_ids.size()));
    }
    std::vector<int64_t> added_off(packs.packs.size() + 1), added(pool_ids.size() + 1);
    std::vector<uint8_t> keep(pool_ids.size() + 1);
    check(hbp_greedy_fill(ctx(), &fp.in, static_cast<int32_t>(smaller_pools.size()), pool_off.data(), pool_ids.data(),
                          pool_lens.data(), added_off.data(), added.data(), keep.data()));
    for (size_t p = 0; p < packs.packs.size(); ++p)
        for (int64_t k = added_off[p]; k < added_off[p + 1]; ++k)
            packs.packs[p].add(Sample{pool_ids[added[k]], pool_lens[added[k]]});
    for (size_t j = 0; j < smaller_pools.size(); ++j) {
        std::vector<Sample> rest;
        for (int64_t k = pool_off[j]; k < pool_off[j + 1]; ++k)
            if (keep[k]) rest.push_back(Sample{pool_ids[k], pool_lens[k]});
        smaller_pools[j].samples = std::move(rest);
    }
}

namespace {
std::vector<Iteration> batching(const PackList& packs, int device_count, int group_index, bool sp_comm, bool random,
                                std::uint64_t seed) {
    if (device_count < 1) throw ValidationError("device count must be >= 1");
    if (packs.packs.empty()) return {};
    FlatPacks fp(packs.packs);
    std::vector<Sample> members;
    for (const auto& p : packs.packs) members.insert(members.end(), p.samples.begin(), p.samples.end());
    PlanHandle h;
    check(hbp_balance_batching(ctx(), &fp.in, packs.capacity, device_count, group_index, random ? 1 : 0, seed, &h.p));
    return iterations_from_view(h.view(), members, nullptr, sp_comm);
}
}  // namespace

std::vector<Iteration> balance_batching(const PackList& packs, int device_count, int group_index, bool sp_comm) {
    return batching(packs, device_count, group_index, sp_comm, false, 0);
}

std::vector<Iteration> random_pack_batching(const PackList& packs, int device_count, int group_index, bool sp_comm,
                                            std::uint64_t seed) {
    return batching(packs, device_count, group_index, sp_comm, true, seed);
}

Plan build_plan(const SampleSet& samples, const HierarchicalGroups& groups, const PlanOptions& options) {
    const SoA s = soa(samples.samples);
    const hbp_samples v = s.view(samples.source);
    auto g = flat_groups(groups);
    const hbp_groups hg{g.data(), static_cast<int32_t>(g.size()), groups.l_best, groups.l_max};
    const hbp_plan_options o{flat_strategy(options.strategy), options.device_count, options.balance_batching ? 1 : 0,
                             options.greedy_fill ? 1 : 0, options.seed};
    PlanHandle h;
    check(hbp_build_plan(ctx(), &v, &hg, &o, &h.p));
    Plan plan;
    plan.groups = groups;
    plan.device_count = options.device_count;
    plan.seed = options.seed;
    plan.iterations = iterations_from_view(h.view(), samples.samples, &groups, false);
    return plan;
}

Plan build_batching_plan(const SampleSet& samples, GroupConfig group, int device_count, BatchingMode mode,
                         std::uint64_t seed) {
    const SoA s = soa(samples.samples);
    const hbp_samples v = s.view(samples.source);
    const hbp_group_config g{group.length, group.config.sp, group.config.ckpt};
    PlanHandle h;
    check(hbp_build_batching_plan(ctx(), &v, g, device_count,
                                  mode == BatchingMode::Sorted ? HBP_BATCHING_SORTED : HBP_BATCHING_RANDOM, seed, &h.p));
    Plan plan;
    plan.groups = HierarchicalGroups::single(group);
    plan.device_count = device_count;
    plan.seed = seed;
    plan.iterations = iterations_from_view(h.view(), samples.samples, &plan.groups, false);
    return plan;
}

// ---------------------------------------------------------------------------
// sim.hpp
// ---------------------------------------------------------------------------

hbp_hardware_profile to_flat(const HardwareProfile& p);

SimReport simulate(const Plan& plan, const HardwareProfile& profile, const std::string& name) {
    FlatPlan f(plan);
    const hbp_hardware_profile hp = to_flat(profile);
    hbp_sim_totals t{};
    std::vector<double> secs(plan.iterations.size() + 1), comp(f.dev_index.size() + 1), comm(f.dev_index.size() + 1),
        idle(f.dev_index.size() + 1);
    check(hbp_simulate(ctx(), &f.v, &hp, &t, secs.data(), comp.data(), comm.data(), idle.data()));
    SimReport r;
    r.name = name;
    r.device_count = plan.device_count;
    r.total_seconds = t.total_seconds;
    r.gpu_days = t.gpu_days;
    r.switch_count = t.switch_count;
    r.metrics = report(plan);
    r.corpus = plan.corpus();
    size_t d = 0;
    for (size_t i = 0; i < plan.iterations.size(); ++i) {
        IterationSim is;
        is.seconds = secs[i];
        for (const auto& dev : plan.iterations[i].devices) {
            DeviceSim ds;
            ds.tokens = dev.tokens;
            ds.compute_seconds = comp[d];
            ds.comm_seconds = comm[d];
            ds.idle_seconds = idle[d];
            is.devices.push_back(ds);
            ++d;
        }
        r.iterations.push_back(std::move(is));
    }
    return r;
}

std::vector<CompareRow> compare(std::span<const SimReport> reports) {
    if (reports.size() < 2) throw ValidationError("compare needs at least two reports");
    const auto& base = reports.front();
    for (const auto& r : reports)
        if (!(r.corpus == base.corpus))
            throw ValidationError("compare: report '" + r.name + "' describes a different corpus than '" + base.name +
                                  "'");
    std::vector<CompareRow> rows;
    for (const auto& r : reports) {
        CompareRow row;
        row.name = r.name;
        row.total_seconds = r.total_seconds;
        row.gpu_days = r.gpu_days;
        row.speedup = base.total_seconds / r.total_seconds;
        row.abr = r.metrics.abr;
        row.cr = r.metrics.cr;
        row.dbr = r.metrics.dbr;
        row.pr = r.metrics.pr;
        rows.push_back(row);
    }
    std::stable_sort(rows.begin(), rows.end(), [](const CompareRow& a, const CompareRow& b) { return a.speedup < b.speedup; });
    return rows;
}

}  // namespace hbp
