// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// Exposes the compiled reference planner (/root/reference/proj/src, built in
// place with the namespace renamed hbp -> hbp_ref by oracle/Makefile) through
// the oracle ABI of oracle/oracle.h. Nothing here re-implements an algorithm:
// every function converts flat arrays to the reference's types, calls the
// reference entry point named in its comment, and flattens the result.

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "hbp/autoselect.hpp"
#include "hbp/balance.hpp"
#include "hbp/io.hpp"
#include "hbp/schedule.hpp"
#include "hbp/costmodel.hpp"
#include "hbp/errors.hpp"
#include "hbp/ingest.hpp"
#include "hbp/metrics.hpp"
#include "hbp/packing.hpp"
#include "hbp/rng.hpp"
#include "hbp/sim.hpp"
#include "hbp/types.hpp"

#include "oracle.h"

namespace R = hbp_ref;

namespace {

void put_err(char* err, int errlen, const char* msg) {
    if (err == nullptr || errlen <= 0) return;
    std::strncpy(err, msg, static_cast<std::size_t>(errlen) - 1);
    err[errlen - 1] = '\0';
}

template <typename F>
int guarded(char* err, int errlen, F&& fn) {
    try {
        fn();
        return 0;
    } catch (const R::ValidationError& e) {
        put_err(err, errlen, e.what());
        return 2;
    } catch (const R::InfeasibleError& e) {
        put_err(err, errlen, e.what());
        return 3;
    } catch (const R::IoError& e) {
        put_err(err, errlen, e.what());
        return 4;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 5;
    }
}

R::SampleSet make_set(const int64_t* ids, const int64_t* lengths, int64_t n) {
    R::SampleSet s;
    s.source = "oracle";
    s.samples.resize(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
        s.samples[i] = R::Sample{ids ? ids[i] : i, lengths[i]};
    }
    return s;
}

R::HierarchicalGroups make_groups(const hbp_groups* g) {
    R::HierarchicalGroups h;
    for (int i = 0; i < g->count; ++i) {
        h.groups.push_back(R::GroupConfig{
            g->groups[i].length,
            R::RuntimeConfig{g->groups[i].sp, g->groups[i].ckpt}});
    }
    h.l_best = g->l_best;
    h.l_max = g->l_max;
    return h;
}

R::PackingStrategy make_strategy(const hbp_strategy* s) {
    R::PackingStrategy st;
    st.kind = static_cast<R::StrategyKind>(s->kind);
    st.isf_iterations = s->isf_iterations;
    st.isf_fill_threshold = s->isf_fill_threshold;
    return st;
}

R::HardwareProfile make_profile(const hbp_hardware_profile* p) {
    R::HardwareProfile h;
    h.per_token_linear_cost = p->per_token_linear_cost;
    h.per_token2_attention_cost = p->per_token2_attention_cost;
    h.sp_comm_cost = p->sp_comm_cost;
    h.gc_recompute_factor = p->gc_recompute_factor;
    h.fixed_iteration_cost = p->fixed_iteration_cost;
    h.layer_count = p->layer_count;
    h.base_memory = p->base_memory;
    h.per_token_activation_memory = p->per_token_activation_memory;
    h.gc_memory_saving_per_layer = p->gc_memory_saving_per_layer;
    h.reference_length = p->reference_length;
    h.device_memory = p->device_memory;
    return h;
}

// Owns whichever concrete reference profiler the flat description names.
struct ProfilerBox {
    std::unique_ptr<R::Profiler> p;
    explicit ProfilerBox(const hbp_profiler* d) {
        if (d->kind == HBP_PROFILER_ANALYTIC) {
            p = std::make_unique<R::AnalyticProfiler>(
                make_profile(&d->profile), d->ckpt_min, d->ckpt_max);
        } else {
            std::vector<R::ProfileRow> rows;
            for (int64_t i = 0; i < d->n_rows; ++i) {
                R::ProfileRow r;
                r.length = d->rows[i].length;
                r.sp = d->rows[i].sp;
                r.ckpt = d->rows[i].ckpt;
                r.memory_bytes = d->rows[i].memory_bytes;
                r.seconds = d->rows[i].seconds;
                r.oom = d->rows[i].oom != 0;
                rows.push_back(r);
            }
            p = std::make_unique<R::TableProfiler>(std::move(rows),
                                                   d->device_memory);
        }
    }
};

template <typename T>
T* dup(const std::vector<T>& v) {
    T* out = static_cast<T*>(std::malloc(sizeof(T) * (v.size() + 1)));
    if (!v.empty()) std::memcpy(out, v.data(), sizeof(T) * v.size());
    return out;
}

// Flattens pack lists (iterations empty) or full plans.
struct Flat {
    std::vector<int32_t> iter_group;
    std::vector<int64_t> iter_dev_offsets{0};
    std::vector<int32_t> dev_index;
    std::vector<int64_t> dev_pack_offsets{0};
    std::vector<int64_t> cap, tot, att, member_off{0}, mid, mlen;

    void add_pack(const R::Pack& p) {
        cap.push_back(p.capacity);
        tot.push_back(p.total);
        att.push_back(p.attention);
        for (const auto& s : p.samples) {
            mid.push_back(s.id);
            mlen.push_back(s.length);
        }
        member_off.push_back(static_cast<int64_t>(mid.size()));
    }
    void add_iteration(const R::Iteration& it) {
        iter_group.push_back(it.group_index);
        for (const auto& d : it.devices) {
            dev_index.push_back(d.device_index);
            for (const auto& p : d.packs) add_pack(p);
            dev_pack_offsets.push_back(static_cast<int64_t>(cap.size()));
        }
        iter_dev_offsets.push_back(static_cast<int64_t>(dev_index.size()));
    }
    oracle_plan* finish(int32_t device_count, uint64_t seed) const {
        auto* o = static_cast<oracle_plan*>(std::calloc(1, sizeof(oracle_plan)));
        o->device_count = device_count;
        o->seed = seed;
        o->n_iterations = static_cast<int64_t>(iter_group.size());
        o->n_devices = static_cast<int64_t>(dev_index.size());
        o->n_packs = static_cast<int64_t>(cap.size());
        o->n_members = static_cast<int64_t>(mid.size());
        o->iter_group = dup(iter_group);
        o->iter_dev_offsets = dup(iter_dev_offsets);
        o->dev_index = dup(dev_index);
        o->dev_pack_offsets = dup(dev_pack_offsets);
        o->pack_capacity = dup(cap);
        o->pack_total = dup(tot);
        o->pack_attention = dup(att);
        o->pack_member_offsets = dup(member_off);
        o->member_id = dup(mid);
        o->member_length = dup(mlen);
        return o;
    }
};

R::PackList packlist_from(const oracle_plan* o) {
    R::PackList l;
    l.capacity = o->n_packs > 0 ? o->pack_capacity[0] : 0;
    for (int64_t p = 0; p < o->n_packs; ++p) {
        R::Pack pk = R::Pack::make(o->pack_capacity[p]);
        for (int64_t k = o->pack_member_offsets[p];
             k < o->pack_member_offsets[p + 1]; ++k) {
            pk.add(R::Sample{o->member_id[k], o->member_length[k]});
        }
        l.packs.push_back(std::move(pk));
    }
    return l;
}

// Plan from a view: packs carry only capacity / total / attention.
R::Plan plan_from_view(const hbp_plan_view* v) {
    R::Plan plan;
    plan.groups = make_groups(&v->groups);
    plan.device_count = v->device_count;
    plan.seed = v->seed;
    plan.iterations.resize(static_cast<std::size_t>(v->n_iterations));
    for (int64_t i = 0; i < v->n_iterations; ++i) {
        auto& it = plan.iterations[i];
        it.group_index = v->iter_group[i];
        for (int64_t d = v->iter_dev_offsets[i]; d < v->iter_dev_offsets[i + 1];
             ++d) {
            R::DeviceBatch b;
            b.device_index = v->dev_index ? v->dev_index[d] : 0;
            std::vector<R::Pack> packs;
            for (int64_t p = v->dev_pack_offsets[d]; p < v->dev_pack_offsets[d + 1];
                 ++p) {
                R::Pack pk = R::Pack::make(v->pack_capacity[p]);
                pk.total = v->pack_total[p];
                pk.attention = v->pack_attention[p];
                packs.push_back(std::move(pk));
            }
            const bool sp = plan.groups.groups.at(it.group_index).config.sp > 1;
            b = R::DeviceBatch::build(b.device_index, std::move(packs), sp);
            it.devices.push_back(std::move(b));
        }
    }
    return plan;
}

} // namespace

extern "C" {

void oracle_plan_free(oracle_plan* p) {
    if (p == nullptr) return;
    std::free(p->iter_group);
    std::free(p->iter_dev_offsets);
    std::free(p->dev_index);
    std::free(p->dev_pack_offsets);
    std::free(p->pack_capacity);
    std::free(p->pack_total);
    std::free(p->pack_attention);
    std::free(p->pack_member_offsets);
    std::free(p->member_id);
    std::free(p->member_length);
    std::free(p);
}

int oracle_kind(void) { return 2; }

int oracle_synth_lengths(int64_t count, const char* short_dist,
                         double long_fraction, const char* long_dist,
                         int64_t max_length, uint64_t seed, int64_t* lengths,
                         char* err, int errlen) {
    return guarded(err, errlen, [&] {
        R::SynthSpec spec;
        spec.count = count;
        spec.short_dist = R::parse_distribution(short_dist);
        spec.long_fraction = long_fraction;
        spec.long_dist = (long_dist == nullptr || long_dist[0] == '\0')
                             ? spec.short_dist
                             : R::parse_distribution(long_dist);
        spec.max_length = max_length;
        spec.seed = seed;
        const auto s = R::synth_lengths(spec);
        for (std::size_t i = 0; i < s.samples.size(); ++i) {
            lengths[i] = s.samples[i].length;
        }
    });
}

int oracle_shuffle_positions(uint64_t seed, int64_t m, uint32_t* out) {
    std::vector<uint32_t> v(static_cast<std::size_t>(m));
    for (int64_t i = 0; i < m; ++i) v[i] = static_cast<uint32_t>(i);
    R::Rng rng(seed);
    rng.shuffle(v);
    std::memcpy(out, v.data(), sizeof(uint32_t) * v.size());
    return 0;
}

int oracle_validate(const int64_t* ids, const int64_t* lengths, int64_t n,
                    char* err, int errlen) {
    return guarded(err, errlen, [&] { make_set(ids, lengths, n).validate(); });
}

int oracle_fingerprint(const int64_t* ids, const int64_t* lengths, int64_t n,
                       uint64_t* hash, int64_t* count, int64_t* tokens) {
    const auto fp = R::fingerprint(make_set(ids, lengths, n).samples);
    *hash = fp.id_hash;
    *count = fp.sample_count;
    *tokens = fp.total_tokens;
    return 0;
}

int oracle_group_data(const int64_t* ids, const int64_t* lengths, int64_t n,
                      const hbp_groups* groups, oracle_plan** out, char* err,
                      int errlen) {
    return guarded(err, errlen, [&] {
        const auto g = make_groups(groups);
        const auto parts = R::group_data(make_set(ids, lengths, n), g);
        Flat f;
        for (std::size_t i = 0; i < parts.size(); ++i) {
            R::Pack p = R::Pack::make(g.groups[i].length);
            for (const auto& s : parts[i].samples) p.add(s);
            f.add_pack(p);
        }
        *out = f.finish(0, 0);
    });
}

int oracle_pack(const int64_t* ids, const int64_t* lengths, int64_t n,
                int64_t capacity, const hbp_strategy* strategy, uint64_t seed,
                oracle_plan** out, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const auto l = R::pack(make_set(ids, lengths, n), capacity,
                               make_strategy(strategy), seed);
        Flat f;
        for (const auto& p : l.packs) f.add_pack(p);
        *out = f.finish(0, seed);
    });
}

int oracle_greedy_fill(const oracle_plan* packs, const oracle_plan* pools,
                       oracle_plan** out_packs, oracle_plan** out_pools,
                       char* err, int errlen) {
    return guarded(err, errlen, [&] {
        R::PackList list = packlist_from(packs);
        std::vector<R::SampleSet> ps(static_cast<std::size_t>(pools->n_packs));
        for (int64_t j = 0; j < pools->n_packs; ++j) {
            for (int64_t k = pools->pack_member_offsets[j];
                 k < pools->pack_member_offsets[j + 1]; ++k) {
                ps[j].samples.push_back(
                    R::Sample{pools->member_id[k], pools->member_length[k]});
            }
        }
        R::greedy_fill(list, ps);
        Flat a;
        for (const auto& p : list.packs) a.add_pack(p);
        *out_packs = a.finish(0, 0);
        Flat b;
        for (std::size_t j = 0; j < ps.size(); ++j) {
            R::Pack p = R::Pack::make(pools->pack_capacity[j]);
            for (const auto& s : ps[j].samples) p.add(s);
            b.add_pack(p);
        }
        *out_pools = b.finish(0, 0);
    });
}

int oracle_balance_batching(const oracle_plan* packs, int32_t device_count,
                            int32_t group_index, int32_t sp_comm,
                            int32_t random_batching, uint64_t seed,
                            oracle_plan** out, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const R::PackList list = packlist_from(packs);
        const auto its =
            random_batching
                ? R::random_pack_batching(list, device_count, group_index,
                                          sp_comm != 0, seed)
                : R::balance_batching(list, device_count, group_index,
                                      sp_comm != 0);
        Flat f;
        for (const auto& it : its) f.add_iteration(it);
        *out = f.finish(device_count, seed);
    });
}

int oracle_build_plan(const int64_t* ids, const int64_t* lengths, int64_t n,
                      const hbp_groups* groups, const hbp_plan_options* options,
                      oracle_plan** out, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        R::PlanOptions o;
        o.strategy = make_strategy(&options->strategy);
        o.device_count = options->device_count;
        o.seed = options->seed;
        o.balance_batching = options->balance_batching != 0;
        o.greedy_fill = options->greedy_fill != 0;
        const auto plan =
            R::build_plan(make_set(ids, lengths, n), make_groups(groups), o);
        Flat f;
        for (const auto& it : plan.iterations) f.add_iteration(it);
        *out = f.finish(plan.device_count, plan.seed);
    });
}

// plan_from_json (io.cpp:112-160) of a manifest text.
int oracle_plan_from_json(const char* text, int64_t bytes, oracle_plan** out, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const auto plan = R::plan_from_json(std::string(text, static_cast<std::size_t>(bytes)));
        Flat f;
        for (const auto& it : plan.iterations) f.add_iteration(it);
        *out = f.finish(plan.device_count, plan.seed);
    });
}

// The reference's plan manifest (io.cpp plan_to_json) of build_plan's plan;
// *out is malloc'd (oracle_free_text).
int oracle_build_plan_json(const int64_t* ids, const int64_t* lengths, int64_t n,
                           const hbp_groups* groups, const hbp_plan_options* options,
                           char** out, int64_t* out_len, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        R::PlanOptions o;
        o.strategy = make_strategy(&options->strategy);
        o.device_count = options->device_count;
        o.seed = options->seed;
        o.balance_batching = options->balance_batching != 0;
        o.greedy_fill = options->greedy_fill != 0;
        const auto plan =
            R::build_plan(make_set(ids, lengths, n), make_groups(groups), o);
        const std::string text = R::plan_to_json(plan);
        *out = static_cast<char*>(std::malloc(text.size() + 1));
        std::memcpy(*out, text.c_str(), text.size() + 1);
        *out_len = static_cast<int64_t>(text.size());
    });
}

void oracle_free_text(char* p) { std::free(p); }

// curriculum_order(build_plan(...)): its manifest, schedule CSV and
// runtime assignment (sp / ckpt per iteration, switch count).
int oracle_curriculum(const int64_t* ids, const int64_t* lengths, int64_t n,
                      const hbp_groups* groups, const hbp_plan_options* options,
                      int32_t warmup, int32_t cutoff, char** json, int64_t* json_len,
                      char** csv, int64_t* csv_len, int32_t* sp, int32_t* ckpt,
                      int64_t* switch_count, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        R::PlanOptions o;
        o.strategy = make_strategy(&options->strategy);
        o.device_count = options->device_count;
        o.seed = options->seed;
        o.balance_batching = options->balance_batching != 0;
        o.greedy_fill = options->greedy_fill != 0;
        const auto plan =
            R::build_plan(make_set(ids, lengths, n), make_groups(groups), o);
        R::CurriculumSpec spec;
        spec.warmup_iterations = warmup;
        spec.short_group_cutoff = cutoff;
        const auto cur = R::curriculum_order(plan, spec);
        auto dup = [](const std::string& t, char** out, int64_t* len) {
            *out = static_cast<char*>(std::malloc(t.size() + 1));
            std::memcpy(*out, t.c_str(), t.size() + 1);
            *len = static_cast<int64_t>(t.size());
        };
        dup(R::plan_to_json(cur), json, json_len);
        std::ostringstream os;
        R::write_schedule_csv(cur, os);
        dup(os.str(), csv, csv_len);
        const auto ra = R::assign_runtime(cur);
        for (std::size_t i = 0; i < ra.per_iteration.size(); ++i) {
            sp[i] = ra.per_iteration[i].sp;
            ckpt[i] = ra.per_iteration[i].ckpt;
        }
        *switch_count = ra.switch_count;
    });
}

// The reference's build_batching_plan manifest and padded batches
// (mode 0 sorted, 1 random).
int oracle_build_batching_plan_json(const int64_t* ids, const int64_t* lengths, int64_t n,
                                    int64_t length, int32_t sp, int32_t ckpt,
                                    int32_t device_count, int32_t mode, uint64_t seed,
                                    char** out, int64_t* out_len, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        R::GroupConfig g;
        g.length = length;
        g.config.sp = sp;
        g.config.ckpt = ckpt;
        const auto plan = R::build_batching_plan(
            make_set(ids, lengths, n), g, device_count,
            mode == 0 ? R::BatchingMode::Sorted : R::BatchingMode::Random, seed);
        const std::string text = R::plan_to_json(plan);
        *out = static_cast<char*>(std::malloc(text.size() + 1));
        std::memcpy(*out, text.c_str(), text.size() + 1);
        *out_len = static_cast<int64_t>(text.size());
    });
}

int oracle_padded_batching(const int64_t* ids, const int64_t* lengths, int64_t n,
                           int64_t budget, int32_t mode, uint64_t seed, int64_t* order_ids,
                           int64_t* batch_offsets, int64_t* batch_max, int64_t* n_batches,
                           char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const auto set = make_set(ids, lengths, n);
        const auto b = mode == 0 ? R::sorted_batching(set, budget)
                                 : R::random_batching(set, budget, seed);
        int64_t k = 0;
        for (std::size_t i = 0; i < b.size(); ++i) {
            batch_offsets[i] = k;
            batch_max[i] = b[i].max_length;
            for (const auto& smp : b[i].samples) order_ids[k++] = smp.id;
        }
        batch_offsets[b.size()] = k;
        *n_batches = static_cast<int64_t>(b.size());
    });
}

// load_lengths(istream, format, source) (ingest.cpp:147-160) over a text
// buffer: lengths[capacity] (ids are 0..n-1 for csv / raw).
int oracle_load_lengths(const char* text, int64_t bytes, int32_t format, const char* source,
                        int64_t* lengths, int64_t* ids, int64_t capacity, int64_t* n, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        std::istringstream in(std::string(text, static_cast<std::size_t>(bytes)));
        const R::CorpusFormat f = format == 0 ? R::CorpusFormat::Jsonl
                                 : format == 1 ? R::CorpusFormat::Csv : R::CorpusFormat::RawLengths;
        const auto set = R::load_lengths(in, f, source);
        if (static_cast<int64_t>(set.samples.size()) > capacity) throw R::ValidationError("oracle capacity");
        for (std::size_t i = 0; i < set.samples.size(); ++i) {
            lengths[i] = set.samples[i].length;
            ids[i] = set.samples[i].id;
        }
        *n = static_cast<int64_t>(set.samples.size());
    });
}

int oracle_report(const hbp_plan_view* plan, hbp_metrics* out, double* dbr,
                  double* abr, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const auto rep = R::report(plan_from_view(plan));
        out->dbr = rep.dbr;
        out->pr = rep.pr;
        out->abr = rep.abr;
        out->cr = rep.cr;
        out->ave_t = rep.ave_t;
        for (std::size_t i = 0; i < rep.per_iteration.size(); ++i) {
            if (dbr) dbr[i] = rep.per_iteration[i].dbr;
            if (abr) abr[i] = rep.per_iteration[i].abr;
        }
    });
}

int oracle_simulate(const hbp_plan_view* plan,
                    const hbp_hardware_profile* profile, hbp_sim_totals* out,
                    double* iteration_seconds, double* device_compute,
                    double* device_comm, double* device_idle, char* err,
                    int errlen) {
    return guarded(err, errlen, [&] {
        const auto rep = R::simulate(plan_from_view(plan), make_profile(profile));
        out->total_seconds = rep.total_seconds;
        out->gpu_days = rep.gpu_days;
        out->switch_count = rep.switch_count;
        out->device_count = rep.device_count;
        out->metrics.dbr = rep.metrics.dbr;
        out->metrics.pr = rep.metrics.pr;
        out->metrics.abr = rep.metrics.abr;
        out->metrics.cr = rep.metrics.cr;
        out->metrics.ave_t = rep.metrics.ave_t;
        std::size_t d = 0;
        for (std::size_t i = 0; i < rep.iterations.size(); ++i) {
            if (iteration_seconds) iteration_seconds[i] = rep.iterations[i].seconds;
            for (const auto& dev : rep.iterations[i].devices) {
                if (device_compute) device_compute[d] = dev.compute_seconds;
                if (device_comm) device_comm[d] = dev.comm_seconds;
                if (device_idle) device_idle[d] = dev.idle_seconds;
                ++d;
            }
        }
    });
}

int oracle_memory_used(int64_t length, int32_t sp, int32_t ckpt,
                       const hbp_hardware_profile* profile, int64_t* out,
                       char* err, int errlen) {
    return guarded(err, errlen, [&] {
        *out = R::memory_used(length, R::RuntimeConfig{sp, ckpt},
                              make_profile(profile));
    });
}

int oracle_iter_time(const int64_t* capacity, const int64_t* total,
                     const int64_t* attention, int64_t n_packs, int32_t sp,
                     int32_t ckpt, const hbp_hardware_profile* profile,
                     double* out, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        std::vector<R::Pack> packs;
        for (int64_t p = 0; p < n_packs; ++p) {
            R::Pack pk = R::Pack::make(capacity[p]);
            pk.total = total[p];
            pk.attention = attention[p];
            packs.push_back(pk);
        }
        *out = R::iter_time(std::span<const R::Pack>(packs),
                            R::RuntimeConfig{sp, ckpt}, make_profile(profile));
    });
}

int oracle_profile_time(const hbp_profiler* profiler, int64_t length,
                        int32_t sp, int32_t ckpt, double* out, char* err,
                        int errlen) {
    return guarded(err, errlen, [&] {
        ProfilerBox b(profiler);
        *out = b.p->profile_time(length, R::RuntimeConfig{sp, ckpt});
    });
}

int oracle_profile_memory(const hbp_profiler* profiler, int64_t length,
                          int32_t sp, int32_t ckpt, int64_t* out, char* err,
                          int errlen) {
    return guarded(err, errlen, [&] {
        ProfilerBox b(profiler);
        *out = b.p->profile_memory(length, R::RuntimeConfig{sp, ckpt});
    });
}

int oracle_derive_ckpt(const hbp_profiler* profiler, int64_t length,
                       int32_t sp, int32_t* out, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ProfilerBox b(profiler);
        *out = b.p->derive_ckpt(length, sp);
    });
}

int oracle_greedy_profile_ckpt(const hbp_profiler* profiler, int64_t length,
                               int32_t sp, int32_t ckpt_min, int32_t ckpt_max,
                               int32_t* out, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ProfilerBox b(profiler);
        *out = R::greedy_profile_ckpt(*b.p, length, sp, ckpt_min, ckpt_max);
    });
}

int oracle_find_best_sp_ckpt(const hbp_profiler* profiler, int64_t length,
                             const int32_t* sp, int32_t n_sp, int32_t* out_sp,
                             int32_t* out_ckpt, double* out_seconds,
                             char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ProfilerBox b(profiler);
        std::vector<int> sps(sp, sp + n_sp);
        const auto c = R::find_best_sp_ckpt(*b.p, length, sps);
        *out_sp = c.config.sp;
        *out_ckpt = c.config.ckpt;
        *out_seconds = c.seconds;
    });
}

int oracle_select_groups(const int64_t* lengths, int32_t n_lengths,
                         const hbp_profiler* profiler, const int32_t* sp,
                         int32_t n_sp, hbp_group_config* out_groups,
                         int32_t* out_count, int64_t* out_l_best,
                         int64_t* out_l_max, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ProfilerBox b(profiler);
        std::vector<R::Tokens> ls(lengths, lengths + n_lengths);
        std::vector<int> sps(sp, sp + n_sp);
        const auto h = R::select_groups(ls, *b.p, sps);
        *out_count = static_cast<int32_t>(h.groups.size());
        for (std::size_t i = 0; i < h.groups.size(); ++i) {
            out_groups[i].length = h.groups[i].length;
            out_groups[i].sp = h.groups[i].config.sp;
            out_groups[i].ckpt = h.groups[i].config.ckpt;
        }
        *out_l_best = h.l_best;
        *out_l_max = h.l_max;
    });
}

int oracle_sweep(const int64_t* ids, const int64_t* lengths, int64_t n,
                 const hbp_group_config* cand_groups,
                 const int64_t* cand_offsets, const int64_t* cand_l_best,
                 int64_t n_candidates, const hbp_plan_options* options,
                 const hbp_hardware_profile* profile, double* out_seconds,
                 int64_t* out_best, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const auto set = make_set(ids, lengths, n);
        const auto prof = make_profile(profile);
        R::PlanOptions o;
        o.strategy = make_strategy(&options->strategy);
        o.device_count = options->device_count;
        o.seed = options->seed;
        o.balance_batching = options->balance_batching != 0;
        o.greedy_fill = options->greedy_fill != 0;
        int64_t best = -1;
        for (int64_t c = 0; c < n_candidates; ++c) {
            hbp_groups g{cand_groups + cand_offsets[c],
                         static_cast<int32_t>(cand_offsets[c + 1] - cand_offsets[c]),
                         cand_l_best[c],
                         cand_groups[cand_offsets[c + 1] - 1].length};
            double t = std::numeric_limits<double>::infinity();
            try {
                t = R::simulate(R::build_plan(set, make_groups(&g), o), prof)
                        .total_seconds;
            } catch (const R::InfeasibleError&) {
            }
            out_seconds[c] = t;
            if (t != std::numeric_limits<double>::infinity() &&
                (best < 0 || t < out_seconds[best])) {
                best = c;
            }
        }
        *out_best = best;
    });
}

} // extern "C"
