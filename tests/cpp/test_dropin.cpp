// test_dropin.cpp — the reference C++ API (include/hbp/*.hpp) exercised
// through the B200 façade: known answers of the reference's own test suite
// (proj/tests/*.cpp, cited per case). Built by tests/cpp/Makefile, run by
// tests/test_gpu_dropin.py on a B200. Exit code = number of failures.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "hbp/autoselect.hpp"
#include "hbp/balance.hpp"
#include "hbp/costmodel.hpp"
#include "hbp/ingest.hpp"
#include "hbp/io.hpp"
#include "hbp/schedule.hpp"
#include "hbp/metrics.hpp"
#include "hbp/packing.hpp"
#include "hbp/rng.hpp"
#include "hbp/sim.hpp"

using namespace hbp;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                            \
    do {                                                                    \
        ++g_checks;                                                         \
        if (!(c)) {                                                         \
            ++g_fail;                                                       \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);        \
        }                                                                   \
    } while (0)

template <typename E, typename F>
static void expect_throw(F&& f, const std::string& needle, int line) {
    ++g_checks;
    try {
        f();
    } catch (const E& e) {
        if (std::string(e.what()).find(needle) == std::string::npos) {
            ++g_fail;
            std::printf("FAIL line %d: message '%s' lacks '%s'\n", line, e.what(), needle.c_str());
        }
        return;
    } catch (const std::exception& e) {
        ++g_fail;
        std::printf("FAIL line %d: wrong exception: %s\n", line, e.what());
        return;
    }
    ++g_fail;
    std::printf("FAIL line %d: no exception\n", line);
}
#define EXPECT_THROW(E, expr, needle) expect_throw<E>([&] { expr; }, needle, __LINE__)

static SampleSet make_set(const std::vector<Tokens>& lengths) {
    SampleSet s;
    s.source = "test";
    for (size_t i = 0; i < lengths.size(); ++i) s.samples.push_back(Sample{static_cast<SampleId>(i), lengths[i]});
    return s;
}

static Pack make_pack(const std::vector<Tokens>& lengths, Tokens cap) {
    Pack p = Pack::make(cap);
    SampleId id = 0;
    for (auto t : lengths) p.add(Sample{id++, t});
    return p;
}

static HierarchicalGroups two_level(Tokens s = 16384, Tokens l = 131072, int sp = 8) {
    HierarchicalGroups g;
    g.groups = {GroupConfig{s, RuntimeConfig{1, 28}}, GroupConfig{l, RuntimeConfig{sp, 29}}};
    g.l_best = s;
    g.l_max = l;
    return g;
}

static SampleSet hybrid(size_t count, double lf, Tokens short_cap, Tokens max_len, uint64_t seed) {
    Rng rng(seed);  // tests/helpers.hpp hybrid_corpus
    SampleSet set;
    set.source = "hybrid-test";
    const auto nlong = static_cast<size_t>(static_cast<double>(count) * lf);
    for (size_t i = 0; i < count; ++i) {
        Tokens len;
        if (i < count - nlong) {
            const double v = std::exp(7.0 + 0.8 * rng.normal());
            len = std::max<Tokens>(1, std::min<Tokens>(static_cast<Tokens>(v), short_cap));
        } else {
            len = rng.uniform_int(short_cap + 1, max_len);
        }
        set.samples.push_back(Sample{static_cast<SampleId>(i), len});
    }
    return set;
}

static std::multiset<std::vector<Tokens>> compositions(const PackList& l) {
    std::multiset<std::vector<Tokens>> out;
    for (const auto& p : l.packs) {
        std::vector<Tokens> v;
        for (const auto& s : p.samples) v.push_back(s.length);
        std::sort(v.begin(), v.end());
        out.insert(v);
    }
    return out;
}

int main() {
    // ---- metrics (test_metrics.cpp:43-49, acceptance.cpp:104-113) ----
    {
        std::vector<DeviceBatch> it;
        it.push_back(DeviceBatch::build(0, {make_pack({1024, 1024, 1024, 1024}, 4096)}, false));
        it.push_back(DeviceBatch::build(1, {make_pack({2048, 2048}, 4096)}, false));
        CHECK(abr(it) == 0.25);
    }
    // ---- packing (test_packing.cpp) ----
    {
        PackingStrategy ffd;
        ffd.kind = StrategyKind::Ffd;
        const auto l = pack(make_set({3, 3, 2, 2, 1, 1}), 4, ffd, 0);  // :84-90
        const std::multiset<std::vector<Tokens>> want = {{1, 3}, {1, 3}, {2, 2}};
        CHECK(compositions(l) == want);
        EXPECT_THROW(ValidationError, pack(make_set({3, 9, 2}), 4, ffd, 0), "sample 1");  // :106-110
        {
            PackingStrategy sp;
            sp.kind = StrategyKind::Spfhp;  // :183-193
            const auto l2 = pack(make_set({512, 512, 512, 512, 512, 512, 256, 256, 256, 256}), 1024, sp, 0);
            CHECK(l2.packs.size() == 4);
            for (const auto& p : l2.packs) CHECK(p.total == 1024);
        }
        for (auto kind : {StrategyKind::Random, StrategyKind::Isf, StrategyKind::Ffs, StrategyKind::Ffd,
                          StrategyKind::Bfs, StrategyKind::Spfhp}) {
            PackingStrategy s;
            s.kind = kind;
            const auto r = pack(make_set({4, 4, 4, 4}), 4, s, 1);  // :71-82
            CHECK(r.packs.size() == 4);
            for (const auto& p : r.packs) CHECK(p.total == 4 && p.samples.size() == 1);
        }
    }
    // ---- plan manifest (test_io.cpp:33-71) ----
    {
        SampleSet set;
        set.source = "io";
        for (int i = 0; i < 400; ++i) set.samples.push_back(Sample{i, 100 + (i * 7919) % 60000});
        PlanOptions o;
        o.device_count = 4;
        o.seed = 3;
        const Plan plan = build_plan(set, two_level(), o);
        const std::string text = plan_to_json(plan);
        const Plan parsed = plan_from_json(text);
        CHECK(plan_to_json(parsed) == text);  // :33-53 bit-exact round trip
        CHECK(parsed.iterations.size() == plan.iterations.size() && parsed.device_count == 4 && parsed.seed == 3);
        EXPECT_THROW(ValidationError, plan_from_json("{}"), "plan manifest");           // :55-59
        // schedule (test_schedule.cpp): runtime per iteration and the CSV rows
        const RuntimeAssignment ra = assign_runtime(plan);
        CHECK(ra.per_iteration.size() == plan.iterations.size());
        std::ostringstream csv;
        write_schedule_csv(plan, csv);
        const std::string rows = csv.str();
        CHECK(rows.rfind("iteration,group,sp,ckpt,phase\n", 0) == 0);
        CHECK(static_cast<size_t>(std::count(rows.begin(), rows.end(), '\n')) == plan.iterations.size() + 1);
        EXPECT_THROW(ValidationError, plan_from_json("not json"), "bad plan manifest");
        std::string bad = text;
        const auto k = bad.find("\"capacity\": ");
        bad.replace(k, bad.find(',', k) - k, "\"capacity\": 1");
        EXPECT_THROW(ValidationError, plan_from_json(bad), "pack exceeds its capacity");  // :61-71
    }
    // ---- ingest (test_ingest.cpp:12-86) ----
    {
        std::istringstream a("{\"length\":4096}\n{\"length\":131072}\n");
        const auto s1 = load_lengths(a, CorpusFormat::Jsonl, "mem");
        CHECK(s1.samples.size() == 2 && s1.samples[1].length == 131072 && s1.samples[1].id == 1);
        std::istringstream b("{\"id\":7,\"length\":10}\n\n{\"length\":20}\n");
        const auto s2 = load_lengths(b, CorpusFormat::Jsonl, "mem");
        CHECK(s2.samples.size() == 2 && s2.samples[0].id == 7 && s2.samples[1].id == 1);
        std::istringstream e("");
        EXPECT_THROW(ValidationError, load_lengths(e, CorpusFormat::Jsonl, "mem"), "empty corpus");
        std::istringstream c("name,length,extra\na,1,x\nb,2,y\nc,3,z\n");
        const auto s3 = load_lengths(c, CorpusFormat::Csv, "mem");
        CHECK(s3.samples.size() == 3 && s3.samples[2].length == 3 && s3.samples[2].id == 2);
        std::istringstream nc("tokens\n5\n");
        EXPECT_THROW(ValidationError, load_lengths(nc, CorpusFormat::Csv, "mem"), "no \"length\" column");
        std::istringstream r("12\n34\n56\n");
        CHECK(load_lengths(r, CorpusFormat::RawLengths, "mem").samples[2].length == 56);
        std::istringstream bad("10\nnonsense\n30\n");
        EXPECT_THROW(ValidationError, load_lengths(bad, CorpusFormat::RawLengths, "mem"), "line 2");
        std::istringstream z("{\"length\":0}\n"), neg("{\"length\":-3}\n");
        EXPECT_THROW(ValidationError, load_lengths(z, CorpusFormat::Jsonl, "mem"), "length must be >= 1");
        EXPECT_THROW(ValidationError, load_lengths(neg, CorpusFormat::Jsonl, "mem"), "got -3");
        SampleSet set;
        set.source = "rt";
        set.samples = {Sample{5, 100}, Sample{9, 7}};
        std::ostringstream out;
        write_jsonl(set, out);
        std::istringstream back(out.str());
        const auto s4 = load_lengths(back, CorpusFormat::Jsonl, "mem");
        CHECK(s4.samples.size() == 2 && s4.samples[0].id == 5 && s4.samples[1].length == 7);
        EXPECT_THROW(ValidationError, parse_corpus_format("xml"), "unknown corpus format: xml");
    }
    // ---- balance (test_balance.cpp) ----
    {
        SampleSet set;
        set.source = "t";
        set.samples = {Sample{0, 4096}, Sample{1, 20480}, Sample{2, 102400}};
        const auto parts = group_data(set, two_level());  // :68-78
        CHECK(parts.size() == 2 && parts[0].samples.size() == 1 && parts[1].samples.size() == 2);
        CHECK(parts[0].source == "t#group0");
        SampleSet edge;
        edge.source = "t";
        edge.samples = {Sample{0, 16384}};
        CHECK(group_data(edge, two_level())[0].samples.size() == 1);  // :80-88
        SampleSet over;
        over.source = "t";
        over.samples = {Sample{0, 131073}};
        EXPECT_THROW(ValidationError, group_data(over, two_level()), "exceeds the largest packing length");
    }
    {
        PackList list;  // greedy_fill hand-run, :108-123
        list.capacity = 131072;
        list.packs.push_back(make_pack({102400}, 131072));
        std::vector<SampleSet> pools(1);
        pools[0].samples = {Sample{10, 20480}, Sample{11, 10240}, Sample{12, 5120}};
        greedy_fill(list, pools);
        CHECK(list.packs[0].total == 128000);
        CHECK(list.packs[0].samples.size() == 3);
        CHECK(pools[0].samples.size() == 1 && pools[0].samples[0].id == 11);
    }
    {
        PackList list;  // nearest pool first, :145-159
        list.capacity = 100;
        list.packs.push_back(make_pack({60}, 100));
        std::vector<SampleSet> pools(2);
        pools[0].samples = {Sample{1, 10}};
        pools[1].samples = {Sample{2, 30}};
        greedy_fill(list, pools);
        CHECK(pools[0].samples.empty() && pools[1].samples.empty());
        CHECK(list.packs[0].total == 100);
    }
    {
        PackList list;  // attention order, :161-178
        list.capacity = 4;
        list.packs = {make_pack({2}, 4), make_pack({1, 1, 2}, 4), make_pack({2, 2}, 4), make_pack({3, 1}, 4)};
        const auto its = balance_batching(list, 2, 0, false);
        CHECK(its.size() == 2);
        CHECK(its[0].devices[0].attention == 10 && its[0].devices[1].attention == 8);
        CHECK(its[1].devices[0].attention == 6 && its[1].devices[1].attention == 4);
        CHECK(std::abs(abr(its[0].devices) - 0.1) < 1e-12);
        CHECK(std::abs(abr(its[1].devices) - 1.0 / 6.0) < 1e-12);
    }
    {
        PackList list;  // spill tail, :201-223
        list.capacity = 100;
        list.packs = {make_pack({50, 30}, 100), make_pack({40, 40}, 100), make_pack({60, 20}, 100)};
        const auto its = balance_batching(list, 2, 0, false);
        CHECK(its.size() == 2);
        CHECK(its.back().devices[0].tokens > 0 && its.back().devices[1].tokens > 0);
        size_t n = 0;
        for (const auto& it : its)
            for (const auto& d : it.devices)
                for (const auto& p : d.packs) {
                    n += p.samples.size();
                    CHECK(p.total <= 100);
                }
        CHECK(n == 6);
    }
    {
        // build_plan conserves samples and is deterministic, :246-267
        const auto corpus = hybrid(600, 0.03, 16384, 131072, 5);
        PlanOptions o;
        o.device_count = 4;
        o.seed = 99;
        const auto plan = build_plan(corpus, two_level(), o);
        std::multiset<std::pair<SampleId, Tokens>> a, b;
        for (const auto& s : plan.all_samples()) a.insert({s.id, s.length});
        for (const auto& s : corpus.samples) b.insert({s.id, s.length});
        CHECK(a == b);
        for (const auto& it : plan.iterations) {
            CHECK(it.devices.size() == 4);
            for (const auto& d : it.devices)
                for (const auto& p : d.packs) CHECK(p.total <= plan.group_of(it).length);
        }
        const auto again = build_plan(corpus, two_level(), o);
        CHECK(again.all_samples() == plan.all_samples());
        // cr equals the long-group token fraction, :269-290
        double lt = 0, tot = 0;
        for (const auto& it : plan.iterations)
            for (const auto& d : it.devices) {
                tot += static_cast<double>(d.tokens);
                if (plan.group_of(it).config.sp > 1) lt += static_cast<double>(d.tokens);
            }
        CHECK(std::abs(report(plan).cr - lt / tot) <= 1e-12);
    }
    {
        // short-only corpus uses group 0, cr 0, :292-304
        const auto corpus = hybrid(300, 0.0, 16384, 131072, 3);
        PlanOptions o;
        o.device_count = 2;
        o.seed = 1;
        const auto plan = build_plan(corpus, two_level(), o);
        for (const auto& it : plan.iterations) CHECK(it.group_index == 0);
        CHECK(report(plan).cr == 0.0);
    }
    {
        // HBP per-iteration ABR is tiny (mean check), :306-327
        const auto corpus = hybrid(100000, 0.02, 16384, 131072, 8);
        PlanOptions o;
        o.device_count = 4;
        o.seed = 13;
        const auto rep = report(build_plan(corpus, two_level(), o));
        CHECK(rep.abr <= 0.01);
    }
    // ---- cost model (test_costmodel.cpp) ----
    {
        AnalyticProfiler prof(HardwareProfile::defaults());
        CHECK(prof.profile_memory(32768, RuntimeConfig{1, 32}) < 0);  // :63-72
        CHECK(prof.profile_memory(32768, RuntimeConfig{2, 32}) >= 0);
        CHECK(prof.profile_memory(131072, RuntimeConfig{8, 32}) >= 0);
        CHECK(prof.profile_memory(131072, RuntimeConfig{4, 32}) < 0);
        std::istringstream csv(
            "length,sp,ckpt,memory_bytes,iter_seconds\n32768,2,28,82678120448,4.45\n32768,4,23,83751862272,4.35\n"
            "32768,8,8,83751862272,4.12\n65536,2,32,oom,0\n65536,4,28,83751862272,6.3\n65536,8,24,84825604096,6.2\n"
            "131072,4,32,oom,0\n131072,8,29,83751862272,10.2\n131072,16,23,84825604096,10.5\n");
        const auto table = TableProfiler::from_csv(csv, "sweep");
        CHECK(table.profile_time(32768, RuntimeConfig{8, 8}) == 4.12);  // :157-166
        CHECK(table.derive_ckpt(65536, 4) == 28);
        CHECK(table.profile_memory(65536, RuntimeConfig{2, 32}) < 0);
        EXPECT_THROW(InfeasibleError, table.profile_time(9999, RuntimeConfig{2, 0}), "no profile row");
        const int sps[] = {2, 4, 8, 16};
        const auto c = find_best_sp_ckpt(table, 32768, sps);  // :168-178
        CHECK(c.config.sp == 8 && c.config.ckpt == 8 && c.seconds == 4.12);
        CHECK(find_best_sp_ckpt(table, 131072, sps).config.sp == 8);
        std::istringstream oomcsv("65536,2,32,oom,0\n65536,4,32,oom,0\n");
        const auto oom = TableProfiler::from_csv(oomcsv, "oom");
        const int sp24[] = {2, 4};
        EXPECT_THROW(InfeasibleError, find_best_sp_ckpt(oom, 65536, sp24), "sp=4");  // :215-221
        CHECK(std::abs(profiling_overhead(3, 3, 3, 5, 1.0) - 60.0) < 1e-12);     // :223-231
        HardwareProfile small = HardwareProfile::defaults();
        small.device_memory = 30LL << 30;
        std::vector<Pack> one = {make_pack({32768}, 32768)};
        EXPECT_THROW(InfeasibleError, iter_time(one, RuntimeConfig{1, 0}, small), "available");  // :112-118
    }
    {
        // user-defined profiler keeps working (host path), :130-149
        struct Fake final : Profiler {
            double profile_time(Tokens, RuntimeConfig) const override { return 1.0; }
            std::int64_t profile_memory(Tokens, RuntimeConfig c) const override {
                if (c.ckpt == 16) return static_cast<std::int64_t>(2e9);
                if (c.ckpt == 32) return static_cast<std::int64_t>(10e9);
                return static_cast<std::int64_t>(2e9 + 0.5e9 * (c.ckpt - 16));
            }
            int derive_ckpt(Tokens l, int sp) const override { return greedy_profile_ckpt(*this, l, sp, 16, 32); }
        } fake;
        CHECK(greedy_profile_ckpt(fake, 1024, 1, 16, 32) == 12);
    }
    // ---- auto-selection (test_autoselect.cpp) ----
    {
        std::istringstream csv(
            "length,sp,ckpt,memory_bytes,iter_seconds\n4096,1,8,81604378624,1.5\n8192,2,8,81604378624,2.0\n"
            "16384,4,8,81604378624,9.0\n131072,8,29,84825604096,30.0\n");
        const auto table = TableProfiler::from_csv(csv, "mem");
        const std::vector<Tokens> lengths = {8192, 131072};
        const std::vector<int> sps = {1, 2, 4, 8, 16};
        const auto g = select_groups(lengths, table, sps);  // :62-83
        CHECK(g.groups.size() == 4);
        if (g.groups.size() == 4) {
            CHECK(g.groups[0].length == 4096 && g.groups[0].config.sp == 1);
            CHECK(g.groups[2].length == 16384 && g.groups[2].config.sp == 4);
            CHECK(g.groups[3].length == 131072 && g.groups[3].config.sp == 8);
        }
        AnalyticProfiler prof(HardwareProfile::defaults());
        const std::vector<Tokens> cands = {8192, 16384, 32768, 65536, 131072};
        const auto a = select_groups(cands, prof, sps);  // :85-96
        CHECK(a.groups.front().config.sp == 1 && a.groups.back().length == a.l_max);
        const std::vector<Tokens> bad = {16384, 8192};
        EXPECT_THROW(ValidationError, select_groups(bad, prof, sps), "strictly ascending");
        const std::vector<int> badsp = {1, 3};
        EXPECT_THROW(ValidationError, select_groups(cands, prof, badsp), "powers of two");
    }
    // ---- simulate (test_sim.cpp) ----
    {
        const auto corpus = hybrid(2000, 0.03, 16384, 131072, 11);
        PlanOptions o;
        o.device_count = 4;
        HierarchicalGroups g = two_level();
        g.groups[0].config.ckpt = 27;
        g.groups[1].config.ckpt = 27;
        const auto plan = build_plan(corpus, g, o);
        const auto r = simulate(plan, HardwareProfile::defaults(), "hbp");
        double sum = 0;
        for (const auto& it : r.iterations) {
            sum += it.seconds;
            for (const auto& d : it.devices)  // idle closed form
                CHECK(std::abs(d.idle_seconds - (it.seconds - d.compute_seconds - d.comm_seconds)) < 1e-12);
        }
        CHECK(std::abs(sum - r.total_seconds) <= 1e-9 * r.total_seconds);
        CHECK(r.corpus == fingerprint(corpus.samples));
        HardwareProfile tiny = HardwareProfile::defaults();
        tiny.device_memory = 25LL << 30;
        EXPECT_THROW(InfeasibleError, simulate(plan, tiny), "iteration 0");  // test_sim.cpp:85-90
    }
    // ---- synthetic generator ----
    {
        const auto spec = parse_synth_spec(
            "count=1000,long_fraction=0.02,short=lognormal:7.2:0.7,long=uniform:16385:131072,max=131072", 7);
        const auto s = synth_lengths(spec);
        CHECK(s.samples.size() == 1000);
        Rng rng(derive_seed(7, "synth-short"));
        const Tokens first = std::max<Tokens>(1, std::min<Tokens>(131072, std::llround(std::exp(7.2 + 0.7 * rng.normal()))));
        CHECK(s.samples[0].length == first);
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail;
}
