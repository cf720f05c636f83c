// TEST/BENCH INFRASTRUCTURE ONLY — the reference arm of bench.py.
//
// A stand-alone program over the reference's own public C++ API, compiled
// from /root/reference/proj/src in place (oracle/Makefile, namespace renamed
// hbp -> hbp_ref so nothing can resolve to this repo's engine). It does what
// the reference CLI's `pack` command does (proj/tools/hbp_main.cpp:280-322)
// for one synthetic corpus, and times the hot path:
//
//   synth_lengths(parse_synth_spec(spec, seed))   ingest.cpp:279-373 (not timed)
//   build_plan(samples, groups, options)           balance.cpp:207-258
//   report(plan)                                   metrics.cpp:107-144
//   simulate(plan, profile)                        sim.cpp:9-60
//
// It never loads libhbp_b200.so: the corpus, the plan and the metrics come
// from the reference alone. Prints one JSON line.
//
//   ref_bench --synth "count=...,short=...,long_fraction=...,long=...,max=..."
//             --seed S --groups 16384:1:28,131072:8:28 --l-best 16384
//             --devices 8 --plan-seed 1 [--profile analytic.json]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>

#include "hbp/autoselect.hpp"
#include "hbp/balance.hpp"
#include "hbp/costmodel.hpp"
#include "hbp/errors.hpp"
#include "hbp/ingest.hpp"
#include "hbp/metrics.hpp"
#include "hbp/sim.hpp"

namespace {

double secs_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// FNV-1a over the plan's structure, in plan order: iteration group, then per
// device its packs' capacity and member ids. Lets bench.py show both arms
// built the same plan without shipping it.
struct Fnv {
    unsigned long long h = 1469598103934665603ull;
    void add(long long v) {
        for (int i = 0; i < 8; ++i) {
            h ^= static_cast<unsigned long long>(v >> (8 * i)) & 0xffull;
            h *= 1099511628211ull;
        }
    }
};

}  // namespace

int main(int argc, char** argv) {
    std::string synth, groups_arg, profile_path;
    unsigned long long seed = 0, plan_seed = 0;
    long long l_best = 0;
    int devices = 8;
    for (int i = 1; i + 1 < argc; i += 2) {
        const std::string k = argv[i], v = argv[i + 1];
        if (k == "--synth") synth = v;
        else if (k == "--seed") seed = std::strtoull(v.c_str(), nullptr, 10);
        else if (k == "--groups") groups_arg = v;
        else if (k == "--l-best") l_best = std::strtoll(v.c_str(), nullptr, 10);
        else if (k == "--devices") devices = std::atoi(v.c_str());
        else if (k == "--plan-seed") plan_seed = std::strtoull(v.c_str(), nullptr, 10);
        else if (k == "--profile") profile_path = v;
        else { std::fprintf(stderr, "unknown flag %s\n", k.c_str()); return 2; }
    }
    try {
        auto t0 = std::chrono::steady_clock::now();
        const hbp_ref::SampleSet samples = hbp_ref::synth_lengths(hbp_ref::parse_synth_spec(synth, seed));
        const double synth_s = secs_since(t0);

        hbp_ref::HierarchicalGroups groups;
        std::stringstream gs(groups_arg);
        std::string item;
        while (std::getline(gs, item, ',')) {
            hbp_ref::GroupConfig g;
            long long len = 0;
            int sp = 1, ckpt = 0;
            if (std::sscanf(item.c_str(), "%lld:%d:%d", &len, &sp, &ckpt) != 3) {
                std::fprintf(stderr, "bad group %s\n", item.c_str());
                return 2;
            }
            g.length = len;
            g.config.sp = sp;
            g.config.ckpt = ckpt;
            groups.groups.push_back(g);
        }
        groups.l_best = l_best;
        groups.l_max = groups.groups.back().length;
        const hbp_ref::HardwareProfile profile =
            profile_path.empty() ? hbp_ref::HardwareProfile::defaults()
                                 : hbp_ref::load_analytic_profile_file(profile_path);

        hbp_ref::PlanOptions opt;
        opt.device_count = devices;
        opt.seed = plan_seed;

        t0 = std::chrono::steady_clock::now();
        const hbp_ref::Plan plan = hbp_ref::build_plan(samples, groups, opt);
        const double build_s = secs_since(t0);
        t0 = std::chrono::steady_clock::now();
        const hbp_ref::MetricsReport rep = hbp_ref::report(plan);
        const double report_s = secs_since(t0);
        t0 = std::chrono::steady_clock::now();
        const hbp_ref::SimReport sim = hbp_ref::simulate(plan, profile);
        const double simulate_s = secs_since(t0);

        Fnv f;
        long long packs = 0;
        for (const auto& it : plan.iterations) {
            f.add(it.group_index);
            for (const auto& d : it.devices) {
                f.add(static_cast<long long>(d.packs.size()));
                for (const auto& p : d.packs) {
                    ++packs;
                    f.add(p.capacity);
                    f.add(static_cast<long long>(p.samples.size()));
                    for (const auto& s : p.samples) f.add(s.id);
                }
            }
        }
        std::printf("{\"samples\": %zu, \"synth_s\": %.6f, \"build_s\": %.6f, \"report_s\": %.6f, "
                    "\"simulate_s\": %.6f, \"step_s\": %.6f, \"iterations\": %zu, \"packs\": %lld, "
                    "\"abr\": %.17g, \"cr\": %.17g, \"total_seconds\": %.17g, \"plan_fnv\": \"%016llx\"}\n",
                    samples.size(), synth_s, build_s, report_s, simulate_s, build_s + report_s + simulate_s,
                    plan.iterations.size(), packs, rep.abr, rep.cr, sim.total_seconds, f.h);
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ref_bench: %s\n", e.what());
        return 1;
    }
}
