// io.cpp — façade for the plan manifest (include/hbp/io.hpp): the host Plan
// goes to the device (hbp_plan_upload) and its text is built there
// (hbp_plan_to_json); reading parses on the device (hbp_plan_from_json) and
// rebuilds the owning Plan. File helpers follow src/io.cpp:275-291.
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "engine_ctx.hpp"
#include "plan_handle.hpp"
#include "hbp/io.hpp"
#include "hbp_b200.h"

namespace hbp {

namespace {

struct Handle {
    hbp_plan* p = nullptr;
    ~Handle() { hbp_plan_free(p); }
};

std::string read_text(const std::filesystem::path& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open file: " + path.string());
    std::ostringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

void write_text(const std::filesystem::path& path, const std::string& content) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot write file: " + path.string());
    out << content;
    if (!out) throw IoError("write failed: " + path.string());
}

}  // namespace

namespace detail {

UploadedPlan upload_plan(const Plan& plan) {
    UploadedPlan u;
    std::vector<hbp_group_config> groups;
    for (const auto& g : plan.groups.groups) groups.push_back(hbp_group_config{g.length, g.config.sp, g.config.ckpt});
    std::vector<int32_t> iter_group, dev_index, member_index;
    std::vector<int8_t> phase;
    std::vector<int64_t> iter_dev{0}, dev_pack{0}, cap, tot, att, moff{0};
    for (const auto& it : plan.iterations) {
        iter_group.push_back(it.group_index);
        phase.push_back(it.phase == Phase::Warmup ? 1 : 0);
        for (const auto& d : it.devices) {
            dev_index.push_back(d.device_index);
            for (const auto& p : d.packs) {
                cap.push_back(p.capacity);
                tot.push_back(p.total);
                att.push_back(p.attention);
                for (const auto& s : p.samples) {
                    member_index.push_back(static_cast<int32_t>(u.ids.size()));
                    u.ids.push_back(s.id);
                    u.lens.push_back(s.length);
                }
                moff.push_back(static_cast<int64_t>(u.ids.size()));
            }
            dev_pack.push_back(static_cast<int64_t>(cap.size()));
        }
        iter_dev.push_back(static_cast<int64_t>(dev_index.size()));
    }
    hbp_plan_view v{};
    v.device_count = plan.device_count;
    v.seed = plan.seed;
    v.groups = hbp_groups{groups.data(), static_cast<int32_t>(groups.size()), plan.groups.l_best, plan.groups.l_max};
    v.n_iterations = static_cast<int64_t>(iter_group.size());
    v.n_devices = static_cast<int64_t>(dev_index.size());
    v.n_packs = static_cast<int64_t>(cap.size());
    v.n_members = static_cast<int64_t>(u.ids.size());
    v.iter_group = iter_group.data();
    v.iter_dev_offsets = iter_dev.data();
    v.dev_index = dev_index.data();
    v.dev_pack_offsets = dev_pack.data();
    v.pack_capacity = cap.data();
    v.pack_total = tot.data();
    v.pack_attention = att.data();
    v.pack_member_offsets = moff.data();
    v.member_index = member_index.data();
    v.iter_phase = phase.data();
    check(hbp_plan_upload(ctx(), &v, &u.h));
    return u;
}

Plan plan_of_handle(hbp_plan* h, const std::vector<int64_t>& ids, const std::vector<int64_t>& lens) {
    hbp_plan_view v{};
    check(hbp_plan_view_get(ctx(), h, &v));
    Plan plan;
    for (int32_t k = 0; k < v.groups.count; ++k) {
        const auto& g = v.groups.groups[k];
        plan.groups.groups.push_back(GroupConfig{g.length, RuntimeConfig{g.sp, g.ckpt}});
    }
    plan.groups.l_best = v.groups.l_best;
    plan.groups.l_max = v.groups.l_max;
    plan.device_count = v.device_count;
    plan.seed = v.seed;
    plan.iterations.resize(static_cast<size_t>(v.n_iterations));
    for (int64_t i = 0; i < v.n_iterations; ++i) {
        Iteration& it = plan.iterations[static_cast<size_t>(i)];
        it.group_index = v.iter_group[i];
        it.phase = (v.iter_phase && v.iter_phase[i]) ? Phase::Warmup : Phase::Hybrid;
        const bool sp = plan.groups.groups.at(static_cast<size_t>(it.group_index)).config.sp > 1;
        for (int64_t d = v.iter_dev_offsets[i]; d < v.iter_dev_offsets[i + 1]; ++d) {
            std::vector<Pack> packs;
            for (int64_t q = v.dev_pack_offsets[d]; q < v.dev_pack_offsets[d + 1]; ++q) {
                Pack p = Pack::make(v.pack_capacity[q]);
                for (int64_t k = v.pack_member_offsets[q]; k < v.pack_member_offsets[q + 1]; ++k) {
                    const auto m = static_cast<size_t>(v.member_index[k]);
                    p.add(Sample{ids[m], lens[m]});
                }
                packs.push_back(std::move(p));
            }
            it.devices.push_back(DeviceBatch::build(v.dev_index[d], std::move(packs), sp));
        }
    }
    return plan;
}

}  // namespace detail

std::string plan_to_json(const Plan& plan) {
    const detail::UploadedPlan u = detail::upload_plan(plan);
    const hbp_samples smp{u.ids.data(), u.lens.data(), static_cast<int64_t>(u.ids.size()), HBP_MEM_HOST, "plan"};
    int64_t n = 0;
    detail::check(hbp_plan_to_json(detail::ctx(), u.h, &smp, nullptr, 0, &n));
    std::string text(static_cast<size_t>(n), '\0');
    detail::check(hbp_plan_to_json(detail::ctx(), u.h, &smp, text.data(), n, &n));
    return text;
}

Plan plan_from_json(const std::string& text) {
    Handle h;
    int64_t m = 0;
    detail::check(hbp_plan_from_json(detail::ctx(), text.data(), static_cast<int64_t>(text.size()), &h.p, &m));
    std::vector<int64_t> ids(static_cast<size_t>(m) + 1), lens(static_cast<size_t>(m) + 1);
    detail::check(hbp_plan_members(detail::ctx(), h.p, ids.data(), lens.data()));
    return detail::plan_of_handle(h.p, ids, lens);
}

void write_plan(const Plan& plan, const std::filesystem::path& path) { write_text(path, plan_to_json(plan)); }

Plan read_plan(const std::filesystem::path& path) { return plan_from_json(read_text(path)); }

}  // namespace hbp
