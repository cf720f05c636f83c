// pipeline.cuh — build_plan / pack orchestration and the device-resident plan.
#pragma once

#include <string>
#include <vector>

#include "stages.cuh"

namespace hbp_b200 {

// Device-resident plan in the flat CSR layout of hbp_plan_view. Host copies
// are made lazily by hbp_plan_view_get.
struct DevicePlan {
    int32_t device_count = 0;
    uint64_t seed = 0;
    std::vector<hbp_group_config> groups;
    int64_t l_best = 0, l_max = 0;
    int64_t n_iterations = 0, n_devices = 0, n_packs = 0, n_members = 0;
    DevBuf<int32_t> iter_group;
    DevBuf<int64_t> iter_dev_offsets;
    DevBuf<int32_t> dev_index;
    DevBuf<int64_t> dev_pack_offsets;
    DevBuf<int64_t> pack_capacity, pack_total, pack_attention, pack_member_offsets;
    DevBuf<int32_t> member_index;
    DevBuf<int8_t> iter_phase;  // 1 = warmup (curriculum_order); empty: every iteration hybrid
    // host mirror, in one pinned block (returned to the context's pool when
    // the plan is freed; freed here if the plan outlives its context)
    bool on_host = false;
    HostBlock host{};
    int32_t *h_iter_group = nullptr, *h_dev_index = nullptr, *h_member_index = nullptr;
    int8_t* h_iter_phase = nullptr;
    int64_t *h_iter_dev_offsets = nullptr, *h_dev_pack_offsets = nullptr, *h_pack_capacity = nullptr,
            *h_pack_total = nullptr, *h_pack_attention = nullptr, *h_pack_member_offsets = nullptr;
    DevicePlan() = default;
    DevicePlan(const DevicePlan&) = delete;
    DevicePlan& operator=(const DevicePlan&) = delete;
    ~DevicePlan() {
        if (host.p) cudaFreeHost(host.p);
    }
    // frees the device arrays (the host mirror stays valid)
    void release_device() {
        iter_group.release();
        iter_dev_offsets.release();
        dev_index.release();
        dev_pack_offsets.release();
        pack_capacity.release();
        pack_total.release();
        pack_attention.release();
        pack_member_offsets.release();
        member_index.release();
        iter_phase.release();
    }
};

// Samples resident on the device after ingest.
struct DeviceCorpus {
    i64 n = 0;
    DevBuf<u32> len32;       // lengths
    DevBuf<u32> key32;       // tie-break key: id rank (general ids) -- empty when ids ascend in input order
    bool ids_ascending = true;
    i64 neg_ids = 0;         // samples with id <= -2 (greedy-fill probe quirk)
    int key_bits = 1;
    std::vector<int64_t> h_ids;      // host copy of ids for error messages (empty -> ids are 0..n-1)
    const int64_t* ids_host = nullptr;
    const int64_t* lengths_host = nullptr;  // caller's lengths when they are host memory
    const int64_t* lengths_dev = nullptr;   // caller's lengths when they are device memory
    u64 first_bad_len = ~0ull;  // first sample with length < 1
    u64 first_huge = ~0ull;     // first sample with length > 2^31-1 (engine limit)
    u64 first_dup = ~0ull;      // first repeated id (input order), general ids only
    int64_t id_of(i64 i) const { return ids_host ? ids_host[i] : static_cast<int64_t>(i); }
    int64_t length_of(Ctx& c, i64 i) const;
};

// Uploads lengths/ids, converts lengths to u32, ranks non-ascending ids and
// records the first offending samples. Throws nothing about the data.
void ingest(Ctx& c, const hbp_samples* in, DeviceCorpus& corpus);
// SampleSet::validate (types.cpp:8-24): "empty corpus", non-positive
// length, duplicate id -- the first offending sample in input order.
void validate_corpus(Ctx& c, const hbp_samples* in, const DeviceCorpus& corpus, const std::string& source);

struct PlanArgs {
    std::vector<hbp_group_config> groups;
    int64_t l_best = 0, l_max = 0;
    hbp_strategy strategy{};
    int32_t device_count = 4;
    bool balance_batching = true;
    bool greedy_fill = true;
    uint64_t seed = 0;
};

// build_plan (balance.cpp:207-258) on a validated corpus.
void build_plan_device(Ctx& c, DeviceCorpus& corpus, const PlanArgs& args, DevicePlan& out);

// pack() of the whole corpus to one capacity (packing.cpp:210-261); output
// is a plan with no iterations.
void pack_device(Ctx& c, DeviceCorpus& corpus, int64_t capacity, const hbp_strategy& st, uint64_t seed,
                 DevicePlan& out);

// group_data (balance.cpp:25-44): per-group offsets and member indices (input order).
void group_data_device(Ctx& c, DeviceCorpus& corpus, const std::vector<hbp_group_config>& groups, int64_t l_max,
                       std::vector<int64_t>& offsets, std::vector<int32_t>& members);

void plan_to_host(Ctx& c, DevicePlan& p);

// greedy_fill over host pack lists (balance.cpp:46-101): returns, per pack,
// the pool samples (flattened pool index) it takes in order, and which pool
// samples remain.
void greedy_fill_device(Ctx& c, i64 n_packs, const int64_t* pack_cap, const int64_t* pack_off, const int64_t* lens,
                        int n_pools, const int64_t* pool_off, const int64_t* pool_ids, const int64_t* pool_lens,
                        std::vector<int64_t>& added_off, std::vector<int64_t>& added, std::vector<uint8_t>& keep);

// balance_batching / random_pack_batching over a host pack list
// (balance.cpp:105-205); no plan shuffle. member_index = member position.
void batching_device(Ctx& c, int64_t capacity, i64 n_packs, const int64_t* pack_cap, const int64_t* pack_off,
                     const int64_t* ids, const int64_t* lens, int32_t N, int32_t gi, bool random, uint64_t seed,
                     DevicePlan& out);

// groups.validate() (autoselect.cpp:18-33)
void validate_groups(const std::vector<hbp_group_config>& g, int64_t l_max);
void validate_strategy(const hbp_strategy& s);

// sorted_batching / random_batching (packing.cpp:265-317): samples in
// (length desc, id asc) order or Rng(derive_seed(seed, "random-batching"))
// order, cut greedily into batches while count * max <= budget -- the cut
// positions are the chain of a monotone next(), found like next-fit's.
struct PaddedBatches {
    u64 n = 0, n_batches = 0;
    DevBuf<u64> order;   // entries (len << 32 | corpus index) in batching order
    DevBuf<u32> bstart;  // first position of each batch
    DevBuf<u32> bidx;    // batch of each position
    DevBuf<u32> bmax;    // longest sample of each batch
};
void padded_batches_device(Ctx& c, const DeviceCorpus& corpus, int64_t budget, bool sorted, uint64_t seed,
                           PaddedBatches& out);
// build_batching_plan (balance.cpp:260-298): device g of iteration i holds
// batch i * N + g as single-sample packs padded to the batch's longest.
void batching_plan_device(Ctx& c, const DeviceCorpus& corpus, const hbp_group_config& group, int32_t device_count,
                          bool sorted, uint64_t seed, DevicePlan& out);

// io.cu: the plan manifest's header / footer text and its body built on the
// device (null text: length only); plan_read.cu: the reader.
std::string header_text(const DevicePlan& dp);
std::string footer_text(const DevicePlan& dp);
u64 plan_json_body(Ctx& c, const DevicePlan& dp, const int64_t* ids, const int64_t* lens, DevBuf<char>* text);
void plan_from_json_device(Ctx& c, const char* text, u64 bytes, DevicePlan& dp, DevBuf<int64_t>& ids,
                           DevBuf<int64_t>& lens);
// plan_json.cu: the reader for any JSON layout (plan_read.cu hands it what
// is not canonical)
void plan_from_json_general(Ctx& c, const char* text, u64 bytes, DevicePlan& dp, DevBuf<int64_t>& ids,
                            DevBuf<int64_t>& lens);
// corpus.cu: text to the device (zero-padded to 16 bytes) and the start of
// every line (starts[0] = 0, then one past each '\n'); returns the '\n' count.
void upload_text(Ctx& c, const char* text, u64 bytes, DevBuf<unsigned char>& t);
u64 text_line_starts(Ctx& c, const unsigned char* t, u64 bytes, DevBuf<u64>& starts);
std::string json_parse_error_text(const std::string& text);

// corpus.cu: load_lengths of a JSONL / CSV / raw-lengths text
// (ingest.cpp:57-160); returns the sample count, ids and lengths (device).
i64 parse_corpus_text(Ctx& c, const char* text, u64 bytes, int format, const std::string& source,
                      DevBuf<int64_t>& lengths, DevBuf<int64_t>& ids);

}  // namespace hbp_b200

// The C-ABI plan handle (include/hbp_b200.h): the device plan, its host view
// once made, and the context that owns it (null once the context is gone).
struct hbp_plan {
    hbp_b200::DevicePlan dp;
    // a plan read from a manifest carries its own samples (member order)
    hbp_b200::DevBuf<int64_t> read_ids, read_lens;
    hbp_plan_view view{};
    hbp_ctx* owner = nullptr;
};
