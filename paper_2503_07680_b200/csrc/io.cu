// io.cu — the plan manifest writer on the GPU.
//
// Reference: plan_to_json (src/io.cpp:85-110) = nlohmann::json::dump(2) of
// {device_count, groups: {groups: [{ckpt, length, sp}], l_best, l_max},
// iterations: [{devices: [[{capacity, samples: [[id, length], ...]}, ...],
// ...], group, phase}], seed, version: 1} plus a newline. Keys come out
// sorted (nlohmann's object is a std::map), arrays one element per line,
// empty arrays as "[]". Output is byte-identical.
//
// At 10M samples the text is ~0.7 GB (about 67 bytes per sample), so it is
// built where the plan lives: one thread per device slot (an iteration's
// device) measures its text -- its packs and samples, plus the iteration's
// opening when it is the first device and closing when it is the last --
// a scan gives every slot its offset, and the same thread writes it. The
// small header and footer are formatted on the host.
#include <algorithm>
#include <cstring>
#include <string>

#include "../../include/hbp_b200.h"
#include "engine.cuh"
#include "pipeline.cuh"

using namespace hbp_b200;


namespace {

__host__ __device__ __forceinline__ u32 digits_u64(u64 v) {
    u32 d = 1;
    u64 p = 10;
    while (d < 20 && v >= p) {  // comparisons, no divisions
        ++d;
        p *= 10;
    }
    return d;
}
__host__ __device__ __forceinline__ u32 digits_i64(int64_t v) {
    return v < 0 ? 1 + digits_u64(0ull - static_cast<u64>(v)) : digits_u64(static_cast<u64>(v));
}

// Text pieces (indentation of dump(2) at each depth).
#define J_ITER_OPEN "\n    {\n      \"devices\": ["
#define J_DEV_OPEN "\n        ["
#define J_DEV_EMPTY "\n        []"
#define J_DEV_CLOSE "\n        ]"
#define J_PACK_OPEN "\n          {\n            \"capacity\": "
#define J_PACK_SAMPLES ",\n            \"samples\": "
#define J_PACK_CLOSE "\n            ]\n          }"
#define J_PACK_CLOSE_EMPTY "[]\n          }"
#define J_SAMPLE_OPEN "\n              [\n                "
#define J_SAMPLE_MID ",\n                "
#define J_SAMPLE_CLOSE "\n              ]"
#define J_ITER_CLOSE "\n      ],\n      \"group\": "
#define J_ITER_PHASE ",\n      \"phase\": \"hybrid\"\n    }"
#define J_ITER_PHASE_W ",\n      \"phase\": \"warmup\"\n    }"
#define JLEN(s) (sizeof(s) - 1)

struct JsonArgs {
    const int32_t* iter_group;
    const int64_t* iter_dev_offsets;
    const int64_t* dev_pack_offsets;
    const int64_t* pack_capacity;
    const int64_t* pack_member_offsets;
    const int32_t* member_index;
    const int64_t* ids;  // null: ids are the corpus indices
    const int64_t* lengths;
    const int8_t* phase;  // null: all hybrid
    int64_t n_iterations, n_devices;
};

// iteration of device slot g: last i with iter_dev_offsets[i] <= g
__device__ __forceinline__ int64_t iter_of(const JsonArgs& a, int64_t g) {
    int64_t lo = 0, hi = a.n_iterations;
    while (lo + 1 < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a.iter_dev_offsets[mid] <= g) lo = mid;
        else hi = mid;
    }
    return lo;
}

struct Writer {
    char* p;
    __device__ __forceinline__ void lit(const char* s, u32 n) {
        for (u32 k = 0; k < n; ++k) p[k] = s[k];
        p += n;
    }
    __device__ __forceinline__ void ch(char c) { *p++ = c; }
    __device__ __forceinline__ void num(int64_t v) {
        u64 u = v < 0 ? 0ull - static_cast<u64>(v) : static_cast<u64>(v);
        if (v < 0) *p++ = '-';
        const u32 d = digits_u64(u);
        u32 k = d;
        while (u > 0xffffffffull) {  // rare: 64-bit digits
            p[--k] = static_cast<char>('0' + u % 10);
            u /= 10;
        }
        u32 x = static_cast<u32>(u);  // 32-bit divisions by 10 are a multiply-shift
        while (k > 0) {
            p[--k] = static_cast<char>('0' + x % 10u);
            x /= 10u;
        }
        p += d;
    }
};

// Text of device slot g; WRITE false: only its length.
template <bool WRITE>
__device__ u64 slot_text(const JsonArgs& a, int64_t g, char* out) {
    const int64_t i = iter_of(a, g);
    const int64_t d = g - a.iter_dev_offsets[i];
    const bool first = d == 0, last = g + 1 == a.iter_dev_offsets[i + 1];
    Writer w{out};
    u64 n = 0;
    if (first) {
        if (i > 0) {
            n += 1;
            if (WRITE) w.ch(',');
        }
        n += JLEN(J_ITER_OPEN);
        if (WRITE) w.lit(J_ITER_OPEN, JLEN(J_ITER_OPEN));
    } else {
        n += 1;
        if (WRITE) w.ch(',');
    }
    const int64_t p0 = a.dev_pack_offsets[g], p1 = a.dev_pack_offsets[g + 1];
    if (p0 == p1) {
        n += JLEN(J_DEV_EMPTY);
        if (WRITE) w.lit(J_DEV_EMPTY, JLEN(J_DEV_EMPTY));
    } else {
        n += JLEN(J_DEV_OPEN);
        if (WRITE) w.lit(J_DEV_OPEN, JLEN(J_DEV_OPEN));
        for (int64_t q = p0; q < p1; ++q) {
            if (q > p0) {
                n += 1;
                if (WRITE) w.ch(',');
            }
            const int64_t cap = a.pack_capacity[q];
            n += JLEN(J_PACK_OPEN) + digits_i64(cap) + JLEN(J_PACK_SAMPLES);
            if (WRITE) {
                w.lit(J_PACK_OPEN, JLEN(J_PACK_OPEN));
                w.num(cap);
                w.lit(J_PACK_SAMPLES, JLEN(J_PACK_SAMPLES));
            }
            const int64_t m0 = a.pack_member_offsets[q], m1 = a.pack_member_offsets[q + 1];
            if (m0 == m1) {
                n += JLEN(J_PACK_CLOSE_EMPTY);
                if (WRITE) w.lit(J_PACK_CLOSE_EMPTY, JLEN(J_PACK_CLOSE_EMPTY));
                continue;
            }
            n += 1;
            if (WRITE) w.ch('[');
            for (int64_t m = m0; m < m1; ++m) {
                const int64_t ix = a.member_index[m];
                const int64_t id = a.ids ? a.ids[ix] : ix;
                const int64_t len = a.lengths[ix];
                n += (m > m0 ? 1 : 0) + JLEN(J_SAMPLE_OPEN) + digits_i64(id) + JLEN(J_SAMPLE_MID) + digits_i64(len) +
                     JLEN(J_SAMPLE_CLOSE);
                if (WRITE) {
                    if (m > m0) w.ch(',');
                    w.lit(J_SAMPLE_OPEN, JLEN(J_SAMPLE_OPEN));
                    w.num(id);
                    w.lit(J_SAMPLE_MID, JLEN(J_SAMPLE_MID));
                    w.num(len);
                    w.lit(J_SAMPLE_CLOSE, JLEN(J_SAMPLE_CLOSE));
                }
            }
            n += JLEN(J_PACK_CLOSE);
            if (WRITE) w.lit(J_PACK_CLOSE, JLEN(J_PACK_CLOSE));
        }
        n += JLEN(J_DEV_CLOSE);
        if (WRITE) w.lit(J_DEV_CLOSE, JLEN(J_DEV_CLOSE));
    }
    if (last) {
        const int64_t grp = a.iter_group[i];
        const bool warm = a.phase && a.phase[i];
        n += JLEN(J_ITER_CLOSE) + digits_i64(grp) + (warm ? JLEN(J_ITER_PHASE_W) : JLEN(J_ITER_PHASE));
        if (WRITE) {
            w.lit(J_ITER_CLOSE, JLEN(J_ITER_CLOSE));
            w.num(grp);
            if (warm) w.lit(J_ITER_PHASE_W, JLEN(J_ITER_PHASE_W));
            else w.lit(J_ITER_PHASE, JLEN(J_ITER_PHASE));
        }
    }
    return n;
}

__global__ void k_json_len(JsonArgs a, u64* len) {
    for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < a.n_devices;
         g += static_cast<int64_t>(gridDim.x) * blockDim.x)
        len[g] = slot_text<false>(a, g, nullptr);
}

__global__ void k_json_write(JsonArgs a, const u64* off, char* out) {
    for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < a.n_devices;
         g += static_cast<int64_t>(gridDim.x) * blockDim.x)
        slot_text<true>(a, g, out + off[g]);
}

}  // namespace

namespace hbp_b200 {

std::string header_text(const DevicePlan& dp) {
    std::string h = "{\n  \"device_count\": " + std::to_string(dp.device_count) + ",\n  \"groups\": {\n    \"groups\": ";
    if (dp.groups.empty()) {
        h += "[]";
    } else {
        h += "[";
        for (size_t k = 0; k < dp.groups.size(); ++k) {
            const auto& g = dp.groups[k];
            h += (k ? ",\n" : "\n");
            h += "      {\n        \"ckpt\": " + std::to_string(g.ckpt) + ",\n        \"length\": " +
                 std::to_string(g.length) + ",\n        \"sp\": " + std::to_string(g.sp) + "\n      }";
        }
        h += "\n    ]";
    }
    h += ",\n    \"l_best\": " + std::to_string(dp.l_best) + ",\n    \"l_max\": " + std::to_string(dp.l_max) +
         "\n  },\n  \"iterations\": ";
    h += dp.n_iterations ? "[" : "[]";
    return h;
}

std::string footer_text(const DevicePlan& dp) {
    return std::string(dp.n_iterations ? "\n  ]" : "") + ",\n  \"seed\": " + std::to_string(dp.seed) +
           ",\n  \"version\": 1\n}\n";
}

// The manifest body (everything between header_text and footer_text) of a
// device plan, built on the device into `text` (null: length only).
// Returns its length.
u64 plan_json_body(Ctx& c, const DevicePlan& dp, const int64_t* ids, const int64_t* lens, DevBuf<char>* text) {
    cudaStream_t s = c.stream;
    JsonArgs a{dp.iter_group.p, dp.iter_dev_offsets.p, dp.dev_pack_offsets.p, dp.pack_capacity.p,
               dp.pack_member_offsets.p, dp.member_index.p, ids, lens, dp.iter_phase.p, dp.n_iterations, dp.n_devices};
    const u64 G = static_cast<u64>(dp.n_devices);
    if (G == 0) return 0;
    DevBuf<u64> len(G + 1, s), off(G + 1, s);
    LAUNCH(k_json_len, grid_for(G, 128, 148u * 32u), 128, 0, s, a, len.p);
    const u64* lp = len.p;
    u64* op = off.p;
    const i64 GG = static_cast<i64>(G);
    scan_exclusive<u64>(
        GG + 1, [=] __device__(i64 i) { return i < GG ? lp[i] : 0ull; }, [=] __device__(i64 i, u64 v) { op[i] = v; },
        s, c.scan, "scan.io1");
    const u64 body = read_scalar(c, off.p + G);
    if (text == nullptr) return body;  // length only
    text->alloc(body, s);
    if (body)
        LAUNCH_B("io.json", static_cast<double>(body), k_json_write, grid_for(G, 128, 148u * 32u), 128, 0, s, a, off.p,
                 text->p);
    return body;
}

}  // namespace hbp_b200

extern "C" int hbp_plan_to_json(hbp_ctx* ctx, hbp_plan* plan, const hbp_samples* samples, char* out,
                                int64_t capacity, int64_t* out_len) {
    if (ctx == nullptr || plan == nullptr || samples == nullptr || out_len == nullptr) return HBP_ERR_VALIDATION;
    try {
        CtxScope scope(*ctx);
        const DevicePlan& dp = plan->dp;
        if (!dp.member_index.p && dp.n_members > 0)
            throw EngineError(HBP_ERR_VALIDATION, "plan_to_json: the plan's device arrays are gone");
        cudaStream_t s = ctx->stream;
        const std::string head = header_text(dp), foot = footer_text(dp);
        // corpus ids / lengths on the device
        DevBuf<int64_t> dids, dlen;
        const int64_t* ids = samples->ids;
        const int64_t* lens = samples->lengths;
        if (samples->memory == HBP_MEM_HOST && samples->n > 0) {
            dlen.alloc(static_cast<size_t>(samples->n), s);
            CUDA_CHECK(cudaMemcpyAsync(dlen.p, lens, sizeof(int64_t) * samples->n, cudaMemcpyHostToDevice, s));
            lens = dlen.p;
            if (ids) {
                dids.alloc(static_cast<size_t>(samples->n), s);
                CUDA_CHECK(cudaMemcpyAsync(dids.p, ids, sizeof(int64_t) * samples->n, cudaMemcpyHostToDevice, s));
                ids = dids.p;
            }
        }
        DevBuf<char> text;
        const u64 body = plan_json_body(*ctx, dp, ids, lens, out == nullptr ? nullptr : &text);
        const u64 total = head.size() + body + foot.size();
        *out_len = static_cast<int64_t>(total);
        if (out == nullptr) {
            ctx->last_error.clear();
            return HBP_OK;
        }
        if (capacity < static_cast<int64_t>(total))
            throw EngineError(HBP_ERR_VALIDATION, "plan_to_json: output buffer of " + std::to_string(capacity) +
                                                      " bytes, the manifest needs " + std::to_string(total));
        std::memcpy(out, head.data(), head.size());
        if (body) {
            // download through two pinned staging blocks: chunk k + 1 crosses
            // PCIe while chunk k is copied into the caller's (pageable) buffer
            constexpr size_t kChunk = size_t(64) << 20;
            HostBlock stage[2] = {ctx->host_pool.acquire(std::min<size_t>(kChunk, body)),
                                  ctx->host_pool.acquire(std::min<size_t>(kChunk, body))};
            cudaEvent_t done[2];
            CUDA_CHECK(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
            CUDA_CHECK(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
            const size_t nchunks = (body + kChunk - 1) / kChunk;
            auto issue = [&](size_t k) {
                const size_t o = k * kChunk, n = std::min(kChunk, body - o);
                CUDA_CHECK(cudaMemcpyAsync(stage[k & 1].p, text.p + o, n, cudaMemcpyDeviceToHost, s));
                CUDA_CHECK(cudaEventRecord(done[k & 1], s));
            };
            issue(0);
            for (size_t k = 0; k < nchunks; ++k) {
                if (k + 1 < nchunks) issue(k + 1);
                CUDA_CHECK(cudaEventSynchronize(done[k & 1]));
                const size_t o = k * kChunk, n = std::min(kChunk, body - o);
                std::memcpy(out + head.size() + o, stage[k & 1].p, n);  // frees stage[k & 1] for chunk k + 2
            }
            CUDA_CHECK(cudaEventDestroy(done[0]));
            CUDA_CHECK(cudaEventDestroy(done[1]));
            ctx->host_pool.release(stage[0]);
            ctx->host_pool.release(stage[1]);
        }
        CUDA_CHECK(cudaStreamSynchronize(s));
        std::memcpy(out + head.size() + body, foot.data(), foot.size());
        ctx->last_error.clear();
        return HBP_OK;
    } catch (const EngineError& e) {
        ctx->last_error = e.what();
        if (e.code == HBP_ERR_CUDA) cudaGetLastError();
        return e.code;
    } catch (const std::exception& e) {
        ctx->last_error = e.what();
        return HBP_ERR_CUDA;
    }
}
