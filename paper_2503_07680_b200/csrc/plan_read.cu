// plan_read.cu — the plan manifest reader on the GPU.
//
// Reference: plan_from_json (src/io.cpp:112-160): nlohmann parse, version
// check, groups (validated), device_count, seed, then per iteration its
// group (range-checked), phase, and per device its packs of [id, length]
// samples, each pack checked against its capacity.
//
// The manifests write_plan produces are canonical (nlohmann dump(2): sorted
// keys, two-space indent, one value per line), so a line's indentation says
// what it is: 4 spaces "{" an iteration, 8 "[" a device, 10 "{" a pack,
// 12 "capacity", 16 a sample id ("N,") or length ("N"), 6 "group" / "phase".
// One thread per line classifies it and reads its number; two scans over the
// lines count iterations / devices / packs / samples before every line and
// scatter the values into the plan's CSR arrays. Exactness: the body is
// re-serialised on the device by the writer (io.cu) and compared byte for
// byte with the input, the small header and footer on the host. A manifest
// that is not in that layout is either not JSON (the error is nlohmann's own
// message, as in the reference) or valid JSON in another layout, which this
// reader refuses with a validation error rather than guess.
#include <cstring>
#include <string>

#include "../../include/hbp_b200.h"
#include "engine.cuh"
#include "pipeline.cuh"
#include "scan.cuh"

namespace hbp_b200 {
namespace {

enum PlanLine : unsigned char { kLOther = 0, kLIter, kLDev, kLPack, kLCap, kLId, kLLen, kLGroup, kLPhase };

__device__ __forceinline__ bool lit(const unsigned char* t, u64 p, u64 e, const char* s, u64& q) {
    u64 k = 0;
    for (; s[k]; ++k)
        if (p + k >= e || t[p + k] != static_cast<unsigned char>(s[k])) return false;
    q = p + k;
    return true;
}

__device__ __forceinline__ i64 num(const unsigned char* t, u64 p, u64 e, u64& q) {
    const bool neg = p < e && t[p] == '-';
    if (neg) ++p;
    u64 v = 0;
    while (p < e && t[p] >= '0' && t[p] <= '9') v = v * 10 + (t[p++] - '0');
    q = p;
    return neg ? static_cast<i64>(0ull - v) : static_cast<i64>(v);
}

__global__ void k_plan_lines(const unsigned char* __restrict__ t, u64 bytes, const u64* __restrict__ starts, u64 nl,
                             u64 lines, unsigned char* __restrict__ kind, i64* __restrict__ val) {
    for (u64 L = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; L < lines;
         L += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u64 a = starts[L];
        const u64 e = L < nl ? starts[L + 1] - 1 : bytes;
        u64 p = a;
        while (p < e && t[p] == ' ') ++p;
        const u64 ind = p - a;
        unsigned char k = kLOther;
        i64 v = 0;
        u64 q = p;
        if (p < e) {
            const unsigned char c = t[p];
            if (ind == 4 && c == '{') k = kLIter;
            else if (ind == 8 && c == '[') k = kLDev;
            else if (ind == 10 && c == '{') k = kLPack;
            else if (ind == 12 && lit(t, p, e, "\"capacity\": ", q)) k = kLCap, v = num(t, q, e, q);
            else if (ind == 16 && (c == '-' || (c >= '0' && c <= '9'))) {
                v = num(t, p, e, q);
                k = (q < e && t[q] == ',') ? kLId : kLLen;
            } else if (ind == 6 && lit(t, p, e, "\"group\": ", q)) k = kLGroup, v = num(t, q, e, q);
            else if (ind == 6 && lit(t, p, e, "\"phase\": ", q)) k = kLPhase, v = lit(t, q, e, "\"warmup\"", q) ? 1 : 0;
        }
        kind[L] = k;
        val[L] = v;
    }
}

struct PlanOut {
    int32_t* iter_group;
    int8_t* iter_phase;
    int64_t* iter_dev_offsets;
    int32_t* dev_iter;
    int64_t* dev_pack_offsets;
    int64_t* pack_capacity;
    int32_t* pack_iter;
    int64_t* pack_member_offsets;
    int64_t* ids;
    int64_t* lens;
};

__global__ void k_plan_dev_index(const int32_t* __restrict__ dev_iter, const int64_t* __restrict__ iter_dev_offsets,
                                 u64 D, int32_t* __restrict__ dev_index) {
    for (u64 d = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; d < D;
         d += static_cast<u64>(gridDim.x) * blockDim.x)
        dev_index[d] = static_cast<int32_t>(static_cast<i64>(d) - iter_dev_offsets[dev_iter[d]]);
}

// pack totals, Σ L², member index; first semantic error in the reference's
// order: iteration i's group range (key 2i) before its packs (key 2i + 1)
__global__ void k_plan_packs(const int64_t* __restrict__ moff, const int64_t* __restrict__ lens,
                             const int64_t* __restrict__ cap, const int32_t* __restrict__ pack_iter, u64 P,
                             int64_t* __restrict__ total, int64_t* __restrict__ att,
                             unsigned long long* __restrict__ err) {
    for (u64 p = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; p < P;
         p += static_cast<u64>(gridDim.x) * blockDim.x) {
        int64_t t = 0, a = 0;
        for (int64_t m = moff[p]; m < moff[p + 1]; ++m) {
            t += lens[m];
            a += lens[m] * lens[m];
        }
        total[p] = t;
        att[p] = a;
        if (t > cap[p]) atomicMin(err, 2ull * static_cast<u64>(pack_iter[p]) + 1ull);
    }
}

__global__ void k_plan_groups(const int32_t* __restrict__ g, u64 I, int32_t G, unsigned long long* __restrict__ err) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < I;
         i += static_cast<u64>(gridDim.x) * blockDim.x)
        if (g[i] < 0 || g[i] >= G) atomicMin(err, 2ull * i);
}

__global__ void k_iota_i32(int32_t* __restrict__ v, u64 n) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<u64>(gridDim.x) * blockDim.x)
        v[i] = static_cast<int32_t>(i);
}

__global__ void k_bytes_differ(const unsigned char* __restrict__ a, const char* __restrict__ b, u64 n,
                               unsigned int* __restrict__ differ) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<u64>(gridDim.x) * blockDim.x)
        if (a[i] != static_cast<unsigned char>(b[i])) {
            *differ = 1u;
            return;
        }
}

// ---- host: the small header and footer (canonical layout) -----------------

struct Cursor {
    const char* s;
    size_t n, p = 0;
    bool eat(const char* lit) {
        const size_t k = std::strlen(lit);
        if (p + k > n || std::memcmp(s + p, lit, k) != 0) return false;
        p += k;
        return true;
    }
    bool number(int64_t& v) {
        size_t q = p;
        bool neg = false;
        if (q < n && s[q] == '-') neg = true, ++q;
        const size_t d0 = q;
        uint64_t x = 0;
        while (q < n && s[q] >= '0' && s[q] <= '9' && q - d0 < 20) x = x * 10 + static_cast<uint64_t>(s[q++] - '0');
        if (q == d0) return false;
        p = q;
        v = neg ? static_cast<int64_t>(0ull - x) : static_cast<int64_t>(x);
        return true;
    }
};

// Parses the canonical header; false if the text does not follow it.
bool parse_header(const char* text, u64 bytes, DevicePlan& dp, bool& has_iterations, size_t& head_len) {
    Cursor c{text, static_cast<size_t>(bytes)};
    int64_t v = 0;
    if (!c.eat("{\n  \"device_count\": ") || !c.number(v) || !c.eat(",\n  \"groups\": {\n    \"groups\": ")) return false;
    dp.device_count = static_cast<int32_t>(v);
    if (!c.eat("[]")) {
        if (!c.eat("[")) return false;
        do {
            hbp_group_config g{};
            int64_t ck = 0, len = 0, sp = 0;
            if (!c.eat("\n      {\n        \"ckpt\": ") || !c.number(ck) || !c.eat(",\n        \"length\": ") ||
                !c.number(len) || !c.eat(",\n        \"sp\": ") || !c.number(sp) || !c.eat("\n      }"))
                return false;
            g.length = len;
            g.sp = static_cast<int32_t>(sp);
            g.ckpt = static_cast<int32_t>(ck);
            dp.groups.push_back(g);
        } while (c.eat(","));
        if (!c.eat("\n    ]")) return false;
    }
    if (!c.eat(",\n    \"l_best\": ") || !c.number(dp.l_best) || !c.eat(",\n    \"l_max\": ") || !c.number(dp.l_max) ||
        !c.eat("\n  },\n  \"iterations\": "))
        return false;
    if (c.eat("[]")) has_iterations = false;
    else if (c.eat("[")) has_iterations = true;
    else return false;
    head_len = c.p;
    return true;
}

// Parses the canonical footer from the end; false if it does not follow it.
bool parse_footer(const char* text, u64 bytes, bool has_iterations, DevicePlan& dp, int64_t& version,
                  size_t& foot_len) {
    const std::string t(text + (bytes > 256 ? bytes - 256 : 0), text + bytes);
    const size_t k = t.rfind(",\n  \"seed\": ");
    if (k == std::string::npos) return false;
    size_t start = k;
    if (has_iterations) {
        if (k < 4 || t.compare(k - 4, 4, "\n  ]") != 0) return false;
        start = k - 4;
    }
    Cursor c{t.data(), t.size(), k};
    c.eat(",\n  \"seed\": ");
    size_t q = c.p;
    uint64_t seed = 0;
    const size_t d0 = q;
    while (q < t.size() && t[q] >= '0' && t[q] <= '9' && q - d0 < 20) seed = seed * 10 + static_cast<uint64_t>(t[q++] - '0');
    if (q == d0) return false;
    c.p = q;
    dp.seed = seed;
    if (!c.eat(",\n  \"version\": ") || !c.number(version) || !c.eat("\n}\n") || c.p != t.size()) return false;
    foot_len = t.size() - start;
    return true;
}

// not the canonical layout: the general reader (plan_json.cu) takes it
struct NotCanonical {};
[[noreturn]] void refuse(const char*, u64) { throw NotCanonical{}; }

void plan_from_json_canonical(Ctx& c, const char* text, u64 bytes, DevicePlan& dp, DevBuf<int64_t>& ids,
                              DevBuf<int64_t>& lens) {
    cudaStream_t s = c.stream;
    bool has_it = false;
    size_t head_len = 0, foot_len = 0;
    int64_t version = 0;
    if (!parse_header(text, bytes, dp, has_it, head_len) ||
        !parse_footer(text, bytes, has_it, dp, version, foot_len) || head_len + foot_len > bytes)
        refuse(text, bytes);
    // check_version (io.cpp:44-55), then the groups (io.cpp:29-42)
    if (version != 1) fail_validation("plan manifest: unsupported version " + std::to_string(static_cast<int>(version)));
    validate_groups(dp.groups, dp.l_max);
    const u64 body = bytes - head_len - foot_len;
    if (!has_it && body != 0) refuse(text, bytes);

    // ---- body: one thread per line -------------------------------------------
    DevBuf<unsigned char> t;
    upload_text(c, text + head_len, body, t);
    DevBuf<u64> starts;
    const u64 nl = text_line_starts(c, t.p, body, starts);
    const u64 lines = nl + ((body > 0 && text[head_len + body - 1] != '\n') ? 1 : 0);
    DevBuf<unsigned char> kind(lines + 1, s);
    DevBuf<i64> val(lines + 1, s);
    if (lines) LAUNCH(k_plan_lines, grid_for(lines, 256), 256, 0, s, t.p, body, starts.p, nl, lines, kind.p, val.p);
    // counts before every line: (iterations << 31 | devices), (packs << 31 | samples)
    DevBuf<u64> pa(lines + 1, s), tot(2, s);
    const i64 NL = static_cast<i64>(lines);
    {
        const unsigned char* kp = kind.p;
        u64* pp = pa.p;
        scan_exclusive<u64>(
            NL + 1,
            [=] __device__(i64 i) {
                if (i >= NL) return 0ull;
                return kp[i] == kLIter ? (1ull << 31) : kp[i] == kLDev ? 1ull : 0ull;
            },
            [=] __device__(i64 i, u64 v) { pp[i] = v; }, s, c.scan, "scan.read1");
    }
    // totals for the allocation
    DevBuf<u64> tb(1, s);
    {
        const unsigned char* kp = kind.p;
        u64* tp = tb.p;
        scan_exclusive<u64>(
            NL + 1,
            [=] __device__(i64 i) {
                if (i >= NL) return 0ull;
                return kp[i] == kLPack ? (1ull << 31) : kp[i] == kLId ? 1ull : 0ull;
            },
            [=] __device__(i64 i, u64 v) {
                if (i == NL) *tp = v;
            },
            s, c.scan, "scan.read2");
    }
    const u64 ca = read_vector(c, pa.p + lines, 1)[0];
    const u64 cb = read_vector(c, tb.p, 1)[0];
    const u64 I = ca >> 31, D = ca & 0x7fffffffull, P = cb >> 31, M = cb & 0x7fffffffull;
    if (has_it && I == 0) refuse(text, bytes);
    dp.n_iterations = static_cast<int64_t>(I);
    dp.n_devices = static_cast<int64_t>(D);
    dp.n_packs = static_cast<int64_t>(P);
    dp.n_members = static_cast<int64_t>(M);
    dp.iter_group.alloc(I + 1, s);
    dp.iter_phase.alloc(I + 1, s);
    dp.iter_dev_offsets.alloc(I + 1, s);
    dp.dev_index.alloc(D + 1, s);
    dp.dev_pack_offsets.alloc(D + 1, s);
    dp.pack_capacity.alloc(P + 1, s);
    dp.pack_total.alloc(P + 1, s);
    dp.pack_attention.alloc(P + 1, s);
    dp.pack_member_offsets.alloc(P + 1, s);
    dp.member_index.alloc(M + 1, s);
    ids.alloc(M + 1, s);
    lens.alloc(M + 1, s);
    DevBuf<int32_t> dev_iter(D + 1, s), pack_iter(P + 1, s);
    CUDA_CHECK(cudaMemsetAsync(dp.iter_group.p, 0, sizeof(int32_t) * (I + 1), s));
    CUDA_CHECK(cudaMemsetAsync(dp.iter_phase.p, 0, I + 1, s));
    CUDA_CHECK(cudaMemsetAsync(dp.pack_capacity.p, 0, sizeof(int64_t) * (P + 1), s));
    CUDA_CHECK(cudaMemsetAsync(lens.p, 0, sizeof(int64_t) * (M + 1), s));
    {
        PlanOut o{dp.iter_group.p, dp.iter_phase.p, dp.iter_dev_offsets.p, dev_iter.p, dp.dev_pack_offsets.p,
                  dp.pack_capacity.p, pack_iter.p, dp.pack_member_offsets.p, ids.p, lens.p};
        const unsigned char* kp = kind.p;
        const i64* vp = val.p;
        const u64* pp = pa.p;
        scan_exclusive<u64>(
            NL + 1,
            [=] __device__(i64 i) {
                if (i >= NL) return 0ull;
                return kp[i] == kLPack ? (1ull << 31) : kp[i] == kLId ? 1ull : 0ull;
            },
            [=] __device__(i64 i, u64 v) {
                if (i >= NL) {
                    o.iter_dev_offsets[pp[i] >> 31] = static_cast<int64_t>(pp[i] & 0x7fffffffull);
                    o.dev_pack_offsets[pp[i] & 0x7fffffffull] = static_cast<int64_t>(v >> 31);
                    o.pack_member_offsets[v >> 31] = static_cast<int64_t>(v & 0x7fffffffull);
                    return;
                }
                const u64 it = pp[i] >> 31, dv = pp[i] & 0x7fffffffull, pk = v >> 31, sm = v & 0x7fffffffull;
                switch (kp[i]) {
                    case kLIter: o.iter_dev_offsets[it] = static_cast<int64_t>(dv); break;
                    case kLDev:
                        o.dev_pack_offsets[dv] = static_cast<int64_t>(pk);
                        o.dev_iter[dv] = static_cast<int32_t>(it - 1);
                        break;
                    case kLPack:
                        o.pack_member_offsets[pk] = static_cast<int64_t>(sm);
                        o.pack_iter[pk] = static_cast<int32_t>(it - 1);
                        break;
                    case kLCap: if (pk) o.pack_capacity[pk - 1] = vp[i]; break;
                    case kLId: o.ids[sm] = vp[i]; break;
                    case kLLen: if (sm) o.lens[sm - 1] = vp[i]; break;
                    case kLGroup: if (it) o.iter_group[it - 1] = static_cast<int32_t>(vp[i]); break;
                    case kLPhase: if (it) o.iter_phase[it - 1] = static_cast<int8_t>(vp[i]); break;
                    default: break;
                }
            },
            s, c.scan, "scan.read3");
    }
    if (D) LAUNCH(k_plan_dev_index, grid_for(D, 256), 256, 0, s, dev_iter.p, dp.iter_dev_offsets.p, D, dp.dev_index.p);
    if (M) LAUNCH(k_iota_i32, grid_for(M, 256), 256, 0, s, dp.member_index.p, M);
    DevBuf<unsigned long long> err(1, s);
    CUDA_CHECK(cudaMemsetAsync(err.p, 0xff, sizeof(unsigned long long), s));
    if (P)
        LAUNCH(k_plan_packs, grid_for(P, 256), 256, 0, s, dp.pack_member_offsets.p, lens.p, dp.pack_capacity.p,
               pack_iter.p, P, dp.pack_total.p, dp.pack_attention.p, err.p);
    if (I)
        LAUNCH(k_plan_groups, grid_for(I, 256), 256, 0, s, dp.iter_group.p, I, static_cast<int32_t>(dp.groups.size()),
               err.p);

    // ---- exactness: re-serialise and compare ---------------------------------
    if (header_text(dp).size() != head_len || footer_text(dp).size() != foot_len) refuse(text, bytes);
    DevBuf<char> again;
    const u64 nb = plan_json_body(c, dp, ids.p, lens.p, &again);
    if (nb != body) refuse(text, bytes);
    DevBuf<unsigned int> differ(1, s);
    differ.zero();
    if (body)
        LAUNCH_B("read.compare", 2.0 * static_cast<double>(body), k_bytes_differ, grid_for(body, 256, 148u * 16u), 256,
                 0, s, t.p, again.p, body, differ.p);
    if (read_vector(c, differ.p, 1)[0]) refuse(text, bytes);

    // ---- the reference's semantic errors, first in its order ---------------
    const unsigned long long e = read_vector(c, err.p, 1)[0];
    if (e != ~0ull) {
        if ((e & 1ull) == 0) fail_validation("plan manifest: iteration group index out of range");
        fail_validation("plan manifest: pack exceeds its capacity");
    }
}

}  // namespace

void plan_from_json_device(Ctx& c, const char* text, u64 bytes, DevicePlan& dp, DevBuf<int64_t>& ids,
                           DevBuf<int64_t>& lens) {
    try {
        plan_from_json_canonical(c, text, bytes, dp, ids, lens);
        return;
    } catch (const NotCanonical&) {
    }
    dp.groups.clear();
    plan_from_json_general(c, text, bytes, dp, ids, lens);
}

}  // namespace hbp_b200
