// corpus.cu — corpus file parsers on the GPU: JSONL, CSV and raw-lengths
// (src/ingest.cpp:57-169, load_jsonl / load_csv / load_raw / load_lengths).
//
// The text is copied to HBM once; everything after that is byte work on the
// device:
//   1. newline count per 16-byte chunk, scanned -> the line number of every
//      chunk's first byte; each '\n' then writes the start of the next line
//      (std::getline semantics: a final line without '\n' is a line, the
//      empty tail after a final '\n' is not);
//   2. one thread per line: blank test (only " \t\r"), the CSV cell (commas
//      before it; getline(ss, cell, ',') + the trailing-comma rule give
//      commas + 1 cells), trim " \t\r", then std::stoll's grammar (leading
//      isspace, sign, base-10 digits, out_of_range on overflow) and the
//      reference's checks in its order: not an integer / trailing garbage /
//      length >= 1. The first failing line wins (atomicMin on the line
//      number), as in the reference's sequential read;
//   3. the kept lines are compacted by a scan into int64 lengths.
// The host only splits the CSV header (one line, split_csv_row's rules) and
// formats the error message from the failing line's bytes; for a JSONL line
// that is not JSON that text is nlohmann's own parse_error message, so the
// host re-parses that one line with it (corpus_host.cpp).
#include <cstring>
#include <string>
#include <vector>

#include "pipeline.cuh"
#include "scan.cuh"

namespace hbp_b200 {

// corpus_host.cpp: nlohmann's parse_error text for one line ("" if it parses)
std::string json_parse_error_text(const std::string& line);

namespace {

constexpr int kChunkBytes = 16;

enum LineStatus : u32 { kOk = 0, kBadInt = 1, kTrailing = 2, kNonPositive = 3, kFewColumns = 4 };

__device__ __forceinline__ u32 nl_in(uint4 v) {
    // bytes equal to '\n' (0x0a) in 16 bytes
    u32 n = 0;
    const u32 w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const u32 x = w[q] ^ 0x0a0a0a0au;
        // zero-byte detector, exact per byte
        const u32 z = ~(((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x | 0x7f7f7f7fu);
        n += __popc(z);
    }
    return n;
}

__global__ void k_line_starts(const unsigned char* __restrict__ t, u64 bytes, const u64* __restrict__ chunk_line,
                              u64* __restrict__ starts) {
    const u64 chunks = (bytes + kChunkBytes - 1) / kChunkBytes;
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < chunks;
         i += static_cast<u64>(gridDim.x) * blockDim.x) {
        const uint4 v = reinterpret_cast<const uint4*>(t)[i];
        if (nl_in(v) == 0) continue;
        u64 L = chunk_line[i];
        const unsigned char* b = reinterpret_cast<const unsigned char*>(&v);
#pragma unroll
        for (int q = 0; q < kChunkBytes; ++q)
            if (b[q] == '\n') starts[++L] = i * kChunkBytes + q + 1;
    }
}

__device__ __forceinline__ bool trim_char(unsigned char ch) { return ch == ' ' || ch == '\t' || ch == '\r'; }
__device__ __forceinline__ bool c_isspace(unsigned char ch) {
    return ch == ' ' || (ch >= '\t' && ch <= '\r');  // \t \n \v \f \r
}

struct Cell {
    u64 a, b;     // trimmed cell [a, b)
    i64 value;
    u32 status;
    bool blank;
};

// One line [a, e): blank test, CSV cell `col` (-1: the whole line), trim,
// std::stoll + the reference's checks (ingest.cpp:17-39).
__device__ Cell parse_line(const unsigned char* __restrict__ t, u64 a, u64 e, int col) {
    Cell r{a, a, 0, kOk, true};
    for (u64 p = a; p < e; ++p)
        if (!trim_char(t[p])) {
            r.blank = false;
            break;
        }
    if (r.blank) return r;
    u64 ca = a, cb = e;
    if (col >= 0) {
        int k = 0;
        u64 p = a;
        for (; p < e && k < col; ++p)
            if (t[p] == ',') ca = p + 1, ++k;
        if (k < col) {
            r.status = kFewColumns;
            return r;
        }
        cb = ca;
        while (cb < e && t[cb] != ',') ++cb;
    }
    while (ca < cb && trim_char(t[ca])) ++ca;
    while (cb > ca && trim_char(t[cb - 1])) --cb;
    r.a = ca;
    r.b = cb;
    u64 p = ca;
    while (p < cb && c_isspace(t[p])) ++p;
    bool neg = false;
    if (p < cb && (t[p] == '+' || t[p] == '-')) neg = t[p++] == '-';
    const u64 d0 = p;
    u64 mag = 0;
    bool over = false;
    const u64 lim = neg ? (1ull << 63) : ((1ull << 63) - 1);
    while (p < cb && t[p] >= '0' && t[p] <= '9') {
        const u64 d = t[p] - '0';
        if (!over) {
            if (mag > (lim - d) / 10) over = true;
            else mag = mag * 10 + d;
        }
        ++p;
    }
    if (p == d0 || over) {
        r.status = kBadInt;  // invalid_argument / out_of_range
        return r;
    }
    if (p != cb) {
        r.status = kTrailing;
        return r;
    }
    r.value = neg ? static_cast<i64>(0ull - mag) : static_cast<i64>(mag);
    if (r.value < 1) r.status = kNonPositive;
    return r;
}

__device__ __forceinline__ void line_range(const u64* starts, u64 L, u64 nl, u64 bytes, u64& a, u64& e) {
    a = starts[L];
    e = L < nl ? starts[L + 1] - 1 : bytes;
}

__global__ void k_parse_lines(const unsigned char* __restrict__ t, u64 bytes, const u64* __restrict__ starts,
                              u64 nl, u64 first, u64 lines, int col, i64* __restrict__ vals,
                              unsigned long long* __restrict__ first_err) {
    for (u64 L = first + blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; L < lines;
         L += static_cast<u64>(gridDim.x) * blockDim.x) {
        u64 a, e;
        line_range(starts, L, nl, bytes, a, e);
        const Cell c = parse_line(t, a, e, col);
        vals[L] = (c.blank || c.status != kOk) ? 0 : c.value;
        if (!c.blank && c.status != kOk) atomicMin(first_err, static_cast<unsigned long long>(L));
    }
}

// the failing line's details: status, cell [a, b), value
__global__ void k_error_detail(const unsigned char* __restrict__ t, u64 bytes, const u64* __restrict__ starts,
                               u64 nl, u64 L, int col, i64* __restrict__ out) {
    u64 a, e;
    line_range(starts, L, nl, bytes, a, e);
    const Cell c = parse_line(t, a, e, col);
    out[0] = c.status;
    out[1] = static_cast<i64>(c.a);
    out[2] = static_cast<i64>(c.b);
    out[3] = c.value;
}

// ---- JSONL (ingest.cpp:57-88): one JSON document per line ------------------
//
// A thread walks its line with the JSON grammar nlohmann's parser accepts
// (RFC 8259; a leading UTF-8 BOM skipped, strings checked for escapes,
// surrogate pairs and well-formed UTF-8, containers matched on a bit stack)
// and records the top-level object's "length" / "id" members (keys compared
// after unescaping, the last duplicate wins). A number is an integer when it
// has no fraction or exponent and fits uint64 (non-negative) / int64
// (negative) -- strtoull / strtoll without ERANGE -- else it is a float;
// get<int64_t>() of an unsigned value wraps.
enum JsonStatus : u32 { kJOk = 0, kJInvalid = 1, kJNoLength = 2, kJNonPositive = 3, kJTooDeep = 4 };
constexpr int kJsonStackWords = 16;  // nesting up to 1024

struct JsonLine {
    u32 status;
    bool blank;
    bool has_id;
    i64 length;
    i64 id;
};

__device__ __forceinline__ bool json_ws(unsigned char ch) { return ch == ' ' || ch == '\t' || ch == '\n' || ch == '\r'; }
__device__ __forceinline__ int hexv(unsigned char ch) {
    if (ch >= '0' && ch <= '9') return ch - '0';
    if (ch >= 'a' && ch <= 'f') return ch - 'a' + 10;
    if (ch >= 'A' && ch <= 'F') return ch - 'A' + 10;
    return -1;
}

// string at t[p] == '"'; returns the index after the closing quote, or 0 on
// error. Tracks whether the decoded text equals "length" / "id".
__device__ u64 json_string(const unsigned char* t, u64 p, u64 e, bool& is_length, bool& is_id) {
    const char* kL = "length";
    int mL = 0, mI = 0;  // matched prefix, -1: mismatch
    ++p;
    while (true) {
        if (p >= e) return 0;
        u32 cp;
        const unsigned char b = t[p];
        if (b == '"') {
            ++p;
            break;
        }
        if (b < 0x20) return 0;
        if (b == '\\') {
            if (p + 1 >= e) return 0;
            const unsigned char x = t[p + 1];
            p += 2;
            switch (x) {
                case '"': cp = '"'; break;
                case '\\': cp = '\\'; break;
                case '/': cp = '/'; break;
                case 'b': cp = '\b'; break;
                case 'f': cp = '\f'; break;
                case 'n': cp = '\n'; break;
                case 'r': cp = '\r'; break;
                case 't': cp = '\t'; break;
                case 'u': {
                    if (p + 4 > e) return 0;
                    int v = 0;
                    for (int q = 0; q < 4; ++q) {
                        const int h = hexv(t[p + q]);
                        if (h < 0) return 0;
                        v = v * 16 + h;
                    }
                    p += 4;
                    if (v >= 0xD800 && v <= 0xDBFF) {
                        if (p + 6 > e || t[p] != '\\' || t[p + 1] != 'u') return 0;
                        int w = 0;
                        for (int q = 0; q < 4; ++q) {
                            const int h = hexv(t[p + 2 + q]);
                            if (h < 0) return 0;
                            w = w * 16 + h;
                        }
                        if (w < 0xDC00 || w > 0xDFFF) return 0;
                        p += 6;
                        cp = 0x10000u;  // non-ASCII: matches neither key
                    } else if (v >= 0xDC00 && v <= 0xDFFF) {
                        return 0;
                    } else {
                        cp = static_cast<u32>(v);
                    }
                    break;
                }
                default: return 0;
            }
        } else if (b < 0x80) {
            cp = b;
            ++p;
        } else {
            // RFC 3629 ranges, as nlohmann's scan_string checks them
            int cont;
            unsigned char lo = 0x80, hi = 0xBF;
            if (b >= 0xC2 && b <= 0xDF) cont = 1;
            else if (b == 0xE0) cont = 2, lo = 0xA0;
            else if ((b >= 0xE1 && b <= 0xEC) || b == 0xEE || b == 0xEF) cont = 2;
            else if (b == 0xED) cont = 2, hi = 0x9F;
            else if (b == 0xF0) cont = 3, lo = 0x90;
            else if (b >= 0xF1 && b <= 0xF3) cont = 3;
            else if (b == 0xF4) cont = 3, hi = 0x8F;
            else return 0;
            ++p;
            for (int q = 0; q < cont; ++q, ++p) {
                if (p >= e) return 0;
                const unsigned char c2 = t[p];
                if (q == 0 ? (c2 < lo || c2 > hi) : (c2 < 0x80 || c2 > 0xBF)) return 0;
            }
            cp = 0x80u;  // non-ASCII
        }
        if (mL >= 0) mL = (mL < 6 && cp == static_cast<u32>(kL[mL])) ? mL + 1 : -1;
        if (mI >= 0) mI = (mI < 2 && cp == static_cast<u32>("id"[mI])) ? mI + 1 : -1;
    }
    is_length = mL == 6;
    is_id = mI == 2;
    return p;
}

// number at t[p]; returns the index after it, or 0 on error
__device__ u64 json_number(const unsigned char* t, u64 p, u64 e, bool& is_int, i64& value) {
    const bool neg = t[p] == '-';
    if (neg) ++p;
    if (p >= e) return 0;
    u64 mag = 0;
    bool over = false;
    auto digit = [&](unsigned char ch) {
        const u64 d = ch - '0';
        if (!over) {
            if (mag > (~0ull - d) / 10) over = true;
            else mag = mag * 10 + d;
        }
    };
    if (t[p] == '0') {
        ++p;
    } else if (t[p] >= '1' && t[p] <= '9') {
        while (p < e && t[p] >= '0' && t[p] <= '9') digit(t[p++]);
    } else {
        return 0;
    }
    is_int = true;
    if (p < e && t[p] == '.') {
        ++p;
        if (p >= e || t[p] < '0' || t[p] > '9') return 0;
        while (p < e && t[p] >= '0' && t[p] <= '9') ++p;
        is_int = false;
    }
    if (p < e && (t[p] == 'e' || t[p] == 'E')) {
        ++p;
        if (p < e && (t[p] == '+' || t[p] == '-')) ++p;
        if (p >= e || t[p] < '0' || t[p] > '9') return 0;
        while (p < e && t[p] >= '0' && t[p] <= '9') ++p;
        is_int = false;
    }
    if (is_int) {
        if (neg) {
            if (over || mag > (1ull << 63)) is_int = false;
            else value = static_cast<i64>(0ull - mag);
        } else {
            if (over) is_int = false;
            else value = static_cast<i64>(mag);  // get<int64_t>() of an unsigned wraps
        }
    }
    return p;
}

// Fast path for the common record shapes, {"id":N,"length":M} and
// {"length":M} (a space allowed after ':' and ',', as json.dumps writes
// them; JSON whitespace after the closing brace): a few uniform byte tests
// instead of the grammar walk, so a warp of such lines does not diverge.
// Anything else -- and numbers of more than 18 digits -- goes to the full
// walk, which gives the same result for these shapes.
__device__ __forceinline__ bool fast_int(const unsigned char* t, u64& p, u64 e, i64& v) {
    const bool neg = p < e && t[p] == '-';
    if (neg) ++p;
    if (p >= e || t[p] < '0' || t[p] > '9') return false;
    const u64 d0 = p;
    i64 x = 0;
    while (p < e && t[p] >= '0' && t[p] <= '9') x = x * 10 + (t[p++] - '0');
    const u64 nd = p - d0;
    if (nd > 18 || (nd > 1 && t[d0] == '0')) return false;
    if (p < e && (t[p] == '.' || t[p] == 'e' || t[p] == 'E')) return false;
    v = neg ? -x : x;
    return true;
}

__device__ __forceinline__ bool fast_lit(const unsigned char* t, u64& p, u64 e, const char* s) {
    for (int k = 0; s[k]; ++k, ++p)
        if (p >= e || t[p] != static_cast<unsigned char>(s[k])) return false;
    if (p < e && t[p] == ' ') ++p;
    return true;
}

__device__ __forceinline__ bool json_fast(const unsigned char* t, u64 a, u64 e, JsonLine& r) {
    u64 p = a;
    if (p >= e || t[p] != '{') return false;
    ++p;
    i64 id = 0, len = 0;
    bool has_id = false;
    if (p + 1 < e && t[p + 1] == 'i') {
        if (!fast_lit(t, p, e, "\"id\":") || !fast_int(t, p, e, id) || !fast_lit(t, p, e, ",")) return false;
        has_id = true;
    }
    if (!fast_lit(t, p, e, "\"length\":") || !fast_int(t, p, e, len) || p >= e || t[p] != '}') return false;
    for (++p; p < e; ++p)
        if (!json_ws(t[p])) return false;
    r.blank = false;
    r.has_id = has_id;
    r.id = id;
    r.length = len;
    r.status = len < 1 ? kJNonPositive : kJOk;
    return true;
}

__device__ JsonLine parse_json_line(const unsigned char* __restrict__ t, u64 a, u64 e) {
    JsonLine r{kJOk, true, false, 0, 0};
    if (json_fast(t, a, e, r)) return r;
    for (u64 p = a; p < e; ++p)
        if (!trim_char(t[p])) {
            r.blank = false;
            break;
        }
    if (r.blank) return r;
    enum { kValue, kValueOrClose, kKey, kKeyOrClose, kAfter };
    u64 stack[kJsonStackWords];  // bit set: object
    int depth = 0, state = kValue;
    bool top_obj = false;
    int len_state = 0, pending = 0;  // len_state: 0 absent, 1 integer, 2 other; pending: 1 length, 2 id
    u64 p = a;
    if (p < e && t[p] == 0xEF) {
        if (p + 2 < e && t[p + 1] == 0xBB && t[p + 2] == 0xBF) p += 3;
        else return r.status = kJInvalid, r;
    }
    auto is_obj = [&](int d) { return (stack[(d - 1) >> 6] >> ((d - 1) & 63)) & 1ull; };
    auto record = [&](bool is_int, i64 v) {
        if (pending == 1) {
            len_state = is_int ? 1 : 2;
            r.length = v;
        } else if (pending == 2) {
            r.has_id = is_int;
            r.id = v;
        }
        pending = 0;
    };
    while (true) {
        while (p < e && json_ws(t[p])) ++p;
        if (p < e && t[p] == 0) e = p;  // nlohmann's lexer reads '\0' outside a string as end of input
        if (p >= e) {
            if (state == kAfter && depth == 0) break;
            return r.status = kJInvalid, r;
        }
        const unsigned char ch = t[p];
        if (state == kValue || state == kValueOrClose) {
            if (state == kValueOrClose && ch == ']') {
                --depth;
                ++p;
                state = kAfter;
                continue;
            }
            if (ch == '{' || ch == '[') {
                record(false, 0);
                if (depth == 0) top_obj = ch == '{';
                if (depth == 64 * kJsonStackWords) return r.status = kJTooDeep, r;
                const u64 bit = 1ull << (depth & 63);
                if (ch == '{') stack[depth >> 6] |= bit;
                else stack[depth >> 6] &= ~bit;
                ++depth;
                ++p;
                state = ch == '{' ? kKeyOrClose : kValueOrClose;
                continue;
            }
            if (ch == '"') {
                bool l_, i_;
                p = json_string(t, p, e, l_, i_);
                if (!p) return r.status = kJInvalid, r;
                record(false, 0);
            } else if (ch == '-' || (ch >= '0' && ch <= '9')) {
                bool is_int = false;
                i64 v = 0;
                p = json_number(t, p, e, is_int, v);
                if (!p) return r.status = kJInvalid, r;
                record(is_int, v);
            } else {
                const char* lit = ch == 't' ? "true" : ch == 'f' ? "false" : ch == 'n' ? "null" : nullptr;
                if (!lit) return r.status = kJInvalid, r;
                for (int q = 0; lit[q]; ++q, ++p)
                    if (p >= e || t[p] != static_cast<unsigned char>(lit[q])) return r.status = kJInvalid, r;
                record(false, 0);
            }
            state = kAfter;
            continue;
        }
        if (state == kKey || state == kKeyOrClose) {
            if (state == kKeyOrClose && ch == '}') {
                --depth;
                ++p;
                state = kAfter;
                continue;
            }
            if (ch != '"') return r.status = kJInvalid, r;
            bool is_len = false, is_id = false;
            p = json_string(t, p, e, is_len, is_id);
            if (!p) return r.status = kJInvalid, r;
            while (p < e && json_ws(t[p])) ++p;
            if (p >= e || t[p] != ':') return r.status = kJInvalid, r;
            ++p;
            pending = depth == 1 ? (is_len ? 1 : is_id ? 2 : 0) : 0;
            state = kValue;
            continue;
        }
        // kAfter: a value just ended
        if (depth == 0) return r.status = kJInvalid, r;
        const bool obj = is_obj(depth);
        if (ch == ',') {
            state = obj ? kKey : kValue;
            ++p;
        } else if (ch == (obj ? '}' : ']')) {
            --depth;
            ++p;
        } else {
            return r.status = kJInvalid, r;
        }
    }
    if (!top_obj || len_state != 1) return r.status = kJNoLength, r;
    if (r.length < 1) r.status = kJNonPositive;
    return r;
}

__global__ void k_parse_jsonl(const unsigned char* __restrict__ t, u64 bytes, const u64* __restrict__ starts, u64 nl,
                              u64 lines, i64* __restrict__ vals, i64* __restrict__ ids,
                              unsigned long long* __restrict__ first_err) {
    for (u64 L = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; L < lines;
         L += static_cast<u64>(gridDim.x) * blockDim.x) {
        u64 a, e;
        line_range(starts, L, nl, bytes, a, e);
        const JsonLine j = parse_json_line(t, a, e);
        const bool keep = !j.blank && j.status == kJOk;
        vals[L] = keep ? j.length : 0;
        ids[L] = j.has_id ? j.id : 0;
        if (keep && j.has_id) vals[L] = -vals[L];  // a negative value marks an explicit id (lengths are >= 1)
        if (!j.blank && j.status != kJOk) atomicMin(first_err, static_cast<unsigned long long>(L));
    }
}

__global__ void k_jsonl_detail(const unsigned char* __restrict__ t, u64 bytes, const u64* __restrict__ starts, u64 nl,
                               u64 L, i64* __restrict__ out) {
    u64 a, e;
    line_range(starts, L, nl, bytes, a, e);
    const JsonLine j = parse_json_line(t, a, e);
    out[0] = j.status;
    out[1] = static_cast<i64>(a);
    out[2] = static_cast<i64>(e);
    out[3] = j.length;
}

// split_csv_row (ingest.cpp:41-55) of the header line
std::vector<std::string> split_csv(const std::string& line) {
    std::vector<std::string> cells;
    size_t p = 0;
    if (!line.empty()) {
        while (true) {
            const size_t q = line.find(',', p);
            std::string cell = line.substr(p, q == std::string::npos ? std::string::npos : q - p);
            const auto b = cell.find_first_not_of(" \t\r");
            const auto e = cell.find_last_not_of(" \t\r");
            cells.push_back(b == std::string::npos ? "" : cell.substr(b, e - b + 1));
            if (q == std::string::npos || q + 1 == line.size()) break;
            p = q + 1;
        }
        if (line.back() == ',') cells.push_back("");
    }
    return cells;
}

}  // namespace

void upload_text(Ctx& c, const char* text, u64 bytes, DevBuf<unsigned char>& t) {
    const u64 chunks = (bytes + kChunkBytes - 1) / kChunkBytes;
    t.alloc(chunks * kChunkBytes + kChunkBytes, c.stream);
    CUDA_CHECK(cudaMemsetAsync(t.p + bytes, 0, t.n - bytes, c.stream));
    staged_copy(c, t.p, text, bytes, true);
}

u64 text_line_starts(Ctx& c, const unsigned char* t, u64 bytes, DevBuf<u64>& starts) {
    cudaStream_t s = c.stream;
    const u64 chunks = (bytes + kChunkBytes - 1) / kChunkBytes;
    DevBuf<u64> chunk_line(chunks + 1, s);
    {
        const uint4* tv = reinterpret_cast<const uint4*>(t);
        u64* cl = chunk_line.p;
        const i64 C = static_cast<i64>(chunks);
        scan_exclusive<u64>(
            C + 1, [=] __device__(i64 i) { return i < C ? static_cast<u64>(nl_in(tv[i])) : 0ull; },
            [=] __device__(i64 i, u64 v) { cl[i] = v; }, s, c.scan, "corpus.lines", 1.0 * kChunkBytes / 1.0);
    }
    const u64 nl = read_vector(c, chunk_line.p + chunks, 1)[0];
    starts.alloc(nl + 2, s);
    CUDA_CHECK(cudaMemsetAsync(starts.p, 0, sizeof(u64), s));
    if (chunks) LAUNCH(k_line_starts, grid_for(chunks, 256), 256, 0, s, t, bytes, chunk_line.p, starts.p);
    return nl;
}

i64 parse_corpus_text(Ctx& c, const char* text, u64 bytes, int format, const std::string& source,
                      DevBuf<int64_t>& lengths, DevBuf<int64_t>& ids) {
    cudaStream_t s = c.stream;
    if (format != HBP_CORPUS_CSV && format != HBP_CORPUS_RAW && format != HBP_CORPUS_JSONL)
        fail_validation("unknown corpus format");
    const bool jsonl = format == HBP_CORPUS_JSONL;
    int col = -1;
    u64 first = 0;
    if (format == HBP_CORPUS_CSV) {
        // load_csv (ingest.cpp:90-104): the header row names the column
        if (bytes == 0) fail_validation("empty corpus: " + source);
        const void* nlp = std::memchr(text, '\n', bytes);
        const size_t hl = nlp ? static_cast<size_t>(static_cast<const char*>(nlp) - text) : bytes;
        const auto header = split_csv(std::string(text, hl));
        size_t k = 0;
        while (k < header.size() && header[k] != "length") ++k;
        if (k == header.size()) fail_validation("csv header has no \"length\" column: " + source);
        col = static_cast<int>(k);
        first = 1;
    }
    DevBuf<unsigned char> t;
    upload_text(c, text, bytes, t);
    DevBuf<u64> starts;
    const u64 nl = text_line_starts(c, t.p, bytes, starts);
    unsigned char last = 0;
    if (bytes) last = static_cast<unsigned char>(text[bytes - 1]);
    const u64 lines = nl + ((bytes > 0 && last != '\n') ? 1 : 0);
    DevBuf<i64> vals(lines + 1, s), lid(jsonl ? lines + 1 : 0, s);
    DevBuf<unsigned long long> ferr(1, s);
    CUDA_CHECK(cudaMemsetAsync(ferr.p, 0xff, sizeof(unsigned long long), s));
    if (jsonl && lines > 0)
        LAUNCH(k_parse_jsonl, grid_for(lines, 128), 128, 0, s, t.p, bytes, starts.p, nl, lines, vals.p, lid.p, ferr.p);
    else if (lines > first)
        LAUNCH(k_parse_lines, grid_for(lines - first, 256), 256, 0, s, t.p, bytes, starts.p, nl, first, lines, col,
               vals.p, ferr.p);
    const unsigned long long fe = read_vector(c, ferr.p, 1)[0];
    if (fe != ~0ull) {
        DevBuf<i64> det(4, s);
        if (jsonl) LAUNCH(k_jsonl_detail, 1, 1, 0, s, t.p, bytes, starts.p, nl, static_cast<u64>(fe), det.p);
        else LAUNCH(k_error_detail, 1, 1, 0, s, t.p, bytes, starts.p, nl, static_cast<u64>(fe), col, det.p);
        const auto d = read_vector(c, det.p, 4);
        const std::string line = "line " + std::to_string(fe + 1) + ": ";
        const std::string cell(text + d[1], text + d[2]);
        if (jsonl) {
            switch (d[0]) {
                case kJInvalid: {
                    // the message is nlohmann's parse_error text of this one line
                    const std::string what = json_parse_error_text(cell);
                    if (what.empty())
                        throw EngineError(HBP_ERR_CUDA, line + "JSON validity disagrees with the host parser");
                    fail_validation(line + "invalid JSON: " + what);
                }
                case kJNoLength: fail_validation(line + "expected object with integer \"length\"");
                case kJNonPositive: fail_validation(line + "length must be >= 1, got " + std::to_string(d[3]));
                default:
                    throw EngineError(HBP_ERR_VALIDATION,
                                      line + "JSON nested deeper than 1024 levels (GPU parser limit)");
            }
        }
        switch (d[0]) {
            case kBadInt: fail_validation(line + "not an integer length: '" + cell + "'");
            case kTrailing: fail_validation(line + "trailing garbage after length: '" + cell + "'");
            case kNonPositive: fail_validation(line + "length must be >= 1, got " + std::to_string(d[3]));
            default: fail_validation(line + "too few columns");
        }
    }
    // compaction of the kept (non-blank) lines; ids by record index unless
    // a JSONL record names its own (marked by a negative value)
    DevBuf<u64> cnt(1, s);
    const i64 NL = static_cast<i64>(lines);
    {
        const i64* vp = vals.p;
        const i64* ip = lid.p;
        const u64 f = first;
        lengths.alloc(lines > first ? lines - first : 1, s);
        ids.alloc(lines > first ? lines - first : 1, s);
        int64_t* op = lengths.p;
        int64_t* oi = ids.p;
        u64* cp = cnt.p;
        scan_exclusive<u64>(
            NL + 1, [=] __device__(i64 i) { return (i < NL && static_cast<u64>(i) >= f && vp[i] != 0) ? 1ull : 0ull; },
            [=] __device__(i64 i, u64 v) {
                if (i == NL) {
                    *cp = v;
                } else if (static_cast<u64>(i) >= f && vp[i] != 0) {
                    const i64 x = vp[i];
                    op[v] = x < 0 ? -x : x;
                    oi[v] = x < 0 ? ip[i] : static_cast<i64>(v);
                }
            },
            s, c.scan, "corpus.compact", 24.0);
    }
    const u64 n = read_vector(c, cnt.p, 1)[0];
    if (n == 0) fail_validation("empty corpus: " + source);
    if (jsonl) {
        // SampleSet::validate (types.cpp:8-24): explicit ids may repeat
        hbp_samples smp{ids.p, lengths.p, static_cast<int64_t>(n), HBP_MEM_DEVICE, source.c_str()};
        DeviceCorpus corpus;
        ingest(c, &smp, corpus);
        validate_corpus(c, &smp, corpus, source);
    }
    return static_cast<i64>(n);
}

}  // namespace hbp_b200
