// corpus.cu — corpus file parsers on the GPU: raw-lengths and CSV
// (src/ingest.cpp:57-169, load_raw / load_csv / load_lengths).
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
// formats the error message from the failing cell's bytes.
#include <cstring>
#include <string>
#include <vector>

#include "pipeline.cuh"
#include "scan.cuh"

namespace hbp_b200 {
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

i64 parse_corpus_text(Ctx& c, const char* text, u64 bytes, int format, const std::string& source,
                      DevBuf<int64_t>& lengths) {
    cudaStream_t s = c.stream;
    if (format != HBP_CORPUS_CSV && format != HBP_CORPUS_RAW)
        throw EngineError(HBP_ERR_VALIDATION, "corpus format not available in the GPU engine: jsonl");
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
    const u64 chunks = (bytes + kChunkBytes - 1) / kChunkBytes;
    DevBuf<unsigned char> t(chunks * kChunkBytes + kChunkBytes, s);
    if (bytes) CUDA_CHECK(cudaMemcpyAsync(t.p, text, bytes, cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaMemsetAsync(t.p + bytes, 0, t.n - bytes, s));
    DevBuf<u64> chunk_line(chunks + 1, s);
    {
        const uint4* tv = reinterpret_cast<const uint4*>(t.p);
        u64* cl = chunk_line.p;
        const i64 C = static_cast<i64>(chunks);
        scan_exclusive<u64>(
            C + 1, [=] __device__(i64 i) { return i < C ? static_cast<u64>(nl_in(tv[i])) : 0ull; },
            [=] __device__(i64 i, u64 v) { cl[i] = v; }, s, c.scan, "corpus.lines", 1.0 * kChunkBytes / 1.0);
    }
    const u64 nl = read_vector(c, chunk_line.p + chunks, 1)[0];
    unsigned char last = 0;
    if (bytes) last = static_cast<unsigned char>(text[bytes - 1]);
    const u64 lines = nl + ((bytes > 0 && last != '\n') ? 1 : 0);
    DevBuf<u64> starts(nl + 2, s);
    CUDA_CHECK(cudaMemsetAsync(starts.p, 0, sizeof(u64), s));
    if (chunks) LAUNCH(k_line_starts, grid_for(chunks, 256), 256, 0, s, t.p, bytes, chunk_line.p, starts.p);
    DevBuf<i64> vals(lines + 1, s);
    DevBuf<unsigned long long> ferr(1, s);
    CUDA_CHECK(cudaMemsetAsync(ferr.p, 0xff, sizeof(unsigned long long), s));
    if (lines > first)
        LAUNCH(k_parse_lines, grid_for(lines - first, 256), 256, 0, s, t.p, bytes, starts.p, nl, first, lines, col,
               vals.p, ferr.p);
    const unsigned long long fe = read_vector(c, ferr.p, 1)[0];
    if (fe != ~0ull) {
        DevBuf<i64> det(4, s);
        LAUNCH(k_error_detail, 1, 1, 0, s, t.p, bytes, starts.p, nl, static_cast<u64>(fe), col, det.p);
        const auto d = read_vector(c, det.p, 4);
        const std::string line = "line " + std::to_string(fe + 1) + ": ";
        const std::string cell(text + d[1], text + d[2]);
        switch (d[0]) {
            case kBadInt: fail_validation(line + "not an integer length: '" + cell + "'");
            case kTrailing: fail_validation(line + "trailing garbage after length: '" + cell + "'");
            case kNonPositive: fail_validation(line + "length must be >= 1, got " + std::to_string(d[3]));
            default: fail_validation(line + "too few columns");
        }
    }
    // compaction of the kept (non-blank) lines
    DevBuf<u64> cnt(1, s);
    const i64 NL = static_cast<i64>(lines);
    {
        const i64* vp = vals.p;
        const u64 f = first;
        lengths.alloc(lines > first ? lines - first : 1, s);
        int64_t* op = lengths.p;
        u64* cp = cnt.p;
        scan_exclusive<u64>(
            NL + 1, [=] __device__(i64 i) { return (i < NL && static_cast<u64>(i) >= f && vp[i] > 0) ? 1ull : 0ull; },
            [=] __device__(i64 i, u64 v) {
                if (i == NL) *cp = v;
                else if (static_cast<u64>(i) >= f && vp[i] > 0) op[v] = vp[i];
            },
            s, c.scan, "corpus.compact", 16.0);
    }
    const u64 n = read_vector(c, cnt.p, 1)[0];
    if (n == 0) fail_validation("empty corpus: " + source);
    return static_cast<i64>(n);
}

}  // namespace hbp_b200
