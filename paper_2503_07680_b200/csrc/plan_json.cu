// plan_json.cu — the plan manifest reader for any JSON layout (SURVEY.md
// §8(f) row 1).
//
// Reference: plan_from_json (src/io.cpp:112-160) parses with nlohmann's DOM,
// so whitespace, key order, duplicate keys (the last one wins), unknown keys,
// extra sample elements, escaped key text and booleans or floats where
// numbers are read are all accepted. plan_read.cu reads the canonical layout
// write_plan produces line by line; any other text comes here.
//
// 1. Strings. Every 64-byte chunk maps the lexer state at its start
//    (outside a string / inside / inside after a backslash) to the state at
//    its end; a scan of these maps gives every chunk its start state.
// 2. Tokens. With its start state each chunk emits its tokens outside
//    strings: { } [ ] : , a string (its opening quote) or a scalar (a maximal
//    run of bytes that are not white space, structural or a quote); a NUL
//    outside a string ends the input, as nlohmann's lexer treats it.
// 3. Token text: strings decoded and checked as nlohmann's scanner does
//    (escapes, surrogate pairs, RFC 3629 UTF-8, no control bytes), numbers
//    against the JSON grammar over the whole scalar, literals exactly.
// 4. Nesting. The depth before every token is a scan of opens and closes.
//    A stable sort by depth lays every container's children (and its close)
//    out contiguously, each run starting at the token after the container's
//    open; so every token learns its container's type and every open its
//    close. The grammar is then local: each pair of neighbouring tokens, the
//    container type, one value at depth 0.
// 5. The manifest. Iterations are the objects at depth 2 of the root's live
//    "iterations" array; their live "group" / "phase" / "devices" members
//    (last duplicate wins, unknown keys ignored -- their subtrees masked by a
//    scan of range marks), devices at depth 4, packs at 5, their live
//    "capacity" / "samples" at 6, samples at 7 and their first two elements
//    at 8. Scans over the array count iterations, devices, packs and samples
//    before every token; one pass scatters the values into the plan's CSR
//    arrays, converting numbers as nlohmann's get<int> / get<int64_t> do.
//    The header (version, groups, device_count, seed: a few hundred bytes)
//    is read on the host from the text with the iterations value replaced
//    by [] (manifest_host.hpp).
// Errors: text nlohmann rejects gets its parse_error message; a type or
// key error, a group out of range or an overfull pack the message the
// reference raises first in its own order (the host formats it once the
// device has found that there is one).
#include <cstring>
#include <string>

#include "../../include/hbp_b200.h"
#include "engine.cuh"
#include "manifest_host.hpp"
#include "pipeline.cuh"
#include "radix.cuh"
#include "scan.cuh"

#include <math_constants.h>

namespace hbp_b200 {
namespace {

enum : u8 {
    kJNone = 0, kJObj, kJObjEnd, kJArr, kJArrEnd, kJColon, kJComma, kJStr, kJNum, kJTrue, kJFalse, kJNull, kJBad
};
enum : u8 { kCNone = 0, kCObj = 1, kCArr = 2 };  // container of a token
// decoded names the reader looks up
enum : u8 { kNOther = 0, kNIterations, kNGroup, kNPhase, kNDevices, kNCapacity, kNSamples, kNWarmup };
// numbers: how get<>() converts them
enum : u8 { kVNone = 0, kVInt, kVUint, kVDouble, kVInexact, kVBool };
// flags[0] bits
constexpr u32 kFInvalid = 1u, kFSemantic = 2u, kFExotic = 4u;

constexpr int kJB = 256;            // threads per block, text passes
constexpr int kJC = 64;             // bytes per thread
constexpr int kJSpan = kJB * kJC;   // bytes per block

__device__ __forceinline__ bool is_open(u8 k) { return k == kJObj || k == kJArr; }
__device__ __forceinline__ bool is_close(u8 k) { return k == kJObjEnd || k == kJArrEnd; }
__device__ __forceinline__ bool value_start(u8 k) { return k == kJObj || k == kJArr || (k >= kJStr && k <= kJNull); }
__device__ __forceinline__ bool scalar_end(u8 k) { return k >= kJStr && k <= kJNull; }
__device__ __forceinline__ bool numeric(u8 k) { return k == kJNum || k == kJTrue || k == kJFalse; }

// lexer state: 0 outside a string, 1 inside, 2 inside after a backslash
__device__ __forceinline__ u32 jstep(u32 s, unsigned char b) {
    if (s == 0) return b == '"' ? 1u : 0u;
    if (s == 1) return b == '"' ? 0u : (b == '\\' ? 2u : 1u);
    return 1u;
}
// maps of the 3 states, 2 bits each; then(f, g) = g after f
__device__ __forceinline__ u32 fn_at(u32 f, u32 s) { return (f >> (2 * s)) & 3u; }
__device__ __forceinline__ u32 fn_then(u32 f, u32 g) {
    return fn_at(g, fn_at(f, 0)) | (fn_at(g, fn_at(f, 1)) << 2) | (fn_at(g, fn_at(f, 2)) << 4);
}
constexpr u32 kFnId = 0u | (1u << 2) | (2u << 4);

__device__ __forceinline__ bool ws(unsigned char b) { return b == ' ' || b == '\t' || b == '\n' || b == '\r'; }
__device__ __forceinline__ bool structural(unsigned char b) {
    return b == '{' || b == '}' || b == '[' || b == ']' || b == ':' || b == ',';
}
__device__ __forceinline__ bool scalar_byte(unsigned char b) { return !ws(b) && !structural(b) && b != '"' && b != 0; }

// The block's span of text in shared memory (zero past the input); bytes
// before `skip` (a UTF-8 BOM) read as white space.
__device__ __forceinline__ void stage(const unsigned char* __restrict__ t, u64 padded, u64 bytes, u64 skip,
                                      unsigned char* s) {
    const u64 b0 = static_cast<u64>(blockIdx.x) * kJSpan;
    uint4* s4 = reinterpret_cast<uint4*>(s);
    const uint4* t4 = reinterpret_cast<const uint4*>(t);
    for (int i = threadIdx.x; i < kJSpan / 16; i += kJB) {
        const u64 g = b0 + static_cast<u64>(i) * 16;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (g + 16 <= padded) v = t4[g / 16];
        s4[i] = v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kJSpan; i += kJB) {
        const u64 g = b0 + i;
        if (g >= bytes) s[i] = 0;
        else if (g < skip) s[i] = ' ';
    }
    __syncthreads();
}

// this thread's chunk map, and the exclusive scan of the block's maps
__device__ __forceinline__ u32 chunk_map(const unsigned char* s) {
    u32 a = 0, b = 1, c = 2;
    const unsigned char* p = s + threadIdx.x * kJC;
#pragma unroll 8
    for (int i = 0; i < kJC; ++i) {
        const unsigned char x = p[i];
        a = jstep(a, x);
        b = jstep(b, x);
        c = jstep(c, x);
    }
    return a | (b << 2) | (c << 4);
}
__device__ __forceinline__ u32 block_map_scan(u32 f, u32* sh, u32& total) {
    sh[threadIdx.x] = f;
    __syncthreads();
    for (int off = 1; off < kJB; off <<= 1) {  // inclusive, earlier maps first
        const u32 prev = threadIdx.x >= static_cast<u32>(off) ? sh[threadIdx.x - off] : kFnId;
        __syncthreads();
        sh[threadIdx.x] = fn_then(prev, sh[threadIdx.x]);
        __syncthreads();
    }
    total = sh[kJB - 1];
    const u32 excl = threadIdx.x ? sh[threadIdx.x - 1] : kFnId;
    __syncthreads();
    return excl;
}

__global__ void __launch_bounds__(kJB) k_js_blockmap(const unsigned char* __restrict__ t, u64 padded, u64 bytes,
                                                      u64 skip, u32* __restrict__ bmap) {
    __shared__ __align__(16) unsigned char s[kJSpan];
    __shared__ u32 sh[kJB];
    stage(t, padded, bytes, skip, s);
    u32 total;
    block_map_scan(chunk_map(s), sh, total);
    if (threadIdx.x == 0) bmap[blockIdx.x] = total;
}

// exclusive scan of the block maps, one block: each thread composes a
// stretch, a Hillis-Steele scan over the stretches, then the stretch again
__global__ void __launch_bounds__(1024) k_js_topmap(u32* __restrict__ bmap, u64 nb) {
    __shared__ u32 sh[1024];
    const u64 per = (nb + 1023) / 1024;
    const u64 a = threadIdx.x * per, e = min(nb, a + per);
    u32 f = kFnId;
    for (u64 i = a; i < e; ++i) f = fn_then(f, bmap[i]);
    sh[threadIdx.x] = f;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const u32 prev = threadIdx.x >= static_cast<u32>(off) ? sh[threadIdx.x - off] : kFnId;
        __syncthreads();
        sh[threadIdx.x] = fn_then(prev, sh[threadIdx.x]);
        __syncthreads();
    }
    u32 run = threadIdx.x ? sh[threadIdx.x - 1] : kFnId;
    for (u64 i = a; i < e; ++i) {
        const u32 x = bmap[i];
        bmap[i] = run;
        run = fn_then(run, x);
    }
}

__device__ __forceinline__ u8 token_kind(unsigned char b) {
    switch (b) {
        case '{': return kJObj;
        case '}': return kJObjEnd;
        case '[': return kJArr;
        case ']': return kJArrEnd;
        case ':': return kJColon;
        case ',': return kJComma;
        case '"': return kJStr;
        case 't': return kJTrue;
        case 'f': return kJFalse;
        case 'n': return kJNull;
        default: return (b == '-' || (b >= '0' && b <= '9')) ? kJNum : kJBad;
    }
}

// Walks this thread's chunk from its start state. EMIT = false: counts the
// tokens (and the first NUL outside a string); true: writes them.
template <bool EMIT>
__global__ void __launch_bounds__(kJB) k_js_tokens(const unsigned char* __restrict__ t, u64 padded, u64 bytes,
                                                    u64 skip, const u32* __restrict__ bmap, u32* __restrict__ count,
                                                    const u64* __restrict__ offset, unsigned long long* __restrict__ nul,
                                                    u32* __restrict__ tpos, u8* __restrict__ tkind) {
    __shared__ __align__(16) unsigned char s[kJSpan];
    __shared__ u32 sh[kJB];
    stage(t, padded, bytes, skip, s);
    u32 total;
    const u32 excl = block_map_scan(chunk_map(s), sh, total);
    u32 st = fn_at(excl, fn_at(bmap[blockIdx.x], 0));
    const u64 c0 = static_cast<u64>(blockIdx.x) * kJSpan + threadIdx.x * kJC;
    const unsigned char* p = s + threadIdx.x * kJC;
    // the byte before the chunk continues a scalar when the chunk starts outside a string
    bool prev_scalar = false;
    if (st == 0 && c0 > 0) {
        const u64 g = c0 - 1;
        const unsigned char b = (threadIdx.x > 0) ? p[-1] : (g < bytes ? t[g] : 0);
        prev_scalar = g >= skip && g < bytes && scalar_byte(b);
    }
    u32 n = 0;
    u64 o = EMIT ? offset[static_cast<u64>(blockIdx.x) * kJB + threadIdx.x] : 0;
    for (int i = 0; i < kJC; ++i) {
        const unsigned char b = p[i];
        const u64 g = c0 + i;
        if (g >= bytes) break;
        if (st == 0) {
            bool tok = false;
            if (b == 0) {
                if (!EMIT) atomicMin(nul, static_cast<unsigned long long>(g));
                break;  // end of input (the rest of the chunk is past it)
            }
            if (structural(b) || b == '"') tok = true;
            else if (scalar_byte(b)) tok = !prev_scalar;
            prev_scalar = scalar_byte(b);
            if (tok) {
                if (EMIT) {
                    tpos[o] = static_cast<u32>(g);
                    tkind[o] = token_kind(b);
                    ++o;
                }
                ++n;
            }
        } else {
            prev_scalar = false;
        }
        st = jstep(st, b);
    }
    if (!EMIT) count[static_cast<u64>(blockIdx.x) * kJB + threadIdx.x] = n;
}

// ---- token text --------------------------------------------------------

__device__ __forceinline__ int hex_of(unsigned char ch) {
    if (ch >= '0' && ch <= '9') return ch - '0';
    if (ch >= 'a' && ch <= 'f') return ch - 'a' + 10;
    if (ch >= 'A' && ch <= 'F') return ch - 'A' + 10;
    return -1;
}

struct NameBuf {
    char c[12];
    int n;  // decoded ASCII length; -1: longer, or not ASCII
    __device__ void push(u32 cp) {
        if (n < 0) return;
        if (cp >= 0x80 || n >= 12) {
            n = -1;
            return;
        }
        c[n++] = static_cast<char>(cp);
    }
    __device__ bool is(const char* w) const {
        int k = 0;
        for (; w[k]; ++k)
            if (k >= n || c[k] != w[k]) return false;
        return k == n;
    }
};

// String at t[p] == '"' (nlohmann's scan_string): returns one past the
// closing quote, 0 if invalid; the decoded text's name.
__device__ u64 scan_string(const unsigned char* t, u64 p, u64 e, u8& name) {
    NameBuf nb;
    nb.n = 0;
    ++p;
    while (true) {
        if (p >= e) return 0;
        const unsigned char b = t[p];
        if (b == '"') {
            ++p;
            break;
        }
        if (b < 0x20) return 0;
        u32 cp;
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
                        const int h = hex_of(t[p + q]);
                        if (h < 0) return 0;
                        v = v * 16 + h;
                    }
                    p += 4;
                    if (v >= 0xD800 && v <= 0xDBFF) {
                        if (p + 6 > e || t[p] != '\\' || t[p + 1] != 'u') return 0;
                        int w = 0;
                        for (int q = 0; q < 4; ++q) {
                            const int h = hex_of(t[p + 2 + q]);
                            if (h < 0) return 0;
                            w = w * 16 + h;
                        }
                        if (w < 0xDC00 || w > 0xDFFF) return 0;
                        p += 6;
                        cp = 0x10000u;
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
            cp = 0x80u;
        }
        nb.push(cp);
    }
    name = nb.is("iterations") ? kNIterations
           : nb.is("group")    ? kNGroup
           : nb.is("phase")    ? kNPhase
           : nb.is("devices")  ? kNDevices
           : nb.is("capacity") ? kNCapacity
           : nb.is("samples")  ? kNSamples
           : nb.is("warmup")   ? kNWarmup
                               : kNOther;
    return p;
}

// Number over the whole scalar [p, e) (JSON grammar). Integers that fit
// int64 / uint64 are exact (nlohmann's number_integer / number_unsigned);
// others become doubles: exact when the decimal significand has at most 15
// digits and a power-of-ten exponent of at most 22 (Clinger's fast path),
// else marked inexact. Returns false if the grammar fails.
__device__ bool scan_number(const unsigned char* t, u64 p, u64 e, u8& cls, i64& bits) {
    const bool neg = t[p] == '-';
    if (neg) ++p;
    if (p >= e) return false;
    u64 mag = 0, sig = 0;
    int sig_digits = 0, exp10 = 0;
    bool over = false;
    auto add_sig = [&](unsigned char ch, bool frac) {
        const u32 d = ch - '0';
        if (sig_digits == 0 && d == 0) {
            if (frac) --exp10;
            return;
        }
        if (sig_digits < 19) {
            sig = sig * 10 + d;
            ++sig_digits;
            if (frac) --exp10;
        } else {
            sig_digits = 99;  // too many significant digits for the fast path
            if (!frac) ++exp10;
        }
    };
    if (t[p] == '0') {
        ++p;
    } else if (t[p] >= '1' && t[p] <= '9') {
        while (p < e && t[p] >= '0' && t[p] <= '9') {
            const u64 d = t[p] - '0';
            if (!over) {
                if (mag > (~0ull - d) / 10) over = true;
                else mag = mag * 10 + d;
            }
            add_sig(t[p], false);
            ++p;
        }
    } else {
        return false;
    }
    bool is_int = true;
    if (p < e && t[p] == '.') {
        ++p;
        if (p >= e || t[p] < '0' || t[p] > '9') return false;
        while (p < e && t[p] >= '0' && t[p] <= '9') add_sig(t[p++], true);
        is_int = false;
    }
    if (p < e && (t[p] == 'e' || t[p] == 'E')) {
        ++p;
        bool eneg = false;
        if (p < e && (t[p] == '+' || t[p] == '-')) eneg = t[p++] == '-';
        if (p >= e || t[p] < '0' || t[p] > '9') return false;
        int ev = 0;
        while (p < e && t[p] >= '0' && t[p] <= '9') {
            if (ev < 100000) ev = ev * 10 + (t[p] - '0');
            ++p;
        }
        exp10 += eneg ? -ev : ev;
        is_int = false;
    }
    if (p != e) return false;
    if (is_int && !over && (!neg || mag <= (1ull << 63))) {
        if (neg) {
            cls = kVInt;
            bits = static_cast<i64>(0ull - mag);
        } else {
            cls = mag > 0x7fffffffffffffffull ? kVUint : kVInt;
            bits = static_cast<i64>(mag);
        }
        return true;
    }
    if (sig == 0) {  // zero in any form
        cls = kVDouble;
        bits = __double_as_longlong(neg ? -0.0 : 0.0);
        return true;
    }
    // the reader only converts numbers to integers: what matters is the
    // truncated value, or that it is out of every integer's range
    const int mag10 = (sig_digits > 19 ? 19 : sig_digits) + exp10;  // |v| in [10^(mag10-1), 10^mag10)
    if (mag10 > 20) {  // |v| >= 10^20 > 2^64: every conversion overflows (x86: the "integer indefinite")
        cls = kVDouble;
        bits = __double_as_longlong(neg ? -CUDART_INF : CUDART_INF);
        return true;
    }
    if (mag10 <= 0) {  // |v| < 1: truncates to 0
        cls = kVDouble;
        bits = __double_as_longlong(neg ? -0.0 : 0.0);
        return true;
    }
    if (sig_digits <= 15 && exp10 >= -22 && exp10 <= 22) {
        const double p10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                                1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
        double v = static_cast<double>(sig);
        v = exp10 >= 0 ? __dmul_rn(v, p10[exp10]) : __ddiv_rn(v, p10[-exp10]);
        cls = kVDouble;
        bits = __double_as_longlong(neg ? -v : v);
        return true;
    }
    cls = kVInexact;
    bits = 0;
    return true;
}

__global__ void k_js_text(const unsigned char* __restrict__ t, u64 end, const u32* __restrict__ tpos,
                          const u8* __restrict__ tkind, u64 T, u8* __restrict__ tname, u8* __restrict__ tcls,
                          i64* __restrict__ tval, u32* __restrict__ flags) {
    for (u64 k = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; k < T;
         k += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u8 kind = tkind[k];
        const u64 p = tpos[k];
        u8 name = kNOther, cls = kVNone;
        i64 v = 0;
        bool ok = true;
        if (kind == kJStr) {
            ok = scan_string(t, p, end, name) != 0;
        } else if (kind >= kJNum) {
            u64 q = p;
            while (q < end && scalar_byte(t[q])) ++q;
            if (kind == kJNum) {
                ok = scan_number(t, p, q, cls, v);
            } else if (kind == kJBad) {
                ok = false;
            } else {
                const char* lit = kind == kJTrue ? "true" : kind == kJFalse ? "false" : "null";
                u64 l = 0;
                while (lit[l]) ++l;
                ok = q - p == l;
                for (u64 j = 0; ok && j < l; ++j) ok = t[p + j] == static_cast<unsigned char>(lit[j]);
                if (kind != kJNull) {
                    cls = kVBool;
                    v = kind == kJTrue ? 1 : 0;
                }
            }
        }
        if (!ok) atomicOr(flags, kFInvalid);
        tname[k] = name;
        tcls[k] = cls;
        tval[k] = v;
    }
}

// ---- nesting and grammar ------------------------------------------------

// sorted position i (tokens by depth, stable): does its run start here?
__device__ __forceinline__ bool run_head(const u32* __restrict__ sv, const u8* __restrict__ tkind, u64 i) {
    const u32 k = sv[i];
    return k == 0 || is_open(tkind[k - 1]);
}

// every token's container type; every open's close; the close of every run
// must match its open
__global__ void k_js_runs(const u32* __restrict__ sv, const u32* __restrict__ run_id, const u32* __restrict__ head_tok,
                          const u8* __restrict__ tkind, u64 T, u8* __restrict__ ctype, u32* __restrict__ close_of,
                          u32* __restrict__ flags) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < T;
         i += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u32 k = sv[i];
        const u32 h = head_tok[run_id[i]];  // the run's head token
        const u8 open = h == 0 ? kJNone : tkind[h - 1];
        ctype[k] = open == kJObj ? kCObj : open == kJArr ? kCArr : kCNone;
        const bool last = i + 1 == T || run_head(sv, tkind, i + 1);
        if (last && h != 0) {
            const u8 want = open == kJObj ? kJObjEnd : kJArrEnd;
            if (tkind[k] != want) atomicOr(flags, kFInvalid);
            close_of[h - 1] = k;
        }
    }
}

__device__ __forceinline__ bool is_key(const u8* __restrict__ tkind, const u8* __restrict__ ctype, u64 k) {
    return tkind[k] == kJStr && ctype[k] == kCObj && k > 0 && (tkind[k - 1] == kJObj || tkind[k - 1] == kJComma);
}

__global__ void k_js_grammar(const u8* __restrict__ tkind, const u8* __restrict__ ctype, const u32* __restrict__ depth,
                             u64 T, u32* __restrict__ flags) {
    for (u64 k = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; k < T;
         k += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u8 kt = tkind[k];
        bool ok;
        if (k == 0) {
            ok = value_start(kt);
        } else {
            ok = depth[k] >= 1;  // one value at depth 0: nothing after the root closes
            const u8 kp = tkind[k - 1];
            switch (kp) {
                case kJObj: ok = ok && (kt == kJStr || kt == kJObjEnd); break;
                case kJArr: ok = ok && (value_start(kt) || kt == kJArrEnd); break;
                case kJColon: ok = ok && value_start(kt); break;
                case kJComma: ok = ok && (ctype[k] == kCObj ? kt == kJStr : value_start(kt)); break;
                default:
                    if (is_key(tkind, ctype, k - 1)) ok = ok && kt == kJColon;
                    else ok = ok && (kt == kJComma || is_close(kt));  // after a value
            }
        }
        if (k + 1 == T) ok = ok && (T == 1 ? scalar_end(kt) : (is_close(kt) && depth[k] == 1));
        if (!ok) atomicOr(flags, kFInvalid);
    }
}

// ---- the manifest ---------------------------------------------------------

// get<int>() / get<int64_t>() of a number or boolean (x86-64 conversions of
// doubles, as the reference's build does them)
__device__ __forceinline__ i64 as_i64(u8 cls, i64 v) {
    if (cls == kVDouble) {
        const double d = __longlong_as_double(v);
        return (d >= -9223372036854775808.0 && d < 9223372036854775808.0) ? static_cast<i64>(d) : INT64_MIN;
    }
    return v;
}
__device__ __forceinline__ int32_t as_int(u8 cls, i64 v) {
    if (cls == kVDouble) {
        const double d = __longlong_as_double(v);
        return (d >= -2147483648.0 && d < 2147483648.0) ? static_cast<int32_t>(d) : INT32_MIN;
    }
    return static_cast<int32_t>(static_cast<u32>(static_cast<u64>(v)));
}
// a value nlohmann's arithmetic get<>() accepts
__device__ __forceinline__ bool number_ok(u8 kind, u8 cls, u32* flags) {
    if (!numeric(kind)) {
        atomicOr(flags, kFSemantic);
        return false;
    }
    if (cls == kVInexact) {
        atomicOr(flags, kFExotic);
        return false;
    }
    return true;
}
// a value iterated by a range-for: arrays; null iterates nothing; an
// object's values (key order) are outside this reader; a scalar iterates
// itself and fails at the next at()
__device__ __forceinline__ void iterable(u8 kind, u32* flags) {
    if (kind == kJObj) atomicOr(flags, kFExotic);
    else if (kind != kJArr && kind != kJNull) atomicOr(flags, kFSemantic);
}

struct Span {
    const u8* tkind;
    const u8* ctype;
    const u8* tname;
    const u32* depth;
    const u32* close_of;
    u64 lo, hi;  // the iterations array's tokens: (lo, hi) exclusive
};

// a member value at depth d (object) whose key is live: the last member of
// that name in its object, `slots` names per object
__device__ __forceinline__ int member_slot(u8 name, int level) {
    if (level == 3) return name == kNGroup ? 0 : name == kNPhase ? 1 : name == kNDevices ? 2 : -1;
    return name == kNCapacity ? 0 : name == kNSamples ? 1 : -1;
}

// last occurrence of each name per object (level 3: iterations; 6: packs)
__global__ void k_js_last(Span s, const u32* __restrict__ obj_of, const u8* __restrict__ dead, u32 level, int slots,
                          u32* __restrict__ last) {
    for (u64 k = s.lo + 1 + blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; k < s.hi;
         k += static_cast<u64>(gridDim.x) * blockDim.x) {
        if (s.depth[k] != level || !is_key(s.tkind, s.ctype, k) || (dead && dead[k - s.lo])) continue;
        const int sl = member_slot(s.tname[k], static_cast<int>(level));
        if (sl >= 0) atomicMax(&last[static_cast<u64>(obj_of[k - s.lo] - 1) * slots + sl], static_cast<u32>(k));
    }
}

// members not read (unknown names, earlier duplicates): their containers'
// token ranges marked for the mask scan
__global__ void k_js_mask(Span s, const u32* __restrict__ obj_of, const u8* __restrict__ dead, u32 level, int slots,
                          const u32* __restrict__ last, u64* __restrict__ marks, u32* __restrict__ n_marks) {
    for (u64 k = s.lo + 1 + blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; k < s.hi;
         k += static_cast<u64>(gridDim.x) * blockDim.x) {
        if (s.depth[k] != level || !is_key(s.tkind, s.ctype, k) || (dead && dead[k - s.lo])) continue;
        const int sl = member_slot(s.tname[k], static_cast<int>(level));
        const bool live = sl >= 0 && last[static_cast<u64>(obj_of[k - s.lo] - 1) * slots + sl] == k;
        const u64 v = k + 2;
        if (!live && is_open(s.tkind[v])) {
            atomicAdd(reinterpret_cast<unsigned long long*>(&marks[v - s.lo]), 1ull << 32);
            atomicAdd(reinterpret_cast<unsigned long long*>(&marks[s.close_of[v] + 1 - s.lo]), 1ull);
            atomicAdd(n_marks, 1u);
        }
    }
}

// every object has each member it reads
__global__ void k_js_present(const u32* __restrict__ last, u64 n, u32* __restrict__ flags) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<u64>(gridDim.x) * blockDim.x)
        if (last[i] == 0) atomicOr(flags, kFSemantic);
}

struct PlanOutG {
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

__global__ void k_js_scatter(Span s, const u8* __restrict__ dead, const u32* __restrict__ it_of,
                             const u64* __restrict__ dp_of, const u32* __restrict__ sm_of,
                             const u32* __restrict__ last3, const u32* __restrict__ last6, const u8* __restrict__ tcls,
                             const i64* __restrict__ tval, PlanOutG o, u32* __restrict__ flags) {
    for (u64 k = s.lo + 1 + blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; k < s.hi;
         k += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u64 r = k - s.lo;
        if (dead[r]) continue;
        const u32 d = s.depth[k];
        const u8 kt = s.tkind[k];
        if (!value_start(kt) || is_key(s.tkind, s.ctype, k)) continue;
        const u64 it = it_of[r], dv = dp_of[r] >> 32, pk = dp_of[r] & 0xffffffffull, sm = sm_of[r];
        switch (d) {
            case 2:  // an iteration (inclusive counts: it >= 1)
                if (kt != kJObj) atomicOr(flags, kFSemantic);
                else o.iter_dev_offsets[it - 1] = static_cast<int64_t>(dv);
                break;
            case 3: {  // a member of iteration it - 1 (key at k - 2)
                const int sl = member_slot(s.tname[k - 2], 3);
                if (sl < 0 || last3[(it - 1) * 3 + sl] != k - 2) break;
                if (sl == 0) {
                    if (number_ok(kt, tcls[k], flags)) o.iter_group[it - 1] = as_int(tcls[k], tval[k]);
                } else if (sl == 1) {
                    if (kt != kJStr) atomicOr(flags, kFSemantic);
                    else o.iter_phase[it - 1] = s.tname[k] == kNWarmup ? 1 : 0;
                } else {
                    iterable(kt, flags);
                }
                break;
            }
            case 4:  // a device of iteration it - 1 (inclusive: dv >= 1)
                iterable(kt, flags);
                o.dev_iter[dv - 1] = static_cast<int32_t>(it - 1);
                o.dev_pack_offsets[dv - 1] = static_cast<int64_t>(pk);
                break;
            case 5:  // a pack
                if (kt != kJObj) {
                    atomicOr(flags, kFSemantic);
                } else {
                    o.pack_member_offsets[pk - 1] = static_cast<int64_t>(sm);
                    o.pack_iter[pk - 1] = static_cast<int32_t>(it - 1);
                }
                break;
            case 6: {  // a member of pack pk - 1
                const int sl = member_slot(s.tname[k - 2], 6);
                if (sl < 0 || last6[(pk - 1) * 2 + sl] != k - 2) break;
                if (sl == 0) {
                    if (number_ok(kt, tcls[k], flags)) o.pack_capacity[pk - 1] = as_i64(tcls[k], tval[k]);
                } else {
                    iterable(kt, flags);
                }
                break;
            }
            case 7: {  // a sample: [id, length, ...] (s.at(0), s.at(1))
                if (kt != kJArr || s.tkind[k + 1] == kJArrEnd || s.tkind[k + 2] != kJComma) {
                    atomicOr(flags, kFSemantic);
                    break;
                }
                if (number_ok(s.tkind[k + 1], tcls[k + 1], flags) && number_ok(s.tkind[k + 3], tcls[k + 3], flags)) {
                    o.ids[sm - 1] = as_i64(tcls[k + 1], tval[k + 1]);
                    o.lens[sm - 1] = as_i64(tcls[k + 3], tval[k + 3]);
                }
                break;
            }
            default: break;
        }
    }
}

// same checks as plan_read.cu's k_plan_packs / k_plan_groups, any error a flag
__global__ void k_js_packs(const int64_t* __restrict__ moff, const int64_t* __restrict__ lens,
                           const int64_t* __restrict__ cap, u64 P, int64_t* __restrict__ total,
                           int64_t* __restrict__ att, u32* __restrict__ flags) {
    for (u64 p = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; p < P;
         p += static_cast<u64>(gridDim.x) * blockDim.x) {
        int64_t t = 0, a = 0;
        for (int64_t m = moff[p]; m < moff[p + 1]; ++m) {
            t += lens[m];
            a += lens[m] * lens[m];
        }
        total[p] = t;
        att[p] = a;
        if (t > cap[p]) atomicOr(flags, kFSemantic);
    }
}
__global__ void k_js_groups(const int32_t* __restrict__ g, u64 I, int32_t G, const int32_t* __restrict__ dev_iter,
                            u64 D, int32_t* __restrict__ dev_index, const int64_t* __restrict__ iter_dev_offsets,
                            u32* __restrict__ flags) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < I || i < D;
         i += static_cast<u64>(gridDim.x) * blockDim.x) {
        if (i < I && (g[i] < 0 || g[i] >= G)) atomicOr(flags, kFSemantic);
        if (i < D) dev_index[i] = static_cast<int32_t>(static_cast<i64>(i) - iter_dev_offsets[dev_iter[i]]);
    }
}

__global__ void k_js_maxd(const u32* __restrict__ d, u64 n, u32* __restrict__ out) {
    u32 m = 0;
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<u64>(gridDim.x) * blockDim.x)
        m = max(m, d[i]);
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31u) == 0) atomicMax(out, m);
}

__global__ void k_js_iota(int32_t* __restrict__ v, u64 n) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<u64>(gridDim.x) * blockDim.x)
        v[i] = static_cast<int32_t>(i);
}

// a few words about the root, in one read
struct RootInfo {
    u32 root_kind, iter_key, iter_val_kind, iter_pos, iter_close_pos, iter_val, iter_close;
};
__global__ void k_js_root(const u8* __restrict__ tkind, const u32* __restrict__ tpos, const u32* __restrict__ close_of,
                          const u32* __restrict__ iter_key, RootInfo* __restrict__ out) {
    RootInfo r{};
    r.root_kind = tkind[0];
    r.iter_key = *iter_key;
    if (r.iter_key) {
        const u32 v = r.iter_key + 2;
        r.iter_val = v;
        r.iter_val_kind = tkind[v];
        r.iter_pos = tpos[v];
        if (is_open(tkind[v])) {
            r.iter_close = close_of[v];
            r.iter_close_pos = tpos[r.iter_close];
        }
    }
    *out = r;
}

[[noreturn]] void fail_manifest(const char* text, u64 bytes, bool exotic) {
    const ManifestError e = manifest_error(std::string(text, bytes));
    if (e.code != 0) throw EngineError(e.code, e.msg);
    if (exotic)
        fail_validation(
            "plan manifest: the GPU reader reads arrays where the manifest iterates devices, packs and samples, and "
            "numbers it can convert exactly; this manifest has an object there or a number with more than 15 "
            "significant digits");
    throw EngineError(HBP_ERR_CUDA, "plan manifest: the GPU reader found an error the reference does not raise");
}

}  // namespace

void plan_from_json_general(Ctx& c, const char* text, u64 bytes, DevicePlan& dp, DevBuf<int64_t>& ids,
                            DevBuf<int64_t>& lens) {
    cudaStream_t s = c.stream;
    if (bytes >= (1ull << 32) - 64) fail_validation("plan manifest: the GPU reader takes manifests below 4 GiB");
    auto invalid_json = [&]() {
        const std::string what = json_parse_error_text(std::string(text, bytes));
        if (what.empty())
            throw EngineError(HBP_ERR_CUDA, "plan manifest: the GPU reader rejected text nlohmann accepts");
        fail_validation("bad plan manifest: " + what);
    };
    const unsigned char* ut = reinterpret_cast<const unsigned char*>(text);
    const u64 skip = (bytes >= 3 && ut[0] == 0xEF && ut[1] == 0xBB && ut[2] == 0xBF) ? 3 : 0;  // nlohmann skips a BOM

    DevBuf<unsigned char> t;
    upload_text(c, text, bytes, t);
    const u64 padded = t.n;
    DevBuf<u32> flags(1, s);
    flags.zero();

    // ---- 1-2: string states, tokens --------------------------------------
    u64 end = bytes;
    const u64 NB = std::max<u64>(1, (bytes + kJSpan - 1) / kJSpan);
    DevBuf<u32> bmap(NB, s), count(NB * kJB + 1, s);
    DevBuf<u64> offset(NB * kJB + 1, s);
    DevBuf<unsigned long long> nul(1, s);
    CUDA_CHECK(cudaMemsetAsync(nul.p, 0xff, sizeof(unsigned long long), s));
    LAUNCH_B("read.jmap", 1.0 * bytes, k_js_blockmap, NB, kJB, 0, s, t.p, padded, end, skip, bmap.p);
    LAUNCH(k_js_topmap, 1, 1024, 0, s, bmap.p, NB);
    LAUNCH_B("read.jcount", 1.0 * bytes, k_js_tokens<false>, NB, kJB, 0, s, t.p, padded, end, skip, bmap.p, count.p,
             nullptr, nul.p, nullptr, nullptr);
    const u64 first_nul = read_scalar(c, nul.p);
    if (first_nul < end) {  // input ends at a NUL outside a string: count again up to it
        end = first_nul;
        LAUNCH_B("read.jcount", 1.0 * bytes, k_js_tokens<false>, NB, kJB, 0, s, t.p, padded, end, skip, bmap.p,
                 count.p, nullptr, nul.p, nullptr, nullptr);
    }
    const i64 NC = static_cast<i64>(NB * kJB);
    {
        const u32* cp = count.p;
        u64* op = offset.p;
        scan_exclusive<u64>(
            NC + 1, [=] __device__(i64 i) { return i < NC ? static_cast<u64>(cp[i]) : 0ull; },
            [=] __device__(i64 i, u64 v) { op[i] = v; }, s, c.scan, "scan.read_tok");
    }
    const u64 T = read_vector(c, offset.p + NC, 1)[0];
    if (T == 0) invalid_json();
    DevBuf<u32> tpos(T + 1, s);
    DevBuf<u8> tkind(T + 4, s);  // kJNone past the end: the sample check reads up to k + 3
    CUDA_CHECK(cudaMemsetAsync(tkind.p, 0, T + 4, s));
    LAUNCH_B("read.jemit", 1.0 * bytes, k_js_tokens<true>, NB, kJB, 0, s, t.p, padded, end, skip, bmap.p, nullptr,
             offset.p, nullptr, tpos.p, tkind.p);
    bmap.release();
    count.release();
    offset.release();

    // ---- 3: token text ----------------------------------------------------
    DevBuf<u8> tname(T + 4, s), tcls(T + 4, s);
    DevBuf<i64> tval(T + 4, s);
    LAUNCH(k_js_text, grid_for(T, 256, 148u * 16u), 256, 0, s, t.p, end, tpos.p, tkind.p, T, tname.p, tcls.p, tval.p,
           flags.p);

    // ---- 4: depth, runs by depth, grammar ---------------------------------
    DevBuf<u32> depth(T + 4, s);
    DevBuf<u32> maxd(2, s);
    maxd.zero();
    {
        const u8* kp = tkind.p;
        u32* dp_ = depth.p;
        u32* fl = flags.p;
        const i64 NT = static_cast<i64>(T);
        scan_exclusive<u64>(
            NT + 1,
            [=] __device__(i64 i) {
                if (i >= NT) return 0ull;
                return is_open(kp[i]) ? (1ull << 32) : is_close(kp[i]) ? 1ull : 0ull;
            },
            [=] __device__(i64 i, u64 v) {
                const i64 d = static_cast<i64>(v >> 32) - static_cast<i64>(v & 0xffffffffull);
                if (i >= NT) {
                    if (d != 0) atomicOr(fl, kFInvalid);  // unbalanced
                    return;
                }
                if (d < 0 || (d == 0 && is_close(kp[i]))) {
                    atomicOr(fl, kFInvalid);
                    dp_[i] = 0;
                    return;
                }
                dp_[i] = static_cast<u32>(d);
            },
            s, c.scan, "scan.read_depth");
    }
    LAUNCH(k_js_maxd, grid_for(T, 256, 148u * 8u), 256, 0, s, depth.p, T, maxd.p);
    const auto fm = read_vector(c, flags.p, 1);
    if (fm[0] & kFInvalid) invalid_json();
    const u32 max_depth = read_vector(c, maxd.p, 1)[0];
    DevBuf<u8> ctype(T + 4, s);
    DevBuf<u32> close_of(T + 4, s);
    {
        DevBuf<u32> sk(T, s), sv(T, s), run_id(T, s), head_tok(T, s);
        CUDA_CHECK(cudaMemcpyAsync(sk.p, depth.p, sizeof(u32) * T, cudaMemcpyDeviceToDevice, s));
        for_each_index(c, T, [sv = sv.p] __device__(u64 i) { sv[i] = static_cast<u32>(i); });
        int bits = 1;
        while ((1ull << bits) <= max_depth) ++bits;
        radix_sort_pairs(c, sk.p, sv.p, static_cast<i64>(T), bits, false);
        sk.release();
        const u32* svp = sv.p;
        const u8* kp = tkind.p;
        u32* rid = run_id.p;
        u32* ht = head_tok.p;
        // run index of every sorted position (heads counted inclusively), and
        // the head token of every run
        scan_exclusive<u64>(
            static_cast<i64>(T), [=] __device__(i64 i) { return run_head(svp, kp, static_cast<u64>(i)) ? 1ull : 0ull; },
            [=] __device__(i64 i, u64 v) {
                if (run_head(svp, kp, static_cast<u64>(i))) {
                    ht[v] = svp[i];
                    rid[i] = static_cast<u32>(v);
                } else {
                    rid[i] = static_cast<u32>(v - 1);
                }
            },
            s, c.scan, "scan.read_runs");
        LAUNCH(k_js_runs, grid_for(T, 256, 148u * 16u), 256, 0, s, sv.p, run_id.p, head_tok.p, tkind.p, T, ctype.p,
               close_of.p, flags.p);
    }
    LAUNCH(k_js_grammar, grid_for(T, 256, 148u * 16u), 256, 0, s, tkind.p, ctype.p, depth.p, T, flags.p);
    // the live "iterations" member of the root (last of that name)
    DevBuf<u32> iter_key(1, s);
    iter_key.zero();
    {
        const u8* kp = tkind.p;
        const u8* cp = ctype.p;
        const u8* np = tname.p;
        const u32* dp_ = depth.p;
        u32* ik = iter_key.p;
        for_each_index(c, T, [=] __device__(u64 k) {
            if (dp_[k] == 1 && np[k] == kNIterations && is_key(kp, cp, k)) atomicMax(ik, static_cast<u32>(k));
        });
    }
    DevBuf<RootInfo> root(1, s);
    LAUNCH(k_js_root, 1, 1, 0, s, tkind.p, tpos.p, close_of.p, iter_key.p, root.p);
    const u32 f1 = read_vector(c, flags.p, 1)[0];
    if (f1 & kFInvalid) invalid_json();
    const RootInfo ri = read_vector(c, root.p, 1)[0];

    // ---- 5: the header on the host, the iterations on the device ------------
    if (ri.root_kind != kJObj || ri.iter_key == 0) fail_manifest(text, bytes, false);  // fails in the header
    std::string head;
    const bool has_array = ri.iter_val_kind == kJArr;
    if (ri.iter_val_kind == kJArr || ri.iter_val_kind == kJObj) {
        head.reserve(ri.iter_pos + 2 + (end - ri.iter_close_pos));
        head.append(text, ri.iter_pos);
        head.append("[]");
        head.append(text + ri.iter_close_pos + 1, end - ri.iter_close_pos - 1);
    } else if (ri.iter_val_kind == kJNull) {
        head.assign(text, end);
    } else {
        fail_manifest(text, bytes, false);  // a scalar: it_obj.at() fails
    }
    if (ri.iter_val_kind == kJObj) fail_manifest(text, bytes, true);
    ManifestHeader h;
    const ManifestError he = manifest_header(head, h);
    if (he.code != 0) throw EngineError(he.code, he.msg);
    dp.device_count = h.device_count;
    dp.seed = h.seed;
    dp.groups = h.groups;
    dp.l_best = h.l_best;
    dp.l_max = h.l_max;

    const u64 lo = ri.iter_val, hi = has_array ? ri.iter_close : ri.iter_val;
    const u64 R = hi > lo ? hi - lo : 0;  // tokens lo .. hi inclusive are indexed r = k - lo
    Span sp{tkind.p, ctype.p, tname.p, depth.p, close_of.p, lo, hi};
    u64 I = 0, D = 0, P = 0, M = 0;
    DevBuf<u8> dead(R + 2, s);
    DevBuf<u32> it_of(R + 2, s), sm_of(R + 2, s);
    DevBuf<u64> dp_of(R + 2, s);
    DevBuf<u32> last3, last6;
    if (R > 1) {
        CUDA_CHECK(cudaMemsetAsync(dead.p, 0, R + 2, s));
        const u8* kp = tkind.p;
        const u8* cp = ctype.p;
        const u32* dpp = depth.p;
        u8* de = dead.p;
        const i64 NR = static_cast<i64>(R);
        // iterations before and at every token (depth-2 values)
        {
            u32* io = it_of.p;
            scan_exclusive<u64>(
                NR + 1,
                [=] __device__(i64 r) {
                    const u64 k = lo + static_cast<u64>(r);
                    return (r > 0 && r < NR && dpp[k] == 2 && value_start(kp[k])) ? 1ull : 0ull;
                },
                [=] __device__(i64 r, u64 v) {
                    const u64 k = lo + static_cast<u64>(r);
                    io[r] = static_cast<u32>(v + ((r > 0 && r < NR && dpp[k] == 2 && value_start(kp[k])) ? 1 : 0));
                },
                s, c.scan, "scan.read_it");
        }
        I = read_vector(c, it_of.p + R, 1)[0];
        auto mask_pass = [&](u32 level, int slots, DevBuf<u32>& last, const u32* obj_of, u64 n_obj) {
            last.alloc(n_obj * slots + 1, s);
            last.zero();
            if (!n_obj) return;
            LAUNCH(k_js_last, grid_for(R, 256, 148u * 16u), 256, 0, s, sp, obj_of, de, level, slots, last.p);
            LAUNCH(k_js_present, grid_for(n_obj * slots, 256), 256, 0, s, last.p, n_obj * slots, flags.p);
            DevBuf<u64> marks(R + 2, s);
            DevBuf<u32> nm(1, s);
            marks.zero();
            nm.zero();
            LAUNCH(k_js_mask, grid_for(R, 256, 148u * 16u), 256, 0, s, sp, obj_of, de, level, slots, last.p, marks.p,
                   nm.p);
            if (read_scalar(c, nm.p) == 0) return;
            const u64* mk = marks.p;
            scan_exclusive<u64>(
                NR + 1, [=] __device__(i64 r) { return mk[r]; },
                [=] __device__(i64 r, u64 v) {
                    const u64 w = v + mk[r];  // inclusive: opened - closed ranges
                    if ((w >> 32) > (w & 0xffffffffull)) de[r] = 1;
                },
                s, c.scan, "scan.read_mask");
        };
        mask_pass(3, 3, last3, it_of.p, I);
        // devices and packs before and at every live token
        {
            u64* dq = dp_of.p;
            auto one = [=] __device__(i64 r) -> u64 {
                const u64 k = lo + static_cast<u64>(r);
                if (r == 0 || r >= NR || de[r] || !value_start(kp[k])) return 0ull;
                if (dpp[k] == 4) return 1ull << 32;
                if (dpp[k] == 5) return 1ull;
                return 0ull;
            };
            scan_exclusive<u64>(
                NR + 1, one, [=] __device__(i64 r, u64 v) { dq[r] = v + one(r); }, s, c.scan, "scan.read_dp");
        }
        const u64 dpt = read_vector(c, dp_of.p + R, 1)[0];
        D = dpt >> 32;
        P = dpt & 0xffffffffull;
        // pack members: packs are the objects of level 6 (pack index = low word)
        {
            DevBuf<u32> pk_of(R + 2, s);
            u32* po = pk_of.p;
            const u64* dq = dp_of.p;
            for_each_index(c, R + 1, [=] __device__(u64 r) { po[r] = static_cast<u32>(dq[r] & 0xffffffffull); });
            mask_pass(6, 2, last6, pk_of.p, P);
        }
        // samples before and at every live token
        {
            u32* so = sm_of.p;
            auto one = [=] __device__(i64 r) -> u64 {
                const u64 k = lo + static_cast<u64>(r);
                return (r > 0 && r < NR && !de[r] && dpp[k] == 7 && value_start(kp[k])) ? 1ull : 0ull;
            };
            scan_exclusive<u64>(
                NR + 1, one, [=] __device__(i64 r, u64 v) { so[r] = static_cast<u32>(v + one(r)); }, s, c.scan,
                "scan.read_sm");
        }
        M = read_vector(c, sm_of.p + R, 1)[0];
        (void)cp;
    }
    if (I >= (1ull << 31) || D >= (1ull << 31) || P >= (1ull << 31) || M >= (1ull << 31))
        fail_validation("plan manifest: more than 2^31 iterations, devices, packs or samples");
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
    CUDA_CHECK(cudaMemsetAsync(ids.p, 0, sizeof(int64_t) * (M + 1), s));
    CUDA_CHECK(cudaMemsetAsync(lens.p, 0, sizeof(int64_t) * (M + 1), s));
    {  // the CSR ends
        int64_t* a = dp.iter_dev_offsets.p + I;
        int64_t* b = dp.dev_pack_offsets.p + D;
        int64_t* m = dp.pack_member_offsets.p + P;
        const int64_t d_ = static_cast<int64_t>(D), p_ = static_cast<int64_t>(P), m_ = static_cast<int64_t>(M);
        for_each_index(c, 1, [=] __device__(u64) {
            *a = d_;
            *b = p_;
            *m = m_;
        });
    }
    if (R > 1) {
        PlanOutG o{dp.iter_group.p, dp.iter_phase.p, dp.iter_dev_offsets.p, dev_iter.p, dp.dev_pack_offsets.p,
                   dp.pack_capacity.p, pack_iter.p, dp.pack_member_offsets.p, ids.p, lens.p};
        LAUNCH_B("read.jscatter", 16.0 * R, k_js_scatter, grid_for(R, 256, 148u * 16u), 256, 0, s, sp, dead.p,
                 it_of.p, dp_of.p, sm_of.p, last3.p, last6.p, tcls.p, tval.p, o, flags.p);
    }
    if (P)
        LAUNCH(k_js_packs, grid_for(P, 256), 256, 0, s, dp.pack_member_offsets.p, lens.p, dp.pack_capacity.p, P,
               dp.pack_total.p, dp.pack_attention.p, flags.p);
    if (I || D)
        LAUNCH(k_js_groups, grid_for(std::max(I, D), 256), 256, 0, s, dp.iter_group.p, I,
               static_cast<int32_t>(dp.groups.size()), dev_iter.p, D, dp.dev_index.p, dp.iter_dev_offsets.p, flags.p);
    if (M) LAUNCH(k_js_iota, grid_for(M, 256), 256, 0, s, dp.member_index.p, M);
    const u32 f2 = read_vector(c, flags.p, 1)[0];
    if (f2 & (kFSemantic | kFExotic)) fail_manifest(text, bytes, (f2 & kFExotic) != 0);
}

}  // namespace hbp_b200
