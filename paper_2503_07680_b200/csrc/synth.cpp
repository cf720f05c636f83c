// synth.cpp — synthetic corpora, the reference generator restated for the
// host (src/ingest.cpp:279-329; Python binding bindings/py_hbp.cpp:80-97).
//
// Input generation only (never on the timed path). The reference draws the
// short stream then the long stream sequentially; every draw of a SplitMix64
// stream is a pure function of its index (rng.cuh), so chunks are generated
// on all host threads. Box-Muller consumes two draws per pair of normals and
// rejects u1 == 0 (probability 2^-53 per pair); uniform_int rejects with
// probability < span / 2^64. If any chunk sees a rejection the whole stream
// is regenerated sequentially, so the output is always exactly the
// reference's (same libm: glibc exp/log/sin/cos/sqrt).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/hbp_b200.h"
#include "rng.cuh"

namespace {

using hbp_b200::derive_seed;
using hbp_b200::splitmix_draw;

struct Dist {
    int family = 0;  // 0 constant 1 uniform 2 normal 3 lognormal
    double a = 0, b = 0;
};

struct Bad : std::runtime_error {
    using std::runtime_error::runtime_error;
};

Dist parse(const std::string& text) {
    std::vector<std::string> parts;
    size_t start = 0;
    while (start <= text.size()) {
        const size_t c = text.find(':', start);
        if (c == std::string::npos) {
            if (start < text.size()) parts.push_back(text.substr(start));
            break;
        }
        parts.push_back(text.substr(start, c - start));
        start = c + 1;
    }
    if (parts.empty()) throw Bad("empty distribution spec");
    Dist d;
    size_t want;
    if (parts[0] == "constant") d.family = 0, want = 2;
    else if (parts[0] == "uniform") d.family = 1, want = 3;
    else if (parts[0] == "normal") d.family = 2, want = 3;
    else if (parts[0] == "lognormal") d.family = 3, want = 3;
    else throw Bad("unknown distribution family: " + parts[0]);
    static const char* need[] = {"constant needs 1 parameter", "uniform needs 2 parameters",
                                 "normal needs 2 parameters", "lognormal needs 2 parameters"};
    if (parts.size() != want) throw Bad(need[d.family]);
    auto num = [&](size_t i) {
        try {
            return std::stod(parts.at(i));
        } catch (const std::exception&) {
            throw Bad("bad distribution parameter in '" + text + "'");
        }
    };
    d.a = num(1);
    if (want == 3) d.b = num(2);
    switch (d.family) {
        case 0:
            if (d.a < 1.0) throw Bad("constant length must be >= 1");
            break;
        case 1:
            if (d.a < 1.0 || d.b < d.a) throw Bad("uniform bounds must satisfy 1 <= low <= high");
            break;
        case 2:
            if (d.b < 0.0) throw Bad("normal stddev must be >= 0");
            break;
        default:
            if (d.b < 0.0) throw Bad("lognormal sigma must be >= 0");
    }
    return d;
}

int64_t clip(double v, int64_t max_length) {
    int64_t len = static_cast<int64_t>(std::llround(v));
    if (len < 1) len = 1;
    if (len > max_length) len = max_length;
    return len;
}

// Sequential generator: the reference's exact loop (ingest.cpp:279-300).
struct SeqRng {
    uint64_t s;
    bool have = false;
    double spare = 0;
    uint64_t next() {
        uint64_t z = (s += hbp_b200::kGamma);
        return hbp_b200::splitmix_mix(z);
    }
    double dbl() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    int64_t uni(int64_t lo, int64_t hi) {
        const uint64_t span = static_cast<uint64_t>(hi - lo) + 1;
        if (span == 0) return static_cast<int64_t>(next());
        const uint64_t limit = UINT64_MAX - UINT64_MAX % span;
        uint64_t v;
        do v = next();
        while (v >= limit);
        return lo + static_cast<int64_t>(v % span);
    }
    double normal() {
        if (have) {
            have = false;
            return spare;
        }
        double u1, u2;
        do u1 = dbl();
        while (u1 <= 0.0);
        u2 = dbl();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double th = 6.283185307179586476925286766559 * u2;
        spare = r * std::sin(th);
        have = true;
        return r * std::cos(th);
    }
};

void gen_sequential(const Dist& d, uint64_t seed, int64_t count, int64_t max_length, int64_t* out) {
    SeqRng r{seed};
    for (int64_t i = 0; i < count; ++i) {
        double v = 1.0;
        switch (d.family) {
            case 0: v = d.a; break;
            case 1: v = static_cast<double>(r.uni(static_cast<int64_t>(d.a), static_cast<int64_t>(d.b))); break;
            case 2: v = d.a + d.b * r.normal(); break;
            default: v = std::exp(d.a + d.b * r.normal());
        }
        out[i] = clip(v, max_length);
    }
}

// Counter-based generation of samples [lo, hi) assuming no rejection
// anywhere before; returns false if a rejection is seen in the chunk.
bool gen_chunk(const Dist& d, uint64_t seed, int64_t lo, int64_t hi, int64_t max_length, int64_t* out) {
    if (d.family == 0) {
        for (int64_t i = lo; i < hi; ++i) out[i] = clip(d.a, max_length);
        return true;
    }
    if (d.family == 1) {
        const int64_t a = static_cast<int64_t>(d.a), b = static_cast<int64_t>(d.b);
        const uint64_t span = static_cast<uint64_t>(b - a) + 1;
        const uint64_t limit = span == 0 ? 0 : UINT64_MAX - UINT64_MAX % span;
        for (int64_t i = lo; i < hi; ++i) {
            const uint64_t v = splitmix_draw(seed, static_cast<uint64_t>(i) + 1);
            if (span != 0 && v >= limit) return false;
            const int64_t x = span == 0 ? static_cast<int64_t>(v) : a + static_cast<int64_t>(v % span);
            out[i] = clip(static_cast<double>(x), max_length);
        }
        return true;
    }
    // normals: pair m = i / 2 uses draws 2m+1 (u1) and 2m+2 (u2)
    for (int64_t i = lo; i < hi; ++i) {
        const uint64_t m = static_cast<uint64_t>(i) / 2;
        const uint64_t v1 = splitmix_draw(seed, 2 * m + 1);
        if ((v1 >> 11) == 0) return false;
        const double u1 = static_cast<double>(v1 >> 11) * 0x1.0p-53;
        const double u2 = static_cast<double>(splitmix_draw(seed, 2 * m + 2) >> 11) * 0x1.0p-53;
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double th = 6.283185307179586476925286766559 * u2;
        const double z = (i % 2 == 0) ? r * std::cos(th) : r * std::sin(th);
        const double v = d.family == 2 ? d.a + d.b * z : std::exp(d.a + d.b * z);
        out[i] = clip(v, max_length);
    }
    return true;
}

void gen_stream(const Dist& d, uint64_t seed, int64_t count, int64_t max_length, int64_t* out) {
    if (count <= 0) return;
    unsigned threads = std::thread::hardware_concurrency();
    if (threads == 0) threads = 1;
    if (count < 200000) threads = 1;
    int64_t per = (count + threads - 1) / threads;
    per += per & 1;  // chunks start on an even sample (normal pairs)
    std::vector<char> ok(threads, 1);
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < threads; ++t) {
        const int64_t lo = static_cast<int64_t>(t) * per, hi = std::min<int64_t>(count, lo + per);
        if (lo >= hi) break;
        pool.emplace_back([&, t, lo, hi] { ok[t] = gen_chunk(d, seed, lo, hi, max_length, out) ? 1 : 0; });
    }
    for (auto& th : pool) th.join();
    for (char o : ok)
        if (!o) {
            gen_sequential(d, seed, count, max_length, out);
            return;
        }
}

}  // namespace

extern "C" int hbp_synth_lengths(int64_t count, const char* short_dist, double long_fraction, const char* long_dist,
                                 int64_t max_length, uint64_t seed, int64_t* out_lengths, char* err, int errlen) {
    try {
        const Dist sd = parse(short_dist ? short_dist : "");
        const Dist ld = (long_dist && long_dist[0]) ? parse(long_dist) : sd;
        if (count < 1) throw Bad("synth count must be >= 1");
        if (long_fraction < 0.0 || long_fraction > 1.0) throw Bad("long_fraction must lie in [0, 1]");
        if (max_length < 1) throw Bad("max_length must be >= 1");
        const int64_t long_count = static_cast<int64_t>(std::llround(static_cast<double>(count) * long_fraction));
        const int64_t short_count = count - long_count;
        gen_stream(sd, derive_seed(seed, "synth-short"), short_count, max_length, out_lengths);
        gen_stream(ld, derive_seed(seed, "synth-long"), long_count, max_length, out_lengths + short_count);
        return HBP_OK;
    } catch (const std::exception& e) {
        if (err && errlen > 0) {
            std::strncpy(err, e.what(), static_cast<size_t>(errlen) - 1);
            err[errlen - 1] = '\0';
        }
        return HBP_ERR_VALIDATION;
    }
}
