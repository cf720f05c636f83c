// rng.cuh — the reference's SplitMix64 stream as a counter-based generator.
//
// Rng(seed).next_u64() (reference include/hbp/rng.hpp:18-23) advances the
// state by the golden gamma and mixes it, so draw k (1-based) of a stream is
// a pure function mix(seed + k * gamma): every draw of a Fisher-Yates
// shuffle can be computed independently on its own thread. derive_seed
// (rng.hpp:80-95) hashes the tag with FNV-1a and one splitmix round.
#pragma once

#include <cstdint>
#include <string_view>

#if defined(__CUDACC__)
#define HBP_HD __host__ __device__ __forceinline__
#else
#define HBP_HD inline
#endif

namespace hbp_b200 {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

HBP_HD uint64_t splitmix_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// k-th draw (k >= 1) of Rng(seed)
HBP_HD uint64_t splitmix_draw(uint64_t seed, uint64_t k) {
    return splitmix_mix(seed + k * kGamma);
}

inline uint64_t derive_seed(uint64_t seed, std::string_view tag) {
    uint64_t h = 0xcbf29ce484222325ULL ^ seed;
    for (const char c : tag) {
        h ^= static_cast<uint8_t>(c);
        h *= 0x100000001b3ULL;
    }
    return splitmix_mix(h);
}

inline uint64_t derive_seed(uint64_t seed, std::string_view tag, uint64_t index) {
    return derive_seed(seed ^ (kGamma * (index + 1)), tag);
}

}  // namespace hbp_b200
