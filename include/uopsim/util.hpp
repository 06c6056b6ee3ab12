#pragma once
// Small integer/RNG helpers shared by the host library.
//
// Bit-compatibility contract (parity): splitmix64 / unit_float / fnv1a must
// produce exactly the reference's streams (reference include/uopsim/util.hpp:15-33),
// because synthetic weights and inputs are keyed by `seed ^ fnv1a(tensor name)`
// (reference workload.cpp:417) and the oracle compares against the same arrays.
// Note: the reference comment says "[-1, 1)" but the arithmetic yields [-1, 3)
// (SURVEY finding 8); we reproduce the arithmetic, not the comment.

#include <cstdint>
#include <cstring>
#include <string_view>

namespace uopsim {

template <typename T>
constexpr T ceil_div(T a, T b) {
    return (a + b - 1) / b;
}

inline uint64_t splitmix64(uint64_t& state) {
    state += 0x9e3779b97f4a7c15ULL;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// 24 high bits -> [0, 2) step 2^-23, times 2, minus 1 => [-1, 3).
inline float unit_float(uint64_t& state) {
    const double scaled = static_cast<double>(splitmix64(state) >> 40) * (1.0 / 8388608.0);
    return static_cast<float>(scaled) * 2.0f - 1.0f;
}

inline uint64_t fnv1a(std::string_view s, uint64_t h = 0xcbf29ce484222325ULL) {
    for (unsigned char c : s) h = (h ^ c) * 0x100000001b3ULL;
    return h;
}

// bf16 helpers (round-to-nearest-even, NaN preserved as quiet NaN).
inline uint16_t f32_to_bf16_bits(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) return static_cast<uint16_t>((u >> 16) | 0x40);
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}
inline float bf16_bits_to_f32(uint16_t b) {
    uint32_t u = static_cast<uint32_t>(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}
inline float round_bf16(float f) { return bf16_bits_to_f32(f32_to_bf16_bits(f)); }

}  // namespace uopsim
