// philox.h — the library's counter-based generator for fastlsh_params_create / keys_create.
//
// Philox4x32-10 (Salmon et al., SC'11) with key = (seed lo32, seed hi32), counter =
// (j, i, stream, 0). Streams: 1 sampled indices, 2 Gaussian coefficients, 3 offsets b,
// 4 key multipliers (reading R11). Each value is addressed by its (i, j) and is
// independent of generation order, so every rank regenerates identical params from the seed.
#pragma once
#include <cmath>
#include <cstdint>

namespace fastlsh {

struct Philox4 {
    uint32_t v[4];
};

inline Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint64_t seed) {
    uint32_t k0 = (uint32_t)(seed & 0xffffffffu), k1 = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        if (r != 9) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    }
    return Philox4{{c0, c1, c2, c3}};
}

enum : uint32_t { kStreamIdx = 1, kStreamA = 2, kStreamB = 3, kStreamKeys = 4 };

inline uint64_t u64_of(uint32_t lo, uint32_t hi) { return ((uint64_t)hi << 32) | lo; }

// idx = floor(u * n / 2^64): uniform on [0, n) (bias < n / 2^64).
inline int32_t draw_index(uint64_t seed, uint32_t i, uint32_t j, uint32_t n) {
    Philox4 r = philox4x32_10(j, i, kStreamIdx, 0, seed);
    unsigned __int128 prod = (unsigned __int128)u64_of(r.v[0], r.v[1]) * n;
    return (int32_t)(uint64_t)(prod >> 64);
}

// Box–Muller (cos branch) in double from two 53-bit uniforms, rounded to f32.
inline float draw_gaussian(uint64_t seed, uint32_t i, uint32_t j) {
    Philox4 r = philox4x32_10(j, i, kStreamA, 0, seed);
    double u1 = ((double)(u64_of(r.v[0], r.v[1]) >> 11) + 1.0) * 0x1p-53;
    double u2 = (double)(u64_of(r.v[2], r.v[3]) >> 11) * 0x1p-53;
    return (float)(std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2));
}

// b = f32(w * u53) clamped into [0, w) (reading R1).
inline float draw_offset(uint64_t seed, uint32_t i, float w) {
    Philox4 r = philox4x32_10(0, i, kStreamB, 0, seed);
    double u = (double)(u64_of(r.v[0], r.v[1]) >> 11) * 0x1p-53;
    float b = (float)((double)w * u);
    if (b >= w) b = std::nextafter(w, 0.0f);
    return b;
}

constexpr uint64_t kP61 = (1ull << 61) - 1;

inline uint64_t draw_key_multiplier(uint64_t seed, uint32_t l, uint32_t j) {
    Philox4 r = philox4x32_10(j, l, kStreamKeys, 0, seed);
    uint64_t x = u64_of(r.v[0], r.v[1]) >> 3;
    return x == kP61 ? 0 : x;
}

}  // namespace fastlsh
