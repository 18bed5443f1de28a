// ez_rng.cuh — counter-based random streams for hit-and-run walks.
//
// EZ_RNG_COUNTER reproduces the reference stream exactly
// (corridor/seeding.py:27-60): h = mix(mix(mix(0 ^ seed) ^ walk) ^ (step*64 +
// slot)), uniform ((h >> 11) + 0.5) * 2^-53, normal = inverse normal CDF of
// that uniform.  The first two mixes depend only on (seed, walk) and are
// hoisted out of the walk loop, so every draw costs one splitmix round.
//
// EZ_RNG_PHILOX is Philox4x32-10 keyed by the seed with counter (walk lo,
// walk hi, step, slot group); normals come from fp32 Box-Muller pairs.
#pragma once

#include <cstdint>

namespace ez {

constexpr uint64_t kSeedStep = 1ull << 32;  // seeding.py:23 SEED_STEP

__device__ __forceinline__ uint64_t splitmix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// hash prefix of walk `walk` under master seed `seed`
__device__ __forceinline__ uint64_t walk_key(uint64_t seed, uint64_t walk) {
    return splitmix(splitmix(seed) ^ walk);
}

__device__ __forceinline__ double u53(uint64_t h) {
    return (static_cast<double>(h >> 11) + 0.5) * 0x1p-53;
}

__device__ __forceinline__ double counter_uniform(uint64_t key, uint64_t step, uint32_t slot) {
    return u53(splitmix(key ^ (step * 64ull + slot)));
}

__device__ __forceinline__ double counter_normal(uint64_t key, uint64_t step, uint32_t slot) {
    return normcdfinv(counter_uniform(key, step, slot));
}

struct Philox4 {
    uint32_t x, y, z, w;
};

__device__ __forceinline__ Philox4 philox(Philox4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = Philox4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

__device__ __forceinline__ Philox4 philox_draw(uint64_t seed, uint64_t walk, uint32_t step, uint32_t group) {
    return philox(Philox4{static_cast<uint32_t>(walk), static_cast<uint32_t>(walk >> 32), step, group},
                  static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
}

__device__ __forceinline__ double philox_u53(uint32_t a, uint32_t b) {
    const uint64_t h = (static_cast<uint64_t>(a) << 32) | b;
    return u53(h);
}

// two standard normals from two 32-bit words (fp32 Box-Muller)
__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, float& n0, float& n1) {
    const float u1 = (static_cast<float>(a >> 8) + 0.5f) * 0x1p-24f;  // (0, 1)
    const float u2 = static_cast<float>(b >> 8) * 0x1p-24f;           // [0, 1)
    const float r = sqrtf(-2.0f * logf(u1));
    float s, c;
    sincospif(2.0f * u2, &s, &c);
    n0 = r * c;
    n1 = r * s;
}

constexpr uint32_t kPhiloxSeedStep = 0xFFFFFFFFu;  // step tag of the walk-start draw

}  // namespace ez
