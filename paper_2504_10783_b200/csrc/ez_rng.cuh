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

// Inverse normal CDF in fp64: Wichura's AS241 (PPND16).  Its central
// rational (|p - 0.5| <= 0.425, 85% of the draws) needs no transcendental; the
// tails take one log and one sqrt.  Against scipy.special.ndtri (the
// reference's, cpoly.py:164 via seeding.py:58-60) the relative error is at
// most 1.2e-15 on 5e6 reference-stream uniforms (checked in numpy).  The
// coefficients live in constant memory so every DFMA reads its operand from
// the constant bank (as literals each double costs two UMOVs).
__constant__ double kAs241[6][8] = {
    {3.3871328727963666080e0, 1.3314166789178437745e+2, 1.9715909503065514427e+3, 1.3731693765509461125e+4,
     4.5921953931549871457e+4, 6.7265770927008700853e+4, 3.3430575583588128105e+4, 2.5090809287301226727e+3},
    {1.0, 4.2313330701600911252e+1, 6.8718700749205790830e+2, 5.3941960214247511077e+3, 2.1213794301586595867e+4,
     3.9307895800092710610e+4, 2.8729085735721942674e+4, 5.2264952788528545610e+3},
    {1.42343711074968357734e0, 4.63033784615654529590e0, 5.76949722146069140550e0, 3.64784832476320460504e0,
     1.27045825245236838258e0, 2.41780725177450611770e-1, 2.27238449892691845833e-2, 7.74545014278341407640e-4},
    {1.0, 2.05319162663775882187e0, 1.67638483018380384940e0, 6.89767334985100004550e-1,
     1.48103976427480074590e-1, 1.51986665636164571966e-2, 5.47593808499534494600e-4, 1.05075007164441684324e-9},
    {6.65790464350110377720e0, 5.46378491116411436990e0, 1.78482653991729133580e0, 2.96560571828504891230e-1,
     2.65321895265761230930e-2, 1.24266094738807843860e-3, 2.71155556874348757815e-5, 2.01033439929228813265e-7},
    {1.0, 5.99832206555887937690e-1, 1.36929880922735805310e-1, 1.48753612908506148525e-2,
     7.86869131145613259100e-4, 1.84631831751005468180e-5, 1.42151175831644588870e-7, 2.04426310338993978564e-15}};

__device__ __forceinline__ double as241_poly(int set, double r) {
    double v = kAs241[set][7];
#pragma unroll
    for (int k = 6; k >= 0; --k) v = fma(v, r, kAs241[set][k]);
    return v;
}

__device__ __forceinline__ bool as241_central(double p) { return fabs(p - 0.5) <= 0.425; }

__device__ __forceinline__ double as241_center(double p) {
    const double q = p - 0.5;
    const double r = 0.180625 - q * q;
    // a correctly rounded reciprocal and two products instead of a division
    // (one more rounding, within the approximation's few ulps)
    return q * as241_poly(0, r) * __drcp_rn(as241_poly(1, r));
}

__device__ __forceinline__ double as241_tail(double p) {
    const double q = p - 0.5;
    double r = sqrt(-log(q < 0.0 ? p : 1.0 - p));
    double v;
    if (r <= 5.0) {
        r -= 1.6;
        v = as241_poly(2, r) / as241_poly(3, r);
    } else {
        r -= 5.0;
        v = as241_poly(4, r) / as241_poly(5, r);
    }
    return q < 0.0 ? -v : v;
}

__device__ __forceinline__ double ndtri_as241(double p) { return as241_central(p) ? as241_center(p) : as241_tail(p); }

__device__ __forceinline__ double counter_normal(uint64_t key, uint64_t step, uint32_t slot) {
    return ndtri_as241(counter_uniform(key, step, slot));
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
