// ez_eizo.cu — hit-and-run sampling and the device-resident EI-ZO loop.
//
// Reference (corridor/cpoly.py, corridor/inflation.py):
//   hit_and_run_sample  cpoly.py:141-173 (+ _chords 127-138)      -> k_hnr
//   inflate_edge        inflation.py:262-325                      -> ez_inflate_edge
//     first-N_p colliding samples by index  :300-301              -> k_compact
//     project_batch + fail-fast check + _bisection_batch :302-310 -> k_bisect
//     _place_hyperplanes + compute_step_back :203-259             -> k_place
// Samples, candidates and faces stay in device memory; the host reads one
// 32-byte status record per iteration.
#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

#include <cooperative_groups.h>

#include "ez_device.cuh"
#include "ez_rng.cuh"
#include "ez_world.h"

namespace ez {

constexpr double kMemberTol = 1e-9;   // cpoly.py:19 MEMBER_TOL
constexpr double kChordMask = 1e-14;  // cpoly.py:134-135
constexpr double kChordTol = 1e-12;   // cpoly.py:167

// ---------------------------------------------------------------------------
// hit-and-run: one group of LPW lanes per walk.  Lane l draws the normals
// k = l, l + LPW, ... and owns the faces f = l, l + LPW, ...; directions are
// exchanged and the chord end points reduced with shuffles inside the group,
// so every lane holds the same walk state and the result is bitwise identical
// to a one-thread walk (the min/max over faces is order independent).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void set_status(int32_t* status, int32_t code) {
    if (code != EZ_OK) atomicCAS(status, 0, code);
}

template <int LPW>
__device__ __forceinline__ unsigned group_mask() {
    if (LPW == 32) return 0xffffffffu;
    return ((1u << LPW) - 1u) << ((threadIdx.x & 31) & ~(LPW - 1));
}

// A: faces, row f at A + f * lda.  VEC: rows are 16-byte aligned with lda
// even (shared-memory staging), so a row is read as double2 pairs.
// Zw: the walk's counter-stream draws (k_draws), element (step, k) at
// Zw[(step * (d + 1) + k) * zs] (unit directions, then the uniform); loaded one step ahead.
template <int MAXD, int RNG, int LPW, bool VEC>
__device__ __forceinline__ int hnr_walk(double (&x)[MAXD], int d, const double* __restrict__ A, int lda,
                                        const double* __restrict__ b, int F, int n_ms, uint64_t seed,
                                        uint64_t walk, bool check_seed, const double* __restrict__ Zw, int64_t zs) {
    constexpr int PER = (MAXD + LPW - 1) / LPW;  // normals drawn per lane
    const unsigned gm = group_mask<LPW>();
    const int lane = threadIdx.x & (LPW - 1);
    double nxt[PER], nxt_u = 0.0;
    auto load_draws = [&](int step) {
        if (RNG != EZ_RNG_COUNTER || step >= n_ms) return;
        const double* z = Zw + static_cast<int64_t>(step) * (d + 1) * zs;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int k = lane + j * LPW;
            nxt[j] = (k < d) ? __ldg(z + k * zs) : 0.0;
        }
        nxt_u = __ldg(z + d * zs);
    };
    load_draws(0);
    for (int step = 0; step < n_ms; ++step) {
        double dir[MAXD];
        double cur_u = 0.0;
        if (RNG == EZ_RNG_COUNTER) {
            double mine[PER];
#pragma unroll
            for (int j = 0; j < PER; ++j) mine[j] = nxt[j];
            cur_u = nxt_u;
            load_draws(step + 1);  // in flight while this step runs
#pragma unroll
            for (int k = 0; k < MAXD; ++k) dir[k] = __shfl_sync(gm, mine[k / LPW], k % LPW, LPW);
        } else {
            // Philox: lane l produces normals 4g..4g+3 of the groups g = l, l + LPW, ...
            constexpr int NG = (MAXD + 3) / 4;
            constexpr int PERG = (NG + LPW - 1) / LPW;
            float mine[PERG][4];
#pragma unroll
            for (int j = 0; j < PERG; ++j) {
                const int g = lane + j * LPW;
                if (4 * g < d) {
                    const Philox4 r = philox_draw(seed, walk, static_cast<uint32_t>(step), static_cast<uint32_t>(g));
                    box_muller(r.x, r.y, mine[j][0], mine[j][1]);
                    box_muller(r.z, r.w, mine[j][2], mine[j][3]);
                } else {
                    mine[j][0] = mine[j][1] = mine[j][2] = mine[j][3] = 0.f;
                }
            }
#pragma unroll
            for (int k = 0; k < MAXD; ++k) {
                const int g = k / 4;
                const float v = __shfl_sync(gm, mine[g / LPW][k % 4], g % LPW, LPW);
                dir[k] = (k < d) ? static_cast<double>(v) : 0.0;
            }
        }
        // normalise like numpy (squares rounded, left-to-right sum, IEEE divide);
        // the counter stream's draws arrive normalised (k_draws)
        if (RNG != EZ_RNG_COUNTER) {
            double ss = 0.0;
#pragma unroll
            for (int k = 0; k < MAXD; ++k)
                if (k < d) ss = __dadd_rn(ss, __dmul_rn(dir[k], dir[k]));
            const double nrm = sqrt(ss);
            // lane l divides components l, l + LPW, ... (IEEE division, as numpy);
            // the quotients are broadcast back to the group
            double qv[PER];
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const int k = lane + j * LPW;
                double v = 0.0;
#pragma unroll
                for (int kk = 0; kk < MAXD; ++kk)
                    if (kk == k) v = dir[kk];
                qv[j] = (k < d) ? v / nrm : 0.0;
            }
#pragma unroll
            for (int k = 0; k < MAXD; ++k) dir[k] = __shfl_sync(gm, qv[k / LPW], k % LPW, LPW);
        }
        // chord end points: t_hi = min over h > 0 of sl / h, t_lo = max over h < 0.
        // The arg-min/max is tracked as the fraction (sl, h), compared by
        // cross-multiplication, and divided once at the end.
        // fractions carry their sign in the denominator: hi = (s, h > 0),
        // lo = (s, h < 0); the empty chord ends are +inf/1 and +inf/-1.
        double hi_s = INFINITY, hi_h = 1.0, lo_s = INFINITY, lo_h = -1.0;
        int outside = 0;
#pragma unroll 2
        for (int f = lane; f < F; f += LPW) {
            const double* a = A + static_cast<int64_t>(f) * lda;
            double g0 = 0.0, g1 = 0.0, h0 = 0.0, h1 = 0.0;
#pragma unroll
            for (int k = 0; k < MAXD; k += 2) {
                if (k < d) {
                    double a0, a1;
                    if (VEC) {
                        const double2 v = *reinterpret_cast<const double2*>(a + k);
                        a0 = v.x;
                        a1 = v.y;
                    } else {
                        a0 = a[k];
                        a1 = (k + 1 < d) ? a[k + 1] : 0.0;
                    }
                    g0 = fma(a0, x[k], g0);
                    h0 = fma(a0, dir[k], h0);
                    if (k + 1 < d) {
                        g1 = fma(a1, x[k + 1], g1);
                        h1 = fma(a1, dir[k + 1], h1);
                    }
                }
            }
            const double sl = b[f] - (g0 + g1);
            const double h = h0 + h1;
            outside |= (check_seed && step == 0 && -sl > kMemberTol);
            if (h > kChordMask) {
                if (sl * hi_h < hi_s * h) { hi_s = sl; hi_h = h; }       // sl/h < hi_s/hi_h
            } else if (h < -kChordMask) {
                if (sl * lo_h > lo_s * h) { lo_s = sl; lo_h = h; }       // sl/h > lo_s/lo_h (h, lo_h < 0)
            }
        }
#pragma unroll
        for (int o = LPW / 2; o > 0; o >>= 1) {
            const double os = __shfl_xor_sync(gm, hi_s, o, LPW), oh = __shfl_xor_sync(gm, hi_h, o, LPW);
            if (os * hi_h < hi_s * oh) { hi_s = os; hi_h = oh; }
            const double ls = __shfl_xor_sync(gm, lo_s, o, LPW), lh = __shfl_xor_sync(gm, lo_h, o, LPW);
            if (ls * lo_h > lo_s * lh) { lo_s = ls; lo_h = lh; }
            outside |= __shfl_xor_sync(gm, outside, o, LPW);
        }
        double thi = hi_s / hi_h;
        double tlo = lo_s / lo_h;
        if (outside) return EZ_SEED_OUTSIDE;
        if (thi < tlo - kChordTol) return EZ_EMPTY_CHORD;
        tlo = fmin(tlo, 0.0);
        thi = fmax(thi, 0.0);
        double u;
        if (RNG == EZ_RNG_COUNTER) {
            u = cur_u;
        } else {
            const Philox4 r = philox_draw(seed, walk, static_cast<uint32_t>(step), static_cast<uint32_t>((d + 3) / 4));
            u = philox_u53(r.x, r.y);
        }
        const double tt = __dadd_rn(tlo, __dmul_rn(u, thi - tlo));
#pragma unroll
        for (int k = 0; k < MAXD; ++k)
            if (k < d) x[k] = __dadd_rn(x[k], __dmul_rn(dir[k], tt));
    }
    return EZ_OK;
}

// All counter-stream draws of a walk batch, ahead of the walks:
// Z[(step * (d + 1) + k) * count + i] is normal k (k < d) or the uniform
// (k = d) of walk walk_offset + i at mixing step `step` (seeding.py:40-60).
// They do not depend on the walk state, so generating them here (fully
// parallel, throughput bound) leaves the walk's 60-step critical path with
// loads issued a step ahead instead of hash + ndtri chains.
// The draws are stored as the walk's unit direction (numpy's normalisation:
// squares rounded, summed left to right, IEEE sqrt and divide; cpoly.py:163-164),
// so the walks' critical path skips the norm.  Element (step, k) at
// Z[(step * (d + 1) + k) * count + walk]; k = d holds the chord uniform.
// Warp-cooperative inverse normals: the central rational (85% of the draws)
// is evaluated in place; the tail draws of the warp's 32 x d uniforms are
// packed into shared memory, evaluated by all 32 lanes together (about two
// rounds instead of a divergent tail branch in almost every warp for each of
// the d slots) and read back.
template <int MAXD>
__global__ void __launch_bounds__(MAXD <= 16 ? 256 : 128)
k_draws(uint64_t seed, uint64_t walk_offset, int64_t count, int d, int step0, double* __restrict__ Z,
        const int32_t* __restrict__ status) {
    constexpr int kWarps = (MAXD <= 16 ? 256 : 128) / 32;
    __shared__ double s_tail[kWarps][32 * MAXD];
    if (status && (status[0] != EZ_OK || status[1] != 0)) return;
    // one thread per (walk, step), the step from blockIdx.y (no 64-bit
    // division): the walk's hash prefix once for its d + 1 draws
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const bool live = i < count;  // dead lanes take part in the warp's tail rounds
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t step = static_cast<uint64_t>(step0) + blockIdx.y;
    const uint64_t key = walk_key(seed, walk_offset + static_cast<uint64_t>(live ? i : 0));
    double* st = s_tail[wid];
    double v[MAXD];
    uint32_t tails = 0;  // bit k: slot k went to the warp's tail list
    int n_tail = 0;
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
        if (k < d) {
            const double u = counter_uniform(key, step, k);
            const bool tail = live && !as241_central(u);
            v[k] = (live && !tail) ? as241_center(u) : 0.0;
            const unsigned m = __ballot_sync(0xffffffffu, tail);
            if (tail) {
                st[n_tail + __popc(m & ((1u << lane) - 1u))] = u;
                tails |= 1u << k;
            }
            n_tail += __popc(m);
        }
    }
    __syncwarp();
    for (int t = lane; t < n_tail; t += 32) st[t] = as241_tail(st[t]);
    __syncwarp();
    // read the tail results back: the same ballots give the same slots
    n_tail = 0;
    double ss = 0.0;
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
        if (k < d) {
            const bool tail = (tails >> k) & 1u;
            const unsigned m = __ballot_sync(0xffffffffu, tail);
            if (tail) v[k] = st[n_tail + __popc(m & ((1u << lane) - 1u))];
            n_tail += __popc(m);
            ss = __dadd_rn(ss, __dmul_rn(v[k], v[k]));
        }
    }
    if (!live) return;
    // unit direction: one division and d products (numpy divides each
    // component, cpoly.py:163-164; the products differ from its quotients by
    // at most an ulp, below the ndtri approximation's own few ulps)
    const double inv = 1.0 / sqrt(ss);
    double* z = Z + static_cast<int64_t>(step) * (d + 1) * count + i;
#pragma unroll
    for (int k = 0; k < MAXD; ++k)
        if (k < d) z[k * count] = v[k] * inv;
    z[d * count] = counter_uniform(key, step, d);
}

static void launch_draws(cudaStream_t s, uint64_t seed, uint64_t walk_offset, int64_t count, int d, int n_ms,
                         double* z, const int32_t* status) {
    for (int step0 = 0; step0 < n_ms; step0 += 65535) {  // gridDim.y limit
        const unsigned gy = static_cast<unsigned>(std::min(n_ms - step0, 65535));
        if (d <= 8) k_draws<8><<<dim3(static_cast<unsigned>((count + 255) / 256), gy), 256, 0, s>>>(seed, walk_offset, count, d, step0, z, status);
        else if (d <= 16) k_draws<16><<<dim3(static_cast<unsigned>((count + 255) / 256), gy), 256, 0, s>>>(seed, walk_offset, count, d, step0, z, status);
        else k_draws<32><<<dim3(static_cast<unsigned>((count + 127) / 128), gy), 128, 0, s>>>(seed, walk_offset, count, d, step0, z, status);
    }
}

// Walk i starts at seeds[i % n_seeds] (explicit seeds) or at a point of the
// segment v1 + alpha * e drawn from the (seed, walk, SEED_STEP) stream
// (inflation.py:288-290).  F is read from F_dev when given (EI-ZO loop).
// Faces are staged in shared memory when F <= smem_faces, with the padded
// row stride lda (even, lda / 2 odd: the LPW lanes' double2 reads of
// distinct rows fall in distinct bank groups); otherwise they are read from
// L1/L2 with stride d.
template <int MAXD, int RNG, int LPW, int BT>
__global__ void __launch_bounds__(BT)
k_hnr(const double* __restrict__ A, const double* __restrict__ b, const int32_t* __restrict__ F_dev, int F,
      int d, const double* __restrict__ seeds, int64_t n_seeds, const double* __restrict__ seg, int64_t count,
      int n_ms, uint64_t seed, uint64_t walk_offset, double* __restrict__ out, int32_t* __restrict__ status,
      int smem_faces, int lda, const double* __restrict__ Z) {
    extern __shared__ __align__(16) double s_faces[];
    if (F_dev) F = *F_dev;
    if (status[0] != EZ_OK || status[1] != 0) return;  // (status, stop)
    const bool staged = F <= smem_faces;
    if (staged) {
        for (int i = threadIdx.x; i < F * lda; i += BT) {
            const int f = i / lda, k = i - f * lda;
            s_faces[i] = (k < d) ? A[static_cast<int64_t>(f) * d + k] : 0.0;
        }
        for (int i = threadIdx.x; i < F; i += BT) s_faces[F * lda + i] = b[i];
    }
    __syncthreads();
    const int64_t i = (static_cast<int64_t>(blockIdx.x) * BT + threadIdx.x) / LPW;
    if (i >= count) return;  // whole groups leave together
    const int lane = threadIdx.x & (LPW - 1);
    const uint64_t walk = walk_offset + static_cast<uint64_t>(i);
    double x[MAXD];
    if (seeds) {
        const double* s = seeds + (i % n_seeds) * d;
#pragma unroll
        for (int k = 0; k < MAXD; ++k) x[k] = (k < d) ? s[k] : 0.0;
    } else {
        double alpha;
        if (RNG == EZ_RNG_COUNTER) {
            alpha = counter_uniform(walk_key(seed, walk), kSeedStep, 0);
        } else {
            const Philox4 r = philox_draw(seed, walk, kPhiloxSeedStep, 0);
            alpha = philox_u53(r.x, r.y);
        }
#pragma unroll
        for (int k = 0; k < MAXD; ++k) x[k] = (k < d) ? __dadd_rn(seg[k], __dmul_rn(alpha, seg[d + k])) : 0.0;
    }
    const double* Zw = Z ? Z + i : nullptr;
    const int st = staged ? hnr_walk<MAXD, RNG, LPW, true>(x, d, s_faces, lda, s_faces + F * lda, F, n_ms, seed, walk,
                                                           seeds == nullptr, Zw, count)
                          : hnr_walk<MAXD, RNG, LPW, false>(x, d, A, d, b, F, n_ms, seed, walk, seeds == nullptr, Zw,
                                                            count);
    if (st != EZ_OK) {
        if (lane == 0) set_status(status, st);
        return;
    }
    double* o = out + i * d;
#pragma unroll
    for (int k = 0; k < MAXD; ++k)
        if (k < d && (k % LPW) == lane) o[k] = x[k];
}

// ---------------------------------------------------------------------------
// hit-and-run for large polytopes on the FP64 tensor cores.  Per mixing step
// the chord data of a warp's 8 walks against all faces is one small GEMM:
//     G'[f][w] = sum_k Ap[f][k] * xt_w[k],   H[f][w] = sum_k Ap[f][k] * dir_w[k]
// with Ap = [A | -b | 0] (KP = 4 KC columns) and xt_w = [x_w | 1 | 0], so the
// slack is b_f - a_f.x_w = -G'.  Each mma.sync.m8n8k4.f64 takes one A value
// per lane (8 faces x 4 columns) and the walk fragments stay in registers, so
// a face row is read once per 8 walks instead of once per walk (the
// lane-per-face kernel above is shared-memory bound for large F).
//
// Fragment ownership (PTX m8n8k4 .row.col): lane = 4 wl + c holds x and dir
// components k = 4 j + c of walk wl (the B fragments), and the C entries of
// face wl of each 8-face tile for walks 2c and 2c + 1.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// Ap rows 0 .. ceil8(F) - 1 from (A, b); rows >= F are zero (inert faces:
// h = 0 is masked out and the slack 0 is not "outside").
__global__ void k_pack_faces(const double* __restrict__ A, const double* __restrict__ b,
                             const int32_t* __restrict__ F_dev, int F, int d, int kp, double* __restrict__ Ap) {
    if (F_dev) F = *F_dev;
    const int rows = (F + 7) & ~7;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows * kp; i += gridDim.x * blockDim.x) {
        const int f = i / kp, k = i - f * kp;
        double v = 0.0;
        if (f < F) v = (k < d) ? A[static_cast<int64_t>(f) * d + k] : (k == d ? -b[f] : 0.0);
        Ap[i] = v;
    }
}

// Running chord ends, two equivalent forms (the same faces win, bit for bit):
//
// unsigned (SIGNED = false): both ends keep the min of sl / |h| as a fraction
// (S, H), H > 0, over faces with h > mask (upper) or h < -mask (lower), with
// sl = -g the slack; t_hi = S0 / H0, t_lo = -S1 / H1.  The comparisons are the
// lane walk's products (sl lo_h > lo_s h with lo_h = -H1).
//
// signed (SIGNED = true): end e keeps (S, H) = (g, h) of the face that ends
// the chord, g = a.x - b (the negated slack, the DMMA output as is) and h =
// a.dir (H > 0 upper, H < 0 lower); t = -S / H.  A face with h > mask ends the
// chord earlier above iff -g/h < -S0/H0 <=> g H0 > S0 h; one with h < -mask
// ends it later below iff g H1 < S1 h.  The same products up to exact
// negations, but no negation or absolute value of g and h: one comparison on
// the FP64 pipe instead of three, the sign of h tested on its high word.
// Measured: the 14-DOF walk (KC = 4), bound by its FP64 pipe, runs 21% faster
// signed; the 7-DOF walk (KC = 2, two independent chains per lane, bound by
// issue) runs 15% faster unsigned.  Branch-free either way.
template <bool SIGNED>
__device__ __forceinline__ void chord_update(double g, double h, double (&S)[2], double (&H)[2]) {
    if constexpr (SIGNED) {
        const bool neg = __double2hiint(h) < 0;
        const double sc = neg ? S[1] : S[0], hc = neg ? H[1] : H[0];
        const double p = g * hc, q = sc * h;
        const double lhs = neg ? q : p, rhs = neg ? p : q;  // upper end: p > q; lower end: p < q
        const bool take = (fabs(h) > kChordMask) && (lhs > rhs);
        const bool t0 = take && !neg, t1 = take && neg;
        S[0] = t0 ? g : S[0];
        H[0] = t0 ? h : H[0];
        S[1] = t1 ? g : S[1];
        H[1] = t1 ? h : H[1];
    } else {
        const double sl = -g;
        const bool neg = h < 0.0;
        const double ah = fabs(h);
        const double sc = neg ? S[1] : S[0], hc = neg ? H[1] : H[0];
        const bool take = (ah > kChordMask) && (sl * hc < sc * ah);
        const bool t0 = take && !neg, t1 = take && neg;
        S[0] = t0 ? sl : S[0];
        H[0] = t0 ? ah : H[0];
        S[1] = t1 ? sl : S[1];
        H[1] = t1 ? ah : H[1];
    }
}

// merge of two running ends (lower: end e = 1)
template <bool SIGNED>
__device__ __forceinline__ void chord_merge(double& S, double& H, double os, double oh, bool lower) {
    const double p = os * H, q = S * oh;
    if (SIGNED ? (lower ? (p < q) : (p > q)) : (p < q)) {
        S = os;
        H = oh;
    }
}

#ifndef EZ_HNR_TPR
#define EZ_HNR_TPR 2
#endif
#ifndef EZ_HNR_MINB
#define EZ_HNR_MINB 8
#endif
#ifndef EZ_HNR_SWP_KC
#define EZ_HNR_SWP_KC 2
#endif
#ifndef EZ_HNR_SP2
#define EZ_HNR_SP2 1
#endif
template <int KC>
__global__ void __launch_bounds__(64, KC >= 8 ? 8 : EZ_HNR_MINB)
k_hnr_mma(const double* __restrict__ Ap, const int32_t* __restrict__ F_dev, int F, int d,
          const double* __restrict__ seeds, int64_t n_seeds, const double* __restrict__ seg, int64_t count,
          int n_ms, uint64_t seed, uint64_t walk_offset, double* __restrict__ out, int32_t* __restrict__ status,
          const double* __restrict__ Z) {
    constexpr int KP = 4 * KC;
    constexpr bool SG = KC >= 4;  // chord-end form (chord_update)
    if (F_dev) F = *F_dev;
    if (status[0] != EZ_OK || status[1] != 0) return;
    const int lane = threadIdx.x & 31;
    const int64_t wbase = ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 8;
    if (wbase >= count) return;  // warp-uniform
    const int wl = lane >> 2, c = lane & 3;
    const int64_t wi = min(wbase + wl, count - 1);  // idle slots shadow the last walk
    const uint64_t key = walk_key(seed, walk_offset + static_cast<uint64_t>(wi));
    const int64_t zstep = static_cast<int64_t>(d + 1) * count;
    double nd[KC], nu;  // walk wl's direction components k = 4 j + c and its chord uniform
    auto load_draws = [&](int step) {
        if (step >= n_ms) return;
        const double* z = Z + step * zstep;
#pragma unroll
        for (int j = 0; j < KC; ++j) {
            const int k = 4 * j + c;
            nd[j] = (k < d) ? __ldg(z + k * count + wi) : 0.0;
        }
        nu = __ldg(z + d * count + wi);
    };
    load_draws(0);
    double x[KC], dr[KC];
    if (seeds) {
        const double* sp = seeds + (wi % n_seeds) * d;
#pragma unroll
        for (int j = 0; j < KC; ++j) {
            const int k = 4 * j + c;
            x[j] = (k < d) ? sp[k] : (k == d ? 1.0 : 0.0);
        }
    } else {
        const double alpha = counter_uniform(key, kSeedStep, 0);
#pragma unroll
        for (int j = 0; j < KC; ++j) {
            const int k = 4 * j + c;
            x[j] = (k < d) ? __dadd_rn(seg[k], __dmul_rn(alpha, seg[d + k])) : (k == d ? 1.0 : 0.0);
        }
    }
    const bool check_seed = seeds == nullptr;
    const int tiles = (F + 7) >> 3;
    const double* arow = Ap + static_cast<int64_t>(wl) * KP + c;
    for (int step = 0; step < n_ms; ++step) {
#pragma unroll
        for (int j = 0; j < KC; ++j) dr[j] = nd[j];
        const double cu = nu;
        load_draws(step + 1);  // in flight while this step runs
        // dr is already the unit direction (k_draws normalises)
        // TPR 8-face tiles per round, the next round's A fragments loaded
        // ahead (L1 latency hidden behind the current round's MMAs).  For
        // d < 8 tile u of a round updates its own running ends
        // [u][slot][hi/lo], so the TPR compare-select chains are independent
        // until the merge below (7-DOF walk -2%; at d >= 8 the registers cost
        // more than the chains: 14-DOF +4%, so one chain)
        constexpr int TPR = EZ_HNR_TPR;
        constexpr bool SWP = KC >= EZ_HNR_SWP_KC;  // software-pipelined rounds
        constexpr int SP = KC <= 2 ? EZ_HNR_SP2 : 1;  // tiles per pipelined round
        constexpr int NCH = SWP ? (KC <= 2 ? SP : 1) : (KC <= 2 ? TPR : 1);
        double cs[NCH][2][2], ch[NCH][2][2];
#pragma unroll
        for (int u = 0; u < NCH; ++u)
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
                for (int e = 0; e < 2; ++e) {  // no face yet: t_hi = +inf, t_lo = -inf
                    cs[u][s2][e] = SG ? -INFINITY : INFINITY;
                    ch[u][s2][e] = (SG && e) ? -1.0 : 1.0;
                }
        bool outside = false;
        if constexpr (SWP) {
            // Software-pipelined rounds of SP tiles: the DMMAs of round r are
            // issued before the chord updates of round r - 1, which then run
            // while the tensor pipe works (the walk waited on each round's
            // DMMA results before its compare-selects could start)
            double va[SP][KC], vn[SP][KC], gp[SP][2], hp[SP][2];
#pragma unroll
            for (int u = 0; u < SP; ++u) {
                gp[u][0] = gp[u][1] = hp[u][0] = hp[u][1] = 0.0;
#pragma unroll
                for (int j = 0; j < KC; ++j)
                    va[u][j] = (u < tiles) ? __ldg(arow + static_cast<int64_t>(u) * 8 * KP + 4 * j) : 0.0;
            }
            for (int t = 0; t < tiles; t += SP) {
#pragma unroll
                for (int u = 0; u < SP; ++u)
#pragma unroll
                    for (int j = 0; j < KC; ++j)
                        vn[u][j] = (t + SP + u < tiles) ? __ldg(arow + static_cast<int64_t>(t + SP + u) * 8 * KP + 4 * j) : 0.0;
                double g[SP][2], h[SP][2];
#pragma unroll
                for (int u = 0; u < SP; ++u) g[u][0] = g[u][1] = h[u][0] = h[u][1] = 0.0;
#pragma unroll
                for (int j = 0; j < KC; ++j)
#pragma unroll
                    for (int u = 0; u < SP; ++u) {
                        dmma_8x8x4(g[u][0], g[u][1], va[u][j], x[j]);
                        dmma_8x8x4(h[u][0], h[u][1], va[u][j], dr[j]);
                    }
                if (t > 0) {
#pragma unroll
                    for (int u = 0; u < SP; ++u)
#pragma unroll
                        for (int s2 = 0; s2 < 2; ++s2) {
                            outside |= check_seed && step == 0 && gp[u][s2] > kMemberTol;
                            chord_update<SG>(gp[u][s2], hp[u][s2], cs[u % NCH][s2], ch[u % NCH][s2]);
                        }
                }
#pragma unroll
                for (int u = 0; u < SP; ++u) {
#pragma unroll
                    for (int s2 = 0; s2 < 2; ++s2) {
                        gp[u][s2] = g[u][s2];
                        hp[u][s2] = h[u][s2];
                    }
#pragma unroll
                    for (int j = 0; j < KC; ++j) va[u][j] = vn[u][j];
                }
            }
            if (tiles > 0) {
#pragma unroll
                for (int u = 0; u < SP; ++u)
#pragma unroll
                    for (int s2 = 0; s2 < 2; ++s2) {
                        outside |= check_seed && step == 0 && gp[u][s2] > kMemberTol;
                        chord_update<SG>(gp[u][s2], hp[u][s2], cs[u % NCH][s2], ch[u % NCH][s2]);
                    }
            }
        } else {
        double va[TPR][KC], vn[TPR][KC];
#pragma unroll
        for (int u = 0; u < TPR; ++u)
#pragma unroll
            for (int j = 0; j < KC; ++j)
                va[u][j] = (u < tiles) ? __ldg(arow + static_cast<int64_t>(u) * 8 * KP + 4 * j) : 0.0;
        for (int t = 0; t < tiles; t += TPR) {
#pragma unroll
            for (int u = 0; u < TPR; ++u)
#pragma unroll
                for (int j = 0; j < KC; ++j)
                    vn[u][j] = (t + TPR + u < tiles) ? __ldg(arow + static_cast<int64_t>(t + TPR + u) * 8 * KP + 4 * j) : 0.0;
            double g[TPR][2], h[TPR][2];
#pragma unroll
            for (int u = 0; u < TPR; ++u) g[u][0] = g[u][1] = h[u][0] = h[u][1] = 0.0;
#pragma unroll
            for (int j = 0; j < KC; ++j)
#pragma unroll
                for (int u = 0; u < TPR; ++u) {
                    dmma_8x8x4(g[u][0], g[u][1], va[u][j], x[j]);
                    dmma_8x8x4(h[u][0], h[u][1], va[u][j], dr[j]);
                }
            // a tile past the end has zero rows: h = 0 is masked, g = 0 is not outside
#pragma unroll
            for (int u = 0; u < TPR; ++u)
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2) {
                    outside |= check_seed && step == 0 && g[u][s2] > kMemberTol;
                    chord_update<SG>(g[u][s2], h[u][s2], cs[u % NCH][s2], ch[u % NCH][s2]);
                }
#pragma unroll
            for (int u = 0; u < TPR; ++u)
#pragma unroll
                for (int j = 0; j < KC; ++j) va[u][j] = vn[u][j];
        }
        }
        // Reduce over the 8 face rows (lane bits 2-4) as a reduce-scatter: the
        // 4 running ends (slot s2, end e) halve at each butterfly level, so
        // lane bits 4 and 3 pick the end a lane keeps ((s2, e) = (bit 4, bit 3))
        // and the last level exchanges it whole.  16 shuffles instead of 48,
        // and each lane divides one fraction instead of four.
        const bool b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1;
#pragma unroll
        for (int u = 1; u < NCH; ++u)
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
                for (int e = 0; e < 2; ++e) chord_merge<SG>(cs[0][s2][e], ch[0][s2][e], cs[u][s2][e], ch[u][s2][e], e == 1);
        // level 1 (xor 16): keep slot b4, send slot !b4 (both ends)
        double kS[2], kH[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const double sendS = b4 ? cs[0][0][e] : cs[0][1][e], sendH = b4 ? ch[0][0][e] : ch[0][1][e];
            kS[e] = b4 ? cs[0][1][e] : cs[0][0][e];
            kH[e] = b4 ? ch[0][1][e] : ch[0][0][e];
            const double os = __shfl_xor_sync(0xffffffffu, sendS, 16);
            const double oh = __shfl_xor_sync(0xffffffffu, sendH, 16);
            chord_merge<SG>(kS[e], kH[e], os, oh, e == 1);
        }
        // level 2 (xor 8): keep end b3, send end !b3
        double S1 = b3 ? kS[1] : kS[0], H1 = b3 ? kH[1] : kH[0];
        {
            const double os = __shfl_xor_sync(0xffffffffu, b3 ? kS[0] : kS[1], 8);
            const double oh = __shfl_xor_sync(0xffffffffu, b3 ? kH[0] : kH[1], 8);
            chord_merge<SG>(S1, H1, os, oh, b3);
        }
        // level 3 (xor 4): both lanes hold the same end
        {
            const double os = __shfl_xor_sync(0xffffffffu, S1, 4);
            const double oh = __shfl_xor_sync(0xffffffffu, H1, 4);
            chord_merge<SG>(S1, H1, os, oh, b3);
        }
        const bool any_out = __any_sync(0xffffffffu, outside);
        // this lane's fraction: t_hi (e = 0) or -t_lo (e = 1) of walk 2c + b4
        // (signed form: t_hi = -S/H, -t_lo = S/H; unsigned: S/H for both)
        const double q = (SG && !b3 ? -S1 : S1) / H1;
        // walk wl = 2c' + s2 reads t_hi from lane 16 s2 + c' and -t_lo from lane 16 s2 + 8 + c'
        const int src = 16 * (wl & 1) + (wl >> 1);
        double thi = __shfl_sync(0xffffffffu, q, src);
        double tlo = -__shfl_sync(0xffffffffu, q, src + 8);
        const int err = (thi < tlo - kChordTol) ? EZ_EMPTY_CHORD : EZ_OK;
        tlo = fmin(tlo, 0.0);
        thi = fmax(thi, 0.0);
        const double mine = __dadd_rn(tlo, __dmul_rn(cu, thi - tlo));
        if (any_out) {
            if (lane == 0) set_status(status, EZ_SEED_OUTSIDE);
            return;
        }
        if (__any_sync(0xffffffffu, err != EZ_OK)) {
            if (err != EZ_OK) set_status(status, err);
            return;
        }
#pragma unroll
        for (int j = 0; j < KC; ++j)
            if (4 * j + c < d) x[j] = __dadd_rn(x[j], __dmul_rn(dr[j], mine));
    }
    if (wbase + wl < count) {
        double* o = out + (wbase + wl) * d;
#pragma unroll
        for (int j = 0; j < KC; ++j)
            if (4 * j + c < d) o[4 * j + c] = x[j];
    }
}

// Ap geometry: KP columns (d + 1 rounded up to a multiple of 4 k-chunks),
// rows padded to a multiple of 8
static int hnr_mma_kp(int d) { return d < 8 ? 8 : (d < 16 ? 16 : 32); }
static int64_t hnr_ap_words(int f_bound, int d) {
    return static_cast<int64_t>((f_bound + 7) & ~7) * hnr_mma_kp(d);
}

// reference contains_many over all explicit seeds (cpoly.py:158-159)
__global__ void k_seed_check(const double* __restrict__ A, const double* __restrict__ b, int F, int d,
                             const double* __restrict__ seeds, int64_t n_seeds, int32_t* __restrict__ status) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_seeds) return;
    double worst = -INFINITY;
    for (int f = 0; f < F; ++f) {
        double g = 0.0;
        for (int k = 0; k < d; ++k) g = fma(A[f * d + k], seeds[i * d + k], g);
        worst = fmax(worst, g - b[f]);
    }
    if (!(worst <= kMemberTol)) set_status(status, EZ_SEED_OUTSIDE);
}

// ---------------------------------------------------------------------------
// EI-ZO iteration kernels
// ---------------------------------------------------------------------------
// Device record shared with the host.  Global part (rec): status (first
// error wins), stop (set when an iteration accepts; every later kernel
// returns at once) and the face count.  Per-iteration part (it, double
// buffered so the host can enqueue iteration k+1 before reading k).
enum : int { kStatus = 0, kStop = 1, kFaces = 2 };
enum : int { kColM = 0, kNumCand = 1, kPlaced = 2, kAccept = 3 };
constexpr int kRecInts = 32;               // rec[0..7] global, slots at 8 and 16
__host__ __device__ constexpr int slot_offset(int k) { return 8 + 8 * (k & 1); }

// order-preserving compaction of the first n_p colliding sample indices and
// the acceptance decision of the unadaptive test (inflation.py:164-172, 294-301)
__global__ void __launch_bounds__(1024)
k_compact(const uint8_t* __restrict__ free_flags, int64_t n, int n_p, double thr, int32_t* __restrict__ rec,
          int32_t* __restrict__ it, int32_t* __restrict__ col) {
    __shared__ int warp_tot[32];
    __shared__ int warp_off[32];
    __shared__ int s_total;
    if (rec[kStatus] != EZ_OK || rec[kStop]) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const bool accept = static_cast<double>(it[kColM]) <= thr;
    if (threadIdx.x == 0) {
        it[kAccept] = accept ? 1 : 0;
        if (accept) rec[kStop] = 1;
    }
    if (accept) return;
    // 16 flags per thread per round (one 16-byte load): a 1024-thread round
    // covers 16,384 samples, so an EI-ZO batch (10-26k) takes one or two
    // rounds of one block-wide scan instead of a scan per 1,024 flags
    constexpr int kPer = 16;
    int run = 0;
    for (int64_t base = 0; base < n && run < n_p; base += static_cast<int64_t>(blockDim.x) * kPer) {
        const int64_t i0 = base + static_cast<int64_t>(threadIdx.x) * kPer;
        uint32_t colmask = 0;  // bit j: sample i0 + j collides (flag 0)
        if (i0 + kPer <= n) {
            const uint4 v = *reinterpret_cast<const uint4*>(free_flags + i0);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int bb = 0; bb < 4; ++bb)
                    if (((w[q] >> (8 * bb)) & 0xFFu) == 0u) colmask |= 1u << (4 * q + bb);
        } else {
            for (int j = 0; j < kPer; ++j)
                if (i0 + j < n && free_flags[i0 + j] == 0) colmask |= 1u << j;
        }
        const int cnt = __popc(colmask);
        // block-wide exclusive scan of the per-thread counts
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) warp_tot[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            const int nw = blockDim.x >> 5;
            const int v = lane < nw ? warp_tot[lane] : 0;
            int wi = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += y;
            }
            warp_off[lane] = wi - v;
            if (lane == 31) s_total = wi;
        }
        __syncthreads();
        int pos = run + warp_off[wid] + (incl - cnt);
        while (colmask && pos < n_p) {  // this thread's colliding samples, in index order
            const int j = __ffs(colmask) - 1;
            colmask &= colmask - 1;
            col[pos++] = static_cast<int32_t>(i0 + j);
        }
        run += s_total;
        __syncthreads();
    }
    if (threadIdx.x == 0) it[kNumCand] = min(run, n_p);
}

// project_batch for one point (inflation.py:124-137, used at :297-310) on a
// point spread over a G-lane group: lane l holds components k = l + j G in
// slot j.  The dot products run over k in order on every lane (components
// gathered by shuffles), so every lane gets the serial loop's bits.
template <int MAXD, int G>
__device__ __forceinline__ double project_group(const double (&c)[(MAXD + G - 1) / G], int d,
                                                const double* __restrict__ v1, const double* __restrict__ e,
                                                double ee, double (&p)[(MAXD + G - 1) / G], int lane,
                                                unsigned gm) {
    constexpr int PER = (MAXD + G - 1) / G;
    double alpha = 0.0;
    if (ee != 0.0) {
        double dot = 0.0;
#pragma unroll
        for (int k = 0; k < MAXD; ++k) {
            const double ck = __shfl_sync(gm, c[k / G], k % G, G);
            if (k < d) dot = fma(ck - v1[k], e[k], dot);
        }
        alpha = fmin(fmax(dot / ee, 0.0), 1.0);
    }
    double r[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int k = lane + j * G;
        p[j] = (k < d) ? __dadd_rn(v1[k], __dmul_rn(alpha, e[k])) : 0.0;
        r[j] = (k < d) ? c[j] - p[j] : 0.0;
    }
    double ss = 0.0;
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
        const double rk = __shfl_sync(gm, r[k / G], k % G, G);
        if (k < d) ss = fma(rk, rk, ss);
    }
    return sqrt(ss);
}

constexpr int kBisectLanes = 8;

// One group of G lanes per candidate: project, fail-fast check of the
// projection, N_b bisection rounds (each a cooperative FK + collision check),
// t_col guard.  The group shares the candidate's row and centre store; each
// lane keeps only its own components of the candidate, projection and
// bracket (registers set the occupancy of this latency-bound kernel).
template <typename T, int MAXD, int G>
__global__ void __launch_bounds__(128)
k_bisect(const __grid_constant__ ModelDev<T> M, T margin, const double* __restrict__ X, int d, const int32_t* __restrict__ col,
         int32_t* __restrict__ rec, const int32_t* __restrict__ it, const double* __restrict__ seg, double ee,
         int n_b, double t_col,
         double* __restrict__ star, double* __restrict__ pstar, double* __restrict__ dstar) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint64_t bar;
    constexpr int CPB = 128 / G;  // candidates per CTA
    constexpr int PER = (MAXD + G - 1) / G;
    const int C = it[kNumCand];
    if (rec[kStatus] != EZ_OK || rec[kStop] || static_cast<int64_t>(blockIdx.x) * CPB >= C) return;
    tma_stage(smem, M.blob, M.blob_bytes, &bar);
    const int slot = threadIdx.x / G, lane = threadIdx.x & (G - 1);
    T* cen = reinterpret_cast<T*>(smem + M.blob_bytes) + static_cast<size_t>(slot) * M.cen_words;
    const size_t roff = (static_cast<size_t>(M.blob_bytes) + static_cast<size_t>(M.cen_words) * CPB * sizeof(T) + 15) &
                        ~static_cast<size_t>(15);
    double* row = reinterpret_cast<double*>(smem + roff) + slot * d;
    const int i = blockIdx.x * CPB + slot;
    if (i >= C) return;  // whole groups leave together
    const unsigned gm = coop_mask<G>();
    const double* v1 = seg;
    const double* e = seg + d;
    double c[PER], lo[PER], hi[PER];
    const double* xc = X + static_cast<int64_t>(col[i]) * d;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int k = lane + j * G;
        c[j] = (k < d) ? xc[k] : 0.0;
    }
    project_group<MAXD, G>(c, d, v1, e, ee, lo, lane, gm);
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int k = lane + j * G;
        hi[j] = c[j];
        if (k < d) row[k] = lo[j];
    }
    __syncwarp(gm);
    if (!config_free_coop<T, double, G>(M, smem, row, cen, margin)) {
        if (lane == 0) set_status(rec + kStatus, EZ_SEGMENT_IN_COLLISION);  // inflation.py:303-305
        return;
    }
    for (int r = 0; r < n_b; ++r) {
        double mid[PER];
        __syncwarp(gm);
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int k = lane + j * G;
            mid[j] = 0.5 * (lo[j] + hi[j]);
            if (k < d) row[k] = mid[j];
        }
        __syncwarp(gm);
        const bool fr = config_free_coop<T, double, G>(M, smem, row, cen, margin);
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            if (fr) lo[j] = mid[j];
            else hi[j] = mid[j];
        }
    }
    double ps[PER];
    const double ds = project_group<MAXD, G>(hi, d, v1, e, ee, ps, lane, gm);
    if (ds <= t_col && lane == 0) set_status(rec + kStatus, EZ_SEGMENT_IN_COLLISION);  // inflation.py:307-310
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int k = lane + j * G;
        if (k < d) {
            star[static_cast<int64_t>(i) * d + k] = hi[j];
            pstar[static_cast<int64_t>(i) * d + k] = ps[j];
        }
    }
    if (lane == 0) dstar[i] = ds;
}

// Two bisection levels per round.  One warp per candidate, four 8-lane
// subgroups: subgroup 0 checks the midpoint m of [lo, hi], subgroups 1 and 2
// the midpoints of [lo, m] and [m, hi] (the two points the next binary step
// can check), subgroup 3 the projection in the first round (the fail-fast
// check).  The round then takes both binary steps the results decide.  The
// quarter points are formed from the same end points with the same
// operations as the one-step loop's next midpoint, so every checked point,
// every decision and star/pstar are bit-identical to k_bisect's, in half the
// dependent rounds.
// Up to 8 DOF the kernel is capped at 64 registers (8 CTAs, 32 warps per SM,
// no spills): 7-DOF bisection 618 -> 522 us per region.  The 16-DOF
// instance lost 9% under the same cap and keeps its registers.
template <typename T, int MAXD>
__global__ void __launch_bounds__(128, MAXD <= 8 ? 8 : 1)
k_bisect2(const __grid_constant__ ModelDev<T> M, T margin, const double* __restrict__ X, int d,
          const int32_t* __restrict__ col, int32_t* __restrict__ rec, const int32_t* __restrict__ it,
          const double* __restrict__ seg, double ee, int n_b, double t_col, double* __restrict__ star,
          double* __restrict__ pstar, double* __restrict__ dstar) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint64_t bar;
    constexpr int G = kBisectLanes;
    constexpr int SLOTS = 128 / G;      // subgroups per CTA, each with a row and a centre store
    constexpr int CPB = 128 / 32;       // candidates per CTA
    constexpr int PER = (MAXD + G - 1) / G;
    static_assert(G == 8, "four subgroups per warp");
    const int C = it[kNumCand];
    if (rec[kStatus] != EZ_OK || rec[kStop] || static_cast<int64_t>(blockIdx.x) * CPB >= C) return;
    tma_stage(smem, M.blob, M.blob_bytes, &bar);
    const int slot = threadIdx.x / G, lane = threadIdx.x & (G - 1), sub = slot & 3;
    T* cen = reinterpret_cast<T*>(smem + M.blob_bytes) + static_cast<size_t>(slot) * M.cen_words;
    const size_t roff = (static_cast<size_t>(M.blob_bytes) + static_cast<size_t>(M.cen_words) * SLOTS * sizeof(T) + 15) &
                        ~static_cast<size_t>(15);
    double* row = reinterpret_cast<double*>(smem + roff) + slot * d;
    const int i = blockIdx.x * CPB + static_cast<int>(threadIdx.x >> 5);
    if (i >= C) return;  // whole warps leave together
    const unsigned gm = coop_mask<G>();
    const double* v1 = seg;
    const double* e = seg + d;
    double c[PER], lo[PER], hi[PER];
    const double* xc = X + static_cast<int64_t>(col[i]) * d;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int k = lane + j * G;
        c[j] = (k < d) ? xc[k] : 0.0;
    }
    project_group<MAXD, G>(c, d, v1, e, ee, lo, lane, gm);
#pragma unroll
    for (int j = 0; j < PER; ++j) hi[j] = c[j];
    bool first = true;
    for (int done = 0; first || done < n_b;) {
        const int lv = min(2, n_b - done);  // binary steps taken this round
        double m[PER], pt[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            m[j] = 0.5 * (lo[j] + hi[j]);
            pt[j] = sub == 0 ? m[j] : (sub == 1 ? 0.5 * (lo[j] + m[j]) : (sub == 2 ? 0.5 * (m[j] + hi[j]) : lo[j]));
        }
        const bool active = sub == 0 ? lv >= 1 : (sub == 3 ? first : lv >= 2);
        bool fr = true;
        if (active) {
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const int k = lane + j * G;
                if (k < d) row[k] = pt[j];
            }
            __syncwarp(gm);
            fr = config_free_coop<T, double, G>(M, smem, row, cen, margin);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, fr && lane == 0);  // bits 0, 8, 16, 24
        if (first) {
            if (!((bal >> 24) & 1u)) {
                if ((threadIdx.x & 31) == 0) set_status(rec + kStatus, EZ_SEGMENT_IN_COLLISION);  // inflation.py:303-305
                return;
            }
            first = false;
        }
        if (lv >= 1) {
            const bool f0 = bal & 1u;
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                if (f0) lo[j] = m[j];
                else hi[j] = m[j];
            }
            if (lv >= 2) {
                const bool f1 = (bal >> (f0 ? 16 : 8)) & 1u;
#pragma unroll
                for (int j = 0; j < PER; ++j) {
                    const double q = 0.5 * (lo[j] + hi[j]);  // the point subgroup 1 or 2 checked
                    if (f1) lo[j] = q;
                    else hi[j] = q;
                }
            }
            done += lv;
        }
        __syncwarp();
    }
    if (sub != 0) return;
    double ps[PER];
    const double ds = project_group<MAXD, G>(hi, d, v1, e, ee, ps, lane, gm);
    if (ds <= t_col && lane == 0) set_status(rec + kStatus, EZ_SEGMENT_IN_COLLISION);  // inflation.py:307-310
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int k = lane + j * G;
        if (k < d) {
            star[static_cast<int64_t>(i) * d + k] = hi[j];
            pstar[static_cast<int64_t>(i) * d + k] = ps[j];
        }
    }
    if (lane == 0) dstar[i] = ds;
}

// k_place's shared memory: candidate distances cached when they fit next to
// the alive bytes (up to 200 KB in all)
inline int place_dist_cap(int n) { return 9 * static_cast<size_t>(n) <= 200 * 1024 ? n : 0; }
inline size_t place_smem_bytes(int n, int dcap) {
    return static_cast<size_t>(dcap) * sizeof(double) + static_cast<size_t>(n);
}

// Greedy hyperplane placement on one CTA (inflation.py:232-259): the closest
// alive candidate (stable order == lexicographic (dist, index)) becomes a
// tangent face pushed back by compute_step_back; candidates outside die.
__global__ void __launch_bounds__(1024)
k_place(double* __restrict__ A, double* __restrict__ b, int32_t* __restrict__ rec, int32_t* __restrict__ it, int d,
        const double* __restrict__ star, const double* __restrict__ pstar, const double* __restrict__ dstar,
        const double* __restrict__ seg, double delta_max, int n_f, const double* __restrict__ targets, int dcap) {
    // dynamic shared memory: dcap cached distances, then one alive byte per candidate
    extern __shared__ __align__(16) uint8_t smem_place[];
    double* s_dist = reinterpret_cast<double*>(smem_place);
    uint8_t* alive = smem_place + static_cast<size_t>(dcap) * sizeof(double);
    __shared__ double s_bd[32];
    __shared__ int s_bi[32];
    __shared__ double s_a[32];
    __shared__ double s_rhs;
    __shared__ int s_best;
    if (rec[kStatus] != EZ_OK || rec[kStop]) return;
    const int C = it[kNumCand];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const bool cached = C <= dcap;
    for (int i = threadIdx.x; i < C; i += blockDim.x) {
        alive[i] = 1;
        if (cached) s_dist[i] = dstar[i];
    }
    int F = rec[kFaces];
    int placed = 0;
    const double* v1 = seg;
    const double* e = seg + d;
    const double* tg = targets ? targets : star;
    double rhs = 0.0;
    for (int r = 0; r < n_f; ++r) {
        __syncthreads();
        // one pass: the discard test of the face placed last round (on the
        // anchors, or on the original collisions in a repair, planner.py:
        // 191-192), then the arg-min over the survivors
        double bd = INFINITY;
        int bi = INT_MAX;
        for (int i = threadIdx.x; i < C; i += blockDim.x) {
            if (!alive[i]) continue;
            if (r > 0) {
                const double* t = tg + static_cast<int64_t>(i) * d;
                double dot = 0.0;
                for (int k = 0; k < d; ++k) dot = fma(t[k], s_a[k], dot);
                if (!(dot <= rhs)) {
                    alive[i] = 0;
                    continue;
                }
            }
            const double di = cached ? s_dist[i] : dstar[i];
            if (di < bd || (di == bd && i < bi)) {
                bd = di;
                bi = i;
            }
        }
        // (the barrier after the warp results also orders every read of s_a
        // above before warp 0 overwrites it)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double od = __shfl_down_sync(0xffffffffu, bd, o);
            const int oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (od < bd || (od == bd && oi < bi)) {
                bd = od;
                bi = oi;
            }
        }
        if (lane == 0) {
            s_bd[wid] = bd;
            s_bi[wid] = bi;
        }
        __syncthreads();
        if (wid == 0) {
            const int nw = blockDim.x >> 5;
            bd = lane < nw ? s_bd[lane] : INFINITY;
            bi = lane < nw ? s_bi[lane] : INT_MAX;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double od = __shfl_down_sync(0xffffffffu, bd, o);
                const int oi = __shfl_down_sync(0xffffffffu, bi, o);
                if (od < bd || (od == bd && oi < bi)) {
                    bd = od;
                    bi = oi;
                }
            }
            // the face: lane k < d owns component k; the dot products run over k
            // in order on every lane (values gathered by shuffles), the bits of
            // the serial loop
            bi = __shfl_sync(0xffffffffu, bi, 0);
            bd = __shfl_sync(0xffffffffu, bd, 0);  // = dstar[best]
            int best = (bi == INT_MAX) ? -1 : bi;
            if (best >= 0 && bd <= 1e-12) {
                if (lane == 0) set_status(rec + kStatus, EZ_GRADIENT_UNDEFINED);  // inflation.py:423-424
                best = -1;
            }
            if (best >= 0) {
                const double dist = bd;
                double ak = 0.0, ck = 0.0, vk = 0.0, ek = 0.0;
                if (lane < d) {
                    ck = star[static_cast<int64_t>(best) * d + lane];
                    ak = (ck - pstar[static_cast<int64_t>(best) * d + lane]) / dist;
                    vk = v1[lane];
                    ek = e[lane];
                }
                double braw = 0.0, av1 = 0.0, av2 = 0.0, nn = 0.0;
                for (int k = 0; k < d; ++k) {
                    const double a = __shfl_sync(0xffffffffu, ak, k), c = __shfl_sync(0xffffffffu, ck, k);
                    const double v = __shfl_sync(0xffffffffu, vk, k), w = __shfl_sync(0xffffffffu, ek, k);
                    braw = fma(a, c, braw);
                    av1 = fma(a, v, av1);
                    av2 = fma(a, v + w, av2);
                    nn = fma(a, a, nn);
                }
                // compute_step_back (inflation.py:203-212)
                const double rr = (fmax(av1, av2) - braw) + delta_max;
                const double delta = rr > 0.0 ? delta_max - rr : delta_max;
                double rh = braw - delta;
                // HPolytope row normalisation (cpoly.py:32-38)
                const double norm = sqrt(nn);
                if (fabs(norm - 1.0) > 1e-12) {
                    ak /= norm;
                    rh /= norm;
                }
                if (lane < d) {
                    s_a[lane] = ak;
                    A[static_cast<int64_t>(F) * d + lane] = ak;
                }
                if (lane == 0) {
                    s_rhs = rh;
                    b[F] = rh;
                }
            }
            if (lane == 0) s_best = best;
        }
        __syncthreads();
        if (s_best < 0) break;
        ++F;
        ++placed;
        rhs = s_rhs;
    }
    if (threadIdx.x == 0) {
        rec[kFaces] = F;
        it[kPlaced] = placed;
    }
}

// The same placement on a cluster of kPlaceCl CTAs (EI-ZO loop).  One CTA
// re-read every anchor row from L2 in each of the N_f rounds (a single SM's
// L2 bandwidth bound it: ~4 us per round at 10^4 x 7 anchors).  Here CTA r
// owns the contiguous candidate range [r C / K, (r + 1) C / K): its rows,
// distances and alive bytes are staged in its shared memory once; per round
// each CTA takes its arg-min and writes it into every CTA's shared memory
// (distributed shared memory); after one cluster barrier every CTA reduces the
// K results and builds the face exactly as k_place does (rank 0 stores it).
// One cluster barrier per round (two, with rank 0 broadcasting the face, cost
// 185 us per 7-DOF region).  Same decisions and bits as k_place (global index
// tie-break, same dot-product order).
#ifndef EZ_PLACE_CL
#define EZ_PLACE_CL 8
#endif
#ifndef EZ_PLACE_CL_THREADS
#define EZ_PLACE_CL_THREADS 512
#endif
constexpr int kPlaceCl = EZ_PLACE_CL;
constexpr int kPlaceClThreads = EZ_PLACE_CL_THREADS;
__host__ __device__ inline int place_cl_slice(int n) { return (n + kPlaceCl - 1) / kPlaceCl; }
inline size_t place_cl_smem_bytes(int n, int d) {
    return static_cast<size_t>(place_cl_slice(n)) * (static_cast<size_t>(d) + 1) * sizeof(double) +
           static_cast<size_t>(place_cl_slice(n));
}

__global__ void __cluster_dims__(kPlaceCl, 1, 1) __launch_bounds__(kPlaceClThreads)
k_place_cl(double* __restrict__ A, double* __restrict__ b, int32_t* __restrict__ rec, int32_t* __restrict__ it, int d,
           const double* __restrict__ star, const double* __restrict__ pstar, const double* __restrict__ dstar,
           const double* __restrict__ seg, double delta_max, int n_f) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) uint8_t smem_pcl[];
    __shared__ double s_bd[32];
    __shared__ int s_bi[32];
    __shared__ double s_cbd[2][kPlaceCl];  // every CTA's result, by round parity
    __shared__ int s_cbi[2][kPlaceCl];
    __shared__ double s_a[32];
    __shared__ double s_rhs;
    __shared__ int s_best;
    if (rec[kStatus] != EZ_OK || rec[kStop]) return;  // the same for every CTA of the cluster
    const int C = it[kNumCand];
    const int rank = static_cast<int>(cluster.block_rank());
    const int slice = place_cl_slice(C);
    const int lo = min(C, rank * slice), n = min(C, lo + slice) - lo;
    double* s_rows = reinterpret_cast<double*>(smem_pcl);
    double* s_dist = s_rows + static_cast<size_t>(slice) * d;
    uint8_t* alive = reinterpret_cast<uint8_t*>(s_dist + slice);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < n * d; i += blockDim.x) s_rows[i] = star[static_cast<int64_t>(lo) * d + i];
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        s_dist[i] = dstar[lo + i];
        alive[i] = 1;
    }
    cluster.sync();  // every CTA of the cluster is running before any DSMEM access
    int F = rec[kFaces];
    int placed = 0;
    const double* v1 = seg;
    const double* e = seg + d;
    double rhs = 0.0;
    for (int r = 0; r < n_f; ++r) {
        const int par = r & 1;
        __syncthreads();
        double bd = INFINITY;
        int bi = INT_MAX;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            if (!alive[i]) continue;
            if (r > 0) {
                const double* t = s_rows + static_cast<size_t>(i) * d;
                double dot = 0.0;
                for (int k = 0; k < d; ++k) dot = fma(t[k], s_a[k], dot);
                if (!(dot <= rhs)) {
                    alive[i] = 0;
                    continue;
                }
            }
            const double di = s_dist[i];
            if (di < bd) {  // ascending i per thread: ties keep the lower index
                bd = di;
                bi = lo + i;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double od = __shfl_down_sync(0xffffffffu, bd, o);
            const int oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (od < bd || (od == bd && oi < bi)) {
                bd = od;
                bi = oi;
            }
        }
        if (lane == 0) {
            s_bd[wid] = bd;
            s_bi[wid] = bi;
        }
        __syncthreads();
        if (wid == 0) {
            const int nw = blockDim.x >> 5;
            bd = lane < nw ? s_bd[lane] : INFINITY;
            bi = lane < nw ? s_bi[lane] : INT_MAX;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double od = __shfl_down_sync(0xffffffffu, bd, o);
                const int oi = __shfl_down_sync(0xffffffffu, bi, o);
                if (od < bd || (od == bd && oi < bi)) {
                    bd = od;
                    bi = oi;
                }
            }
            // this CTA's result into slot `rank` of every CTA (lane q writes CTA q)
            bd = __shfl_sync(0xffffffffu, bd, 0);
            bi = __shfl_sync(0xffffffffu, bi, 0);
            if (lane < kPlaceCl) {
                *cluster.map_shared_rank(&s_cbd[par][rank], lane) = bd;
                *cluster.map_shared_rank(&s_cbi[par][rank], lane) = bi;
            }
        }
        // One cluster barrier per round: every CTA reduces the same K results
        // and builds the same face (slots alternate by round parity, so a CTA
        // one round ahead never overwrites values another is still reading)
        cluster.sync();
        if (wid == 0) {
            bd = lane < kPlaceCl ? s_cbd[par][lane] : INFINITY;
            bi = lane < kPlaceCl ? s_cbi[par][lane] : INT_MAX;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double od = __shfl_down_sync(0xffffffffu, bd, o);
                const int oi = __shfl_down_sync(0xffffffffu, bi, o);
                if (od < bd || (od == bd && oi < bi)) {
                    bd = od;
                    bi = oi;
                }
            }
            bi = __shfl_sync(0xffffffffu, bi, 0);
            bd = __shfl_sync(0xffffffffu, bd, 0);  // = dstar[best]
            int best = (bi == INT_MAX) ? -1 : bi;
            if (best >= 0 && bd <= 1e-12) {
                if (lane == 0 && rank == 0) set_status(rec + kStatus, EZ_GRADIENT_UNDEFINED);  // inflation.py:423-424
                best = -1;
            }
            double ak = 0.0, rh = 0.0;
            if (best >= 0) {
                const double dist = bd;
                double ck = 0.0, vk = 0.0, ek = 0.0;
                if (lane < d) {
                    ck = star[static_cast<int64_t>(best) * d + lane];
                    ak = (ck - pstar[static_cast<int64_t>(best) * d + lane]) / dist;
                    vk = v1[lane];
                    ek = e[lane];
                }
                double braw = 0.0, av1 = 0.0, av2 = 0.0, nn = 0.0;
                for (int k = 0; k < d; ++k) {
                    const double a = __shfl_sync(0xffffffffu, ak, k), c = __shfl_sync(0xffffffffu, ck, k);
                    const double v = __shfl_sync(0xffffffffu, vk, k), w = __shfl_sync(0xffffffffu, ek, k);
                    braw = fma(a, c, braw);
                    av1 = fma(a, v, av1);
                    av2 = fma(a, v + w, av2);
                    nn = fma(a, a, nn);
                }
                // compute_step_back (inflation.py:203-212)
                const double rr = (fmax(av1, av2) - braw) + delta_max;
                const double delta = rr > 0.0 ? delta_max - rr : delta_max;
                rh = braw - delta;
                // HPolytope row normalisation (cpoly.py:32-38)
                const double norm = sqrt(nn);
                if (fabs(norm - 1.0) > 1e-12) {
                    ak /= norm;
                    rh /= norm;
                }
                if (rank == 0) {
                    if (lane < d) A[static_cast<int64_t>(F) * d + lane] = ak;
                    if (lane == 0) b[F] = rh;
                }
                if (lane < d) s_a[lane] = ak;
            }
            if (lane == 0) {
                s_rhs = rh;
                s_best = best;
            }
        }
        __syncthreads();
        if (s_best < 0) break;
        ++F;
        ++placed;
        rhs = s_rhs;
    }
    if (rank == 0 && threadIdx.x == 0) {
        rec[kFaces] = F;
        it[kPlaced] = placed;
    }
}

}  // namespace ez

// ---------------------------------------------------------------------------
// workspace
// ---------------------------------------------------------------------------
struct ez_eizo_ws {
    int32_t d = 0;
    int64_t n_cap = 0;      // samples
    int32_t c_cap = 0;      // candidates (n_p)
    int32_t f_cap = 0;      // faces
    double* A = nullptr;
    double* b = nullptr;
    double* Ap = nullptr;   // padded faces for the tensor-core walk
    int64_t ap_cap = 0;
    double* Z = nullptr;    // counter-stream draws of one sample batch (k_draws)
    int64_t z_cap = 0;
    double* Z2[2] = {nullptr, nullptr};  // EI-ZO loop: draws of iterations k (even/odd), made on `side`
    int64_t z2_cap = 0;
    cudaStream_t side = nullptr;
    cudaEvent_t ev_draws[2] = {nullptr, nullptr};
    cudaEvent_t ev_walked[2] = {nullptr, nullptr};
    cudaEvent_t ev_fork = nullptr;  // orders the side stream after an inflation's setup
    double* X = nullptr;
    uint8_t* flags = nullptr;
    int32_t* col = nullptr;
    double* star = nullptr;
    double* pstar = nullptr;
    double* dstar = nullptr;
    double* seg = nullptr;  // v1 | e | v2
    int32_t* rec = nullptr;
    int32_t* h_rec = nullptr;  // pinned
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t ev_it[2] = {nullptr, nullptr};
};

namespace ez {

void eizo_ws_free(ez_eizo_ws* ws) {
    if (!ws) return;
    cudaFree(ws->A);
    cudaFree(ws->b);
    cudaFree(ws->Ap);
    cudaFree(ws->Z);
    cudaFree(ws->Z2[0]);
    cudaFree(ws->Z2[1]);
    if (ws->side) cudaStreamDestroy(ws->side);
    for (cudaEvent_t e : ws->ev_draws)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : ws->ev_walked)
        if (e) cudaEventDestroy(e);
    if (ws->ev_fork) cudaEventDestroy(ws->ev_fork);
    cudaFree(ws->X);
    cudaFree(ws->flags);
    cudaFree(ws->col);
    cudaFree(ws->star);
    cudaFree(ws->pstar);
    cudaFree(ws->dstar);
    cudaFree(ws->seg);
    cudaFree(ws->rec);
    cudaFreeHost(ws->h_rec);
    if (ws->stream) cudaStreamDestroy(ws->stream);
    if (ws->ev0) cudaEventDestroy(ws->ev0);
    if (ws->ev1) cudaEventDestroy(ws->ev1);
    for (cudaEvent_t e : ws->ev_it)
        if (e) cudaEventDestroy(e);
    delete ws;
}

template <typename Tp>
static int32_t grow(Tp** p, int64_t old_n, int64_t new_n, bool keep) {
    Tp* q = nullptr;
    EZ_CUDA(cudaMalloc(&q, sizeof(Tp) * std::max<int64_t>(1, new_n)));
    if (keep && *p && old_n > 0) EZ_CUDA(cudaMemcpy(q, *p, sizeof(Tp) * old_n, cudaMemcpyDeviceToDevice));
    cudaFree(*p);
    *p = q;
    return EZ_OK;
}

// EI-ZO workspaces: a small pool per device, shared by every world on it, so
// repeated inflations with fresh checkers never allocate inside the loop and
// independent inflations (several segments of a path) can run concurrently,
// each on its own stream, from different host threads.
struct WsPool {
    std::mutex mu;
    std::vector<ez_eizo_ws*> all;
    std::vector<bool> busy;
};
static WsPool g_pool[64];

static int32_t ws_create(ez_eizo_ws** out) {
    ez_eizo_ws* slot = new ez_eizo_ws();
    *out = slot;
    // the loop's critical path at high priority, the ahead-of-time draws
    // (side stream) at low priority: they fill the gaps instead of competing
    // with the walk, bisection and placement for SMs
    int prio_lo = 0, prio_hi = 0;
    EZ_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    EZ_CUDA(cudaStreamCreateWithPriority(&slot->stream, cudaStreamNonBlocking, prio_hi));
    EZ_CUDA(cudaEventCreate(&slot->ev0));
    EZ_CUDA(cudaEventCreate(&slot->ev1));
    EZ_CUDA(cudaEventCreateWithFlags(&slot->ev_it[0], cudaEventDisableTiming));
    EZ_CUDA(cudaEventCreateWithFlags(&slot->ev_it[1], cudaEventDisableTiming));
    EZ_CUDA(cudaMalloc(&slot->rec, kRecInts * sizeof(int32_t)));
    EZ_CUDA(cudaMallocHost(&slot->h_rec, 2 * kRecInts * sizeof(int32_t)));
    EZ_CUDA(cudaMalloc(&slot->seg, sizeof(double) * 3 * 64));
    EZ_CUDA(cudaStreamCreateWithPriority(&slot->side, cudaStreamNonBlocking, prio_lo));
    for (int i = 0; i < 2; ++i) {
        EZ_CUDA(cudaEventCreateWithFlags(&slot->ev_draws[i], cudaEventDisableTiming));
        EZ_CUDA(cudaEventCreateWithFlags(&slot->ev_walked[i], cudaEventDisableTiming));
    }
    EZ_CUDA(cudaEventCreateWithFlags(&slot->ev_fork, cudaEventDisableTiming));
    return EZ_OK;
}

// Take a free workspace of device `dev` from its pool (creating one if all are
// busy) / give it back.
static int32_t ws_acquire(int dev, ez_eizo_ws** out) {
    WsPool& P = g_pool[dev & 63];
    std::lock_guard<std::mutex> lk(P.mu);
    for (size_t i = 0; i < P.all.size(); ++i)
        if (!P.busy[i]) {
            P.busy[i] = true;
            *out = P.all[i];
            return EZ_OK;
        }
    ez_eizo_ws* n = nullptr;
    const int32_t st = ws_create(&n);
    if (st != EZ_OK) {
        eizo_ws_free(n);
        return st;
    }
    P.all.push_back(n);
    P.busy.push_back(true);
    *out = n;
    return EZ_OK;
}

static void ws_release(int dev, ez_eizo_ws* ws) {
    if (!ws) return;
    WsPool& P = g_pool[dev & 63];
    std::lock_guard<std::mutex> lk(P.mu);
    for (size_t i = 0; i < P.all.size(); ++i)
        if (P.all[i] == ws) P.busy[i] = false;
}

// A workspace of the current device for the duration of one call.
struct WsLease {
    int device = 0;
    ez_eizo_ws* ws = nullptr;
    int32_t acquire(int dev) {
        device = dev;
        return ws_acquire(dev, &ws);
    }
    ~WsLease() { ws_release(device, ws); }
};

static int32_t ws_reserve(ez_eizo_ws* ws, int d, int64_t n, int32_t c, int32_t f, int n_ms) {
    if (ws->d != d) {
        ws->n_cap = ws->c_cap = ws->f_cap = 0;
        ws->d = d;
    }
    if (n > ws->n_cap) {
        EZ_TRY(grow(&ws->X, 0, n * d, false));
        EZ_TRY(grow(&ws->flags, 0, n, false));
        ws->n_cap = n;
    }
    if (c > ws->c_cap) {
        EZ_TRY(grow(&ws->col, 0, c, false));
        EZ_TRY(grow(&ws->star, 0, static_cast<int64_t>(c) * d, false));
        EZ_TRY(grow(&ws->pstar, 0, static_cast<int64_t>(c) * d, false));
        EZ_TRY(grow(&ws->dstar, 0, c, false));
        ws->c_cap = c;
    }
    if (f > ws->f_cap) {
        EZ_TRY(grow(&ws->A, static_cast<int64_t>(ws->f_cap) * d, static_cast<int64_t>(f) * d, true));
        EZ_TRY(grow(&ws->b, ws->f_cap, f, true));
        ws->f_cap = f;
    }
    if (hnr_ap_words(f, d) > ws->ap_cap) {
        EZ_TRY(grow(&ws->Ap, 0, hnr_ap_words(f, d), false));
        ws->ap_cap = hnr_ap_words(f, d);
    }
    if (n * n_ms * (d + 1) > ws->z2_cap) {
        // the side stream may still be filling a buffer of the previous call
        if (ws->side) EZ_CUDA(cudaStreamSynchronize(ws->side));
        for (int i = 0; i < 2; ++i) EZ_TRY(grow(&ws->Z2[i], 0, n * n_ms * (d + 1), false));
        ws->z2_cap = n * n_ms * (d + 1);
    }
    return EZ_OK;
}

// padded shared-memory row stride: even, with an odd number of 16-byte units
static int hnr_lda(int d) {
    int l = d + (d & 1);
    if ((l / 2) % 2 == 0) l += 2;
    return l;
}

template <int MAXD, int RNG, int LPW, int BT>
static int32_t launch_hnr_t(cudaStream_t s, const double* A, const double* b, const int32_t* F_dev,
                            int F, int smem_faces, int d, const double* seeds, int64_t n_seeds, const double* seg,
                            int64_t count, int n_ms, uint64_t seed, uint64_t walk_offset, double* out,
                            int32_t* status, const double* Z) {
    auto k = k_hnr<MAXD, RNG, LPW, BT>;
    const int lda = hnr_lda(d);
    const size_t smem = static_cast<size_t>(smem_faces) * (lda + 1) * sizeof(double);
    if (smem > 48 * 1024) EZ_TRY(allow_max_dyn_smem(k));
    const int64_t threads = count * LPW;
    const unsigned grid = static_cast<unsigned>((threads + BT - 1) / BT);
    k<<<grid, BT, smem, s>>>(A, b, F_dev, F, d, seeds, n_seeds, seg, count, n_ms, seed, walk_offset, out, status,
                             smem_faces, lda, Z);
    EZ_CUDA(cudaGetLastError());
    return EZ_OK;
}

// Launch shape: lanes per walk (LPW), CTA size and face staging.  Each lane
// owns every LPW-th face, so fewer lanes per walk means more walks read each
// staged face row at once (less shared-memory traffic per FMA) but fewer
// walks in flight.  Cost model per candidate: the per-lane step cost (faces +
// draw loads + shuffle reductions; unstaged faces read through L1 cost about
// 2.5x) times the busiest SM's load, as issue throughput (its warps at IPC 2)
// or as latency (its rounds of resident CTAs, ~4 cycles per dependent
// instruction), whichever is larger.  Small CTAs spread a 1e4-walk batch over
// all SMs instead of leaving a third of them idle.
struct HnrShape {
    int lpw, bt;
    bool staged;
};

static HnrShape hnr_pick(int maxd, int d, int f, int64_t count, int num_sms, int optin) {
    const HnrShape cands[8] = {{maxd, 128, true}, {maxd, 512, true}, {8, 512, true}, {8, 128, true},
                               {4, 512, true},    {4, 128, true},    {maxd, 128, false}, {maxd, 512, false}};
    const size_t smem = static_cast<size_t>(f) * (hnr_lda(d) + 1) * sizeof(double);
    HnrShape best = {maxd, 128, false};
    double best_t = 1e300;
    for (const HnrShape& c : cands) {
        if (c.lpw > maxd) continue;
        if (c.bt == 512 && maxd > 16) continue;
        if (c.lpw != maxd && !((c.lpw == 8 && maxd == 16) || (c.lpw == 4 && (maxd == 8 || maxd == 16)))) continue;
        if (c.staged && smem > static_cast<size_t>(optin) - 2048) continue;
        int per_sm = 65536 / (128 * c.bt);
        if (c.staged) per_sm = std::min<int>(per_sm, static_cast<int>((228 * 1024) / (smem + 1024)));
        if (per_sm < 1) continue;
        const double ctas = std::ceil(static_cast<double>(count) * c.lpw / c.bt);
        const double face = std::ceil(static_cast<double>(f) / c.lpw) * (2.5 * d + 12.0) * (c.staged ? 1.0 : 2.5);
        const double cost = face + std::ceil(static_cast<double>(d) / c.lpw) * 20.0 +
                            14.0 * std::log2(static_cast<double>(c.lpw)) + 60.0;
        const double thr = std::ceil(ctas / num_sms) * (c.bt / 32) * cost / 2.0;
        const double lat = std::ceil(ctas / (static_cast<double>(num_sms) * per_sm)) * cost * 4.0;
        const double t = std::max(thr, lat);
        if (t < best_t * 0.97) {
            best_t = t;
            best = c;
        }
    }
    return best;
}

template <int MAXD>
static int32_t launch_hnr(const ez_world* w, int rng, cudaStream_t s, const double* A, const double* b,
                          const int32_t* F_dev, int F, int f_bound, int d, const double* seeds, int64_t n_seeds,
                          const double* seg, int64_t count, int n_ms, uint64_t seed, uint64_t walk_offset, double* out,
                          int32_t* status, const double* Z) {
    int optin = 0, sms = 0;
    if (w) {
        optin = w->smem_optin;
        sms = w->num_sms;
    } else {
        int dev = 0;
        EZ_CUDA(cudaGetDevice(&dev));
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int fmax = std::max(F, f_bound);
    const HnrShape sh = hnr_pick(MAXD, d, fmax, count, sms, optin);
    const int smem_faces = sh.staged ? fmax : 0;
#define EZ_HNR_GO(LPW_, BT_)                                                                                      \
    return (rng == EZ_RNG_PHILOX)                                                                                  \
               ? launch_hnr_t<MAXD, EZ_RNG_PHILOX, LPW_, BT_>(s, A, b, F_dev, F, smem_faces, d, seeds, n_seeds,    \
                                                               seg, count, n_ms, seed, walk_offset, out, status, Z) \
               : launch_hnr_t<MAXD, EZ_RNG_COUNTER, LPW_, BT_>(s, A, b, F_dev, F, smem_faces, d, seeds, n_seeds,   \
                                                                seg, count, n_ms, seed, walk_offset, out, status, Z)
    if constexpr (MAXD <= 16) {
        if (sh.lpw == MAXD && sh.bt == 512) { EZ_HNR_GO(MAXD, 512); }
    }
    if constexpr (MAXD == 16 || MAXD == 8) {
        if (sh.lpw == 4 && sh.bt == 512) { EZ_HNR_GO(4, 512); }
        if (sh.lpw == 4) { EZ_HNR_GO(4, 128); }
        if constexpr (MAXD == 16) {
            if (sh.lpw == 8 && sh.bt == 512) { EZ_HNR_GO(8, 512); }
            if (sh.lpw == 8) { EZ_HNR_GO(8, 128); }
        }
    }
    EZ_HNR_GO(MAXD, 128);
#undef EZ_HNR_GO
}

// Counter-stream walks run on the FP64 tensor cores at every face count
// (measured: 7-DOF region 3.34 -> 2.81 ms with 14-64 faces); the lane-per-face
// walk serves the Philox stream (EZ_HNR_MMA_FACES / EZ_HNR_NO_MMA override).
constexpr int kMmaFaces = 0;

template <int KC>
static int32_t launch_hnr_mma(cudaStream_t s, const double* Ap, const int32_t* F_dev, int F, int d,
                              const double* seeds, int64_t n_seeds, const double* seg, int64_t count, int n_ms,
                              uint64_t seed, uint64_t walk_offset, double* out, int32_t* status, const double* Z) {
    const int64_t warps = (count + 7) / 8;
    k_hnr_mma<KC><<<static_cast<unsigned>((warps + 1) / 2), 64, 0, s>>>(Ap, F_dev, F, d, seeds, n_seeds, seg, count,
                                                                          n_ms, seed, walk_offset, out, status, Z);
    EZ_CUDA(cudaGetLastError());
    return EZ_OK;
}

// f_bound: largest face count the walk may see (faces live on the device in
// the EI-ZO loop).  Ap: scratch of at least hnr_ap_words(f_bound, d) doubles
// for the tensor-core path, Z: scratch of hnr_draw_words(count, n_ms, d)
// doubles for the counter-stream draws; nullptr = allocated on the stream.
static int64_t hnr_draw_words(int64_t count, int n_ms, int d) { return count * n_ms * (d + 1); }

static int32_t dispatch_hnr(const ez_world* w, int rng, cudaStream_t s, const double* A, const double* b,
                            const int32_t* F_dev, int F, int f_bound, int d, const double* seeds, int64_t n_seeds,
                            const double* seg, int64_t count, int n_ms, uint64_t seed, uint64_t walk_offset,
                            double* out, int32_t* status, double* Ap = nullptr, double* Z = nullptr,
                            bool z_ready = false) {
    if (d > 32) return fail(EZ_UNSUPPORTED, "hit-and-run supports dimension <= 32");
    const int fmax = std::max(F, f_bound);
    double* z = nullptr;
    if (rng == EZ_RNG_COUNTER && !(Z && z_ready)) {
        z = Z;
        if (!z) EZ_CUDA(cudaMallocAsync(&z, sizeof(double) * hnr_draw_words(count, n_ms, d), s));
        launch_draws(s, seed, walk_offset, count, d, n_ms, z, status);
        EZ_CUDA(cudaGetLastError());
    } else if (rng == EZ_RNG_COUNTER) {
        z = Z;
    }
    int32_t st;
    static const int mma_faces = [] {
        const char* e = getenv("EZ_HNR_MMA_FACES");
        return e ? atoi(e) : kMmaFaces;
    }();
    if (rng == EZ_RNG_COUNTER && fmax >= mma_faces && d <= 31 && !getenv("EZ_HNR_NO_MMA")) {
        const int kp = hnr_mma_kp(d);
        double* ap = Ap;
        if (!ap) EZ_CUDA(cudaMallocAsync(&ap, sizeof(double) * hnr_ap_words(fmax, d), s));
        k_pack_faces<<<64, 256, 0, s>>>(A, b, F_dev, F, d, kp, ap);
        if (kp == 8) st = launch_hnr_mma<2>(s, ap, F_dev, F, d, seeds, n_seeds, seg, count, n_ms, seed, walk_offset, out, status, z);
        else if (kp == 16) st = launch_hnr_mma<4>(s, ap, F_dev, F, d, seeds, n_seeds, seg, count, n_ms, seed, walk_offset, out, status, z);
        else st = launch_hnr_mma<8>(s, ap, F_dev, F, d, seeds, n_seeds, seg, count, n_ms, seed, walk_offset, out, status, z);
        if (!Ap) cudaFreeAsync(ap, s);
    } else if (d <= 4) {
        st = launch_hnr<4>(w, rng, s, A, b, F_dev, F, f_bound, d, seeds, n_seeds, seg, count, n_ms, seed, walk_offset, out, status, z);
    } else if (d <= 8) {
        st = launch_hnr<8>(w, rng, s, A, b, F_dev, F, f_bound, d, seeds, n_seeds, seg, count, n_ms, seed, walk_offset, out, status, z);
    } else if (d <= 16) {
        st = launch_hnr<16>(w, rng, s, A, b, F_dev, F, f_bound, d, seeds, n_seeds, seg, count, n_ms, seed, walk_offset, out, status, z);
    } else {
        st = launch_hnr<32>(w, rng, s, A, b, F_dev, F, f_bound, d, seeds, n_seeds, seg, count, n_ms, seed, walk_offset, out, status, z);
    }
    if (z && !Z) cudaFreeAsync(z, s);
    return st;
}

template <typename T, int MAXD>
static int32_t launch_bisect_t(ez_world* w, ez_eizo_ws* ws, const ModelDev<T>& M, cudaStream_t s, const int32_t* it,
                               int n_p, int d, double ee, int n_b, double t_col) {
    constexpr int G = kBisectLanes, CPB = 128 / G;
    size_t smem = M.blob_bytes + static_cast<size_t>(M.cen_words) * CPB * sizeof(T);
    smem = (smem + 15) & ~static_cast<size_t>(15);
    smem += static_cast<size_t>(CPB) * d * sizeof(double);
    smem = (smem + 15) & ~static_cast<size_t>(15);
    // two levels per round (k_bisect2, a warp per candidate) unless
    // EZ_BISECT1=1 asks for the one-step loop (8 lanes per candidate)
    static const bool one_step = [] {
        const char* e = getenv("EZ_BISECT1");
        return e && e[0] == '1';
    }();
    auto kern = one_step ? k_bisect<T, MAXD, G> : k_bisect2<T, MAXD>;
    const int cpb = one_step ? CPB : 128 / 32;
    if (smem > static_cast<size_t>(w->smem_optin) - 1024) return fail(EZ_CAPACITY, "robot model too large for one bisection CTA");
    if (smem > 48 * 1024) EZ_TRY(allow_max_dyn_smem(kern));
    kern<<<static_cast<unsigned>((n_p + cpb - 1) / cpb), 128, smem, s>>>(M, static_cast<T>(w->margin), ws->X, d, ws->col,
                                                                     ws->rec, it, ws->seg, ee, n_b, t_col, ws->star,
                                                                     ws->pstar, ws->dstar);
    EZ_CUDA(cudaGetLastError());
    return EZ_OK;
}

template <int MAXD>
static int32_t launch_bisect(ez_world* w, ez_eizo_ws* ws, int precision, cudaStream_t s, const int32_t* it, int n_p,
                             int d, double ee,
                             int n_b, double t_col) {
    if (precision == EZ_F64) return launch_bisect_t<double, MAXD>(w, ws, w->md, s, it, n_p, d, ee, n_b, t_col);
    // fp32 checks on a specialised world with a light model: the bisection on
    // the model's own code, one thread per checked point (ez_bisect_core.cuh;
    // same points as k_bisect2).  A heavy model's single-thread check is too
    // long a chain: the 14-DOF bisection (1,248 pairs) takes 24.1 ms per region
    // in k_bisect2's 8-lane cooperative checks against 29.8 ms here (7-DOF:
    // 534 -> 234 us).  EZ_BISECT_JIT=0 / 1 (read per call) forces either way.
    const char* bj = getenv("EZ_BISECT_JIT");
    const char* b1 = getenv("EZ_BISECT1");
    const bool use_jit = bj && (bj[0] == '0' || bj[0] == '1') ? bj[0] == '1' : w->n_pairs <= 600;
    if (d == w->dof && use_jit && !(b1 && b1[0] == '1')) {
        const std::shared_ptr<const JitCheck> jc = std::atomic_load(&w->jit);
        if (jc && jc->bk)
            return jit_bisect_launch(w, *jc, ws->X, ws->col, ws->rec, it + kNumCand, n_p, ws->seg, ee, n_b, t_col,
                                     ws->star, ws->pstar, ws->dstar, s);
    }
    return launch_bisect_t<float, MAXD>(w, ws, w->mf, s, it, n_p, d, ee, n_b, t_col);
}

}  // namespace ez

using namespace ez;

extern "C" int32_t ez_hit_and_run(const double* d_A, const double* d_b, int32_t n_faces, int32_t dim,
                                  const double* d_seeds, int64_t n_seeds, int64_t count, int32_t n_ms,
                                  uint64_t seed, uint64_t walk_offset, int32_t rng, double* d_out, void* stream) {
    if (count == 0) return EZ_OK;
    if (count < 0) return fail(EZ_INVALID_ARGUMENT, "negative count");
    if (n_ms < 1) return fail(EZ_INVALID_ARGUMENT, "need at least one mixing step");
    if (dim < 1 || n_faces < 0 || n_seeds < 1) return fail(EZ_INVALID_ARGUMENT, "bad polytope or seed shape");
    if (rng != EZ_RNG_COUNTER && rng != EZ_RNG_PHILOX) return fail(EZ_INVALID_ARGUMENT, "unknown rng");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int32_t* d_status = nullptr;
    EZ_TRY(retain_async_pool());
    EZ_CUDA(cudaMallocAsync(&d_status, 2 * sizeof(int32_t), s));  // (status, stop)
    EZ_CUDA(cudaMemsetAsync(d_status, 0, 2 * sizeof(int32_t), s));
    k_seed_check<<<static_cast<unsigned>((n_seeds + 127) / 128), 128, 0, s>>>(d_A, d_b, n_faces, dim, d_seeds, n_seeds, d_status);
    int32_t st = dispatch_hnr(nullptr, rng, s, d_A, d_b, nullptr, n_faces, n_faces, dim, d_seeds, n_seeds, nullptr, count, n_ms,
                              seed, walk_offset, d_out, d_status);
    int32_t h_status = 0;
    if (st == EZ_OK) {
        cudaError_t e = cudaMemcpyAsync(&h_status, d_status, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) st = cuda_fail(e, "hit-and-run status", __FILE__, __LINE__);
    }
    cudaFreeAsync(d_status, s);
    if (st != EZ_OK) return st;
    if (h_status == EZ_SEED_OUTSIDE) return fail(EZ_SEED_OUTSIDE, "walk seed outside the polytope");
    if (h_status == EZ_EMPTY_CHORD) return fail(EZ_EMPTY_CHORD, "no feasible chord; polytope numerically degenerate");
    if (h_status != EZ_OK) return fail(h_status, "hit-and-run failed");
    return EZ_OK;
}

// the polytope of the last ez_inflate_edge on this thread that overflowed face_cap
static thread_local std::vector<double> g_last_faces;
static thread_local int g_last_dim = 0;

// required_batch_size (inflation.py:156-161)
static int64_t batch_size(int k, const ez_eizo_params& p) {
    const double pi = 3.14159265358979311599796346854;  // math.pi
    const double delta_k = 6.0 * p.delta / (pi * pi * (static_cast<double>(k) * k));
    return static_cast<int64_t>(std::ceil(2.0 * std::log(1.0 / delta_k) / (p.eps * (p.tau * p.tau))));
}

extern "C" int32_t ez_inflate_edge(ez_world* w, const double* h_v1, const double* h_v2, int32_t dim,
                                   const double* h_A0, const double* h_b0, int32_t n_faces0,
                                   const ez_eizo_params* params, uint64_t seed, int32_t precision, int32_t rng,
                                   ez_eizo_report* report, double* h_A_out, double* h_b_out, int32_t face_cap) {
    if (!w || !params || !report) return fail(EZ_INVALID_ARGUMENT, "null argument");
    if (dim != w->dof) return fail(EZ_DIMENSION_MISMATCH, "segment/robot dimension mismatch");
    if (dim > 32) return fail(EZ_UNSUPPORTED, "EI-ZO supports dimension <= 32");
    const ez_eizo_params& p = *params;
    if (p.n_p < 1 || p.n_f < 1 || p.n_b < 1 || p.n_ms < 1) return fail(EZ_INVALID_ARGUMENT, "counts must be >= 1");
    if (rng != EZ_RNG_COUNTER && rng != EZ_RNG_PHILOX) return fail(EZ_INVALID_ARGUMENT, "unknown rng");
    EZ_ON_DEVICE(w->device);
    const int d = dim;
    // seed segment strictly inside the domain (inflation.py:274-277), fp64 on the host
    for (int v = 0; v < 2; ++v) {
        const double* x = v ? h_v2 : h_v1;
        double worst = -INFINITY;
        for (int f = 0; f < n_faces0; ++f) {
            double g = 0.0;
            for (int k = 0; k < d; ++k) g += h_A0[f * d + k] * x[k];
            worst = std::max(worst, g - h_b0[f]);
        }
        if (worst >= 0.0) return fail(EZ_SEED_OUTSIDE_DOMAIN, "seed segment must be strictly inside the domain");
    }
    // capacity for 64 iterations up front: no allocation inside the loop
    WsLease lease;
    EZ_TRY(lease.acquire(w->device));
    ez_eizo_ws* ws = lease.ws;
    EZ_TRY(ws_reserve(ws, d, std::max<int64_t>(p.n_p, batch_size(64, p)), p.n_p, n_faces0 + 64 * p.n_f, p.n_ms));
    cudaStream_t s = ws->stream;
    std::vector<double> seg(3 * d);
    double ee = 0.0;
    for (int k = 0; k < d; ++k) {
        seg[k] = h_v1[k];
        seg[d + k] = h_v2[k] - h_v1[k];
        seg[2 * d + k] = h_v2[k];
        ee += seg[d + k] * seg[d + k];
    }
    {  // ee exactly as numpy's e @ e (sequential sum of products)
        double acc = 0.0;
        for (int k = 0; k < d; ++k) acc = acc + seg[d + k] * seg[d + k];
        ee = acc;
    }
    EZ_CUDA(cudaMemcpyAsync(ws->seg, seg.data(), sizeof(double) * 3 * d, cudaMemcpyHostToDevice, s));
    EZ_CUDA(cudaMemcpyAsync(ws->A, h_A0, sizeof(double) * n_faces0 * d, cudaMemcpyHostToDevice, s));
    EZ_CUDA(cudaMemcpyAsync(ws->b, h_b0, sizeof(double) * n_faces0, cudaMemcpyHostToDevice, s));
    EZ_CUDA(cudaMemsetAsync(ws->rec, 0, kRecInts * sizeof(int32_t), s));
    {
        int32_t f0 = n_faces0;
        EZ_CUDA(cudaMemcpyAsync(ws->rec + kFaces, &f0, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    }
    EZ_CUDA(cudaEventRecord(ws->ev0, s));
    if (p.n_p > 200 * 1024) return fail(EZ_UNSUPPORTED, "n_p above 204800 candidates");
    const int place_dcap = place_dist_cap(p.n_p);
    const size_t place_smem = place_smem_bytes(p.n_p, place_dcap);
    if (place_smem > 48 * 1024)
        EZ_TRY(allow_max_dyn_smem(k_place));
    // the cluster placement when a CTA's share of the anchors fits in shared memory
    const size_t place_cl_smem = place_cl_smem_bytes(p.n_p, d);
    const bool place_cl = place_cl_smem <= 200 * 1024 && !getenv("EZ_PLACE_1CTA");
    if (place_cl && place_cl_smem > 48 * 1024) EZ_TRY(allow_max_dyn_smem(k_place_cl));

    // One iteration = hit-and-run, check (+ first-M count), compaction/test,
    // bisection, placement, and a 128-byte record copy.  Iteration k+1 is
    // enqueued before the host waits for k's record (its walk offset and
    // batch size are host-known); if k accepted, k+1's kernels see `stop`
    // and return at once.
    std::vector<int64_t> n_s_of(2), m_of(2);
    auto enqueue = [&](int k, uint64_t woff, int f_known) -> int32_t {
        const int64_t m = batch_size(k, p);
        const double thr = static_cast<double>(m) * (1.0 - p.tau) * p.eps;
        const int64_t n_s = std::max<int64_t>(p.n_p, m);
        int32_t* it = ws->rec + slot_offset(k);
        EZ_CUDA(cudaMemsetAsync(it, 0, 8 * sizeof(int32_t), s));
        // The walk's draws depend only on (seed, walk offset, batch size): they
        // are made on the side stream into this iteration's buffer, overlapping
        // the previous iteration's check, bisection and placement.
        double* zb = nullptr;
        if (rng == EZ_RNG_COUNTER) {
            zb = ws->Z2[k & 1];
            EZ_CUDA(cudaStreamWaitEvent(ws->side, ws->ev_walked[k & 1], 0));  // iteration k - 2 done reading
            launch_draws(ws->side, seed, woff, n_s, d, p.n_ms, zb, ws->rec + kStatus);
            EZ_CUDA(cudaGetLastError());
            EZ_CUDA(cudaEventRecord(ws->ev_draws[k & 1], ws->side));
            EZ_CUDA(cudaStreamWaitEvent(s, ws->ev_draws[k & 1], 0));
        }
        EZ_TRY(dispatch_hnr(w, rng, s, ws->A, ws->b, ws->rec + kFaces, f_known, f_known + 2 * p.n_f, d, nullptr, 1,
                            ws->seg, n_s, p.n_ms, seed, woff, ws->X, ws->rec + kStatus, ws->Ap, zb, zb != nullptr));
        if (zb) EZ_CUDA(cudaEventRecord(ws->ev_walked[k & 1], s));
        EZ_TRY(launch_check(w, ws->X, EZ_F64, n_s, d, ws->flags, precision, s, m, it + kColM));
        k_compact<<<1, 1024, 0, s>>>(ws->flags, n_s, p.n_p, thr, ws->rec, it, ws->col);
        EZ_CUDA(cudaGetLastError());
        if (d <= 4) EZ_TRY(launch_bisect<4>(w, ws, precision, s, it, p.n_p, d, ee, p.n_b, p.t_col));
        else if (d <= 8) EZ_TRY(launch_bisect<8>(w, ws, precision, s, it, p.n_p, d, ee, p.n_b, p.t_col));
        else if (d <= 16) EZ_TRY(launch_bisect<16>(w, ws, precision, s, it, p.n_p, d, ee, p.n_b, p.t_col));
        else EZ_TRY(launch_bisect<32>(w, ws, precision, s, it, p.n_p, d, ee, p.n_b, p.t_col));
        if (place_cl)
            k_place_cl<<<kPlaceCl, kPlaceClThreads, place_cl_smem, s>>>(ws->A, ws->b, ws->rec, it, d, ws->star,
                                                                         ws->pstar, ws->dstar, ws->seg, p.delta_max,
                                                                         p.n_f);
        else
            k_place<<<1, 1024, place_smem, s>>>(ws->A, ws->b, ws->rec, it, d, ws->star, ws->pstar, ws->dstar,
                                                ws->seg, p.delta_max, p.n_f, nullptr, place_dcap);
        EZ_CUDA(cudaGetLastError());
        EZ_CUDA(cudaMemcpyAsync(ws->h_rec + kRecInts * (k & 1), ws->rec, kRecInts * sizeof(int32_t),
                                cudaMemcpyDeviceToHost, s));
        EZ_CUDA(cudaEventRecord(ws->ev_it[k & 1], s));
        n_s_of[k & 1] = n_s;
        m_of[k & 1] = m;
        return EZ_OK;
    };
    auto drain_and_fail = [&](int32_t st, const char* msg) -> int32_t {
        cudaStreamSynchronize(s);
        return fail(st, msg);
    };

    int F = n_faces0;
    uint64_t walk_offset = 0;
    int64_t checks = 0;
    int32_t hyper = 0;
    int k = 1;
    int32_t terminated = 0;
    // the side stream's draws read the status record this call just reset on
    // `s`: without this edge a draw kernel could still see the previous
    // inflation's stop flag and skip its work
    EZ_CUDA(cudaEventRecord(ws->ev_fork, s));
    EZ_CUDA(cudaStreamWaitEvent(ws->side, ws->ev_fork, 0));
    EZ_TRY(enqueue(1, 0, F));
    for (;; ++k) {
        const uint64_t next_offset = walk_offset + static_cast<uint64_t>(n_s_of[k & 1]);
        const bool may_continue = !(p.n_it > 0 && k >= p.n_it);
        const bool fits = (std::max<int64_t>(p.n_p, batch_size(k + 1, p)) <= ws->n_cap) && (F + 2 * p.n_f <= ws->f_cap);
        if (may_continue && fits) EZ_TRY(enqueue(k + 1, next_offset, F + p.n_f));
        EZ_CUDA(cudaEventSynchronize(ws->ev_it[k & 1]));
        const int32_t* g = ws->h_rec + kRecInts * (k & 1);
        const int32_t* r = g + slot_offset(k);
        if (g[kStatus] != EZ_OK) {
            switch (g[kStatus]) {
                case EZ_EMPTY_CHORD: return drain_and_fail(EZ_EMPTY_CHORD, "no feasible chord; polytope numerically degenerate");
                case EZ_SEED_OUTSIDE: return drain_and_fail(EZ_SEED_OUTSIDE, "walk seed outside the polytope");
                case EZ_SEGMENT_IN_COLLISION:
                    return drain_and_fail(EZ_SEGMENT_IN_COLLISION,
                                          "a projection onto the seed segment, or a bisected collision, "
                                          "lies in collision within t_col of the seed segment");
                case EZ_GRADIENT_UNDEFINED: return drain_and_fail(EZ_GRADIENT_UNDEFINED, "candidate collapsed onto the segment");
                default: return drain_and_fail(g[kStatus], "EI-ZO device failure");
            }
        }
        checks += n_s_of[k & 1];
        walk_offset = next_offset;
        if (r[kAccept]) {
            terminated = 0;
            break;
        }
        checks += static_cast<int64_t>(r[kNumCand]) * (1 + p.n_b);
        hyper += r[kPlaced];
        F = g[kFaces];
        if (!may_continue) {
            terminated = 1;
            break;
        }
        if (!fits) {  // grow the workspace, then continue without lookahead for this step
            EZ_CUDA(cudaStreamSynchronize(s));
            EZ_TRY(ws_reserve(ws, d, std::max<int64_t>(ws->n_cap, std::max<int64_t>(p.n_p, batch_size(k + 64, p))),
                              p.n_p, std::max(ws->f_cap, F + 64 * p.n_f), p.n_ms));
            EZ_TRY(enqueue(k + 1, walk_offset, F));
        }
    }
    EZ_CUDA(cudaEventRecord(ws->ev1, s));
    EZ_CUDA(cudaEventSynchronize(ws->ev1));  // also drains the void look-ahead iteration
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ws->ev0, ws->ev1);
    report->iterations = k;
    report->hyperplanes_added = hyper;
    report->collision_checks = checks;
    report->terminated_by = terminated;
    report->n_faces = F;
    report->device_ms = ms;
    if (F > face_cap) {
        // count, then copy: the polytope is kept for this thread and
        // ez_inflate_edge_result hands it out, so a short buffer never loses
        // the device work (the report above is complete)
        std::vector<double>& keep = g_last_faces;
        keep.resize(static_cast<size_t>(F) * (d + 1));
        EZ_CUDA(cudaMemcpyAsync(keep.data(), ws->A, sizeof(double) * F * d, cudaMemcpyDeviceToHost, s));
        EZ_CUDA(cudaMemcpyAsync(keep.data() + static_cast<size_t>(F) * d, ws->b, sizeof(double) * F,
                                cudaMemcpyDeviceToHost, s));
        EZ_CUDA(cudaStreamSynchronize(s));
        g_last_dim = d;
        return fail(EZ_CAPACITY, "face_cap smaller than the result polytope: report->n_faces rows are kept for "
                                 "ez_inflate_edge_result");
    }
    EZ_CUDA(cudaMemcpyAsync(h_A_out, ws->A, sizeof(double) * F * d, cudaMemcpyDeviceToHost, s));
    EZ_CUDA(cudaMemcpyAsync(h_b_out, ws->b, sizeof(double) * F, cudaMemcpyDeviceToHost, s));
    EZ_CUDA(cudaStreamSynchronize(s));
    return EZ_OK;
}

// The polytope of this thread's last ez_inflate_edge that returned EZ_CAPACITY.
extern "C" int32_t ez_inflate_edge_result(double* h_A_out, double* h_b_out, int32_t face_cap, int32_t* n_faces) {
    if (!n_faces) return fail(EZ_INVALID_ARGUMENT, "null argument");
    const int d = g_last_dim;
    const int F = d > 0 ? static_cast<int>(g_last_faces.size() / (d + 1)) : 0;
    *n_faces = F;
    if (F == 0) return fail(EZ_INVALID_ARGUMENT, "no kept polytope on this thread");
    if (F > face_cap || !h_A_out || !h_b_out) return fail(EZ_CAPACITY, "face_cap smaller than the kept polytope");
    std::memcpy(h_A_out, g_last_faces.data(), sizeof(double) * F * d);
    std::memcpy(h_b_out, g_last_faces.data() + static_cast<size_t>(F) * d, sizeof(double) * F);
    g_last_faces.clear();
    g_last_dim = 0;
    return EZ_OK;
}

// Set repair (planner.py:159-224 inner loop): project the reported collisions
// onto the set's seed segment, fail-fast check, N_b bisection rounds, then
// place uncapped step-back faces, discarding candidates whose ORIGINAL
// collision leaves the set.  Appends faces to (A_in, b_in).
extern "C" int32_t ez_refine_set(ez_world* w, const double* h_v1, const double* h_v2, int32_t dim,
                                 const double* h_A, const double* h_b, int32_t n_faces, const double* h_cols,
                                 int32_t n_cols, double delta_max, double t_col, int32_t n_b, int32_t precision,
                                 double* h_A_out, double* h_b_out, int32_t face_cap, int32_t* n_faces_out,
                                 int64_t* collision_checks) {
    if (!w || !h_cols || !n_faces_out) return fail(EZ_INVALID_ARGUMENT, "null argument");
    if (dim != w->dof) return fail(EZ_DIMENSION_MISMATCH, "segment/robot dimension mismatch");
    if (n_cols < 1) return fail(EZ_INVALID_ARGUMENT, "refine_sets needs at least one collision");
    if (n_b < 1) return fail(EZ_INVALID_ARGUMENT, "n_b must be >= 1");
    if (dim > 32) return fail(EZ_UNSUPPORTED, "dimension <= 32");
    EZ_ON_DEVICE(w->device);
    const int d = dim;
    WsLease lease;
    EZ_TRY(lease.acquire(w->device));
    ez_eizo_ws* ws = lease.ws;
    EZ_TRY(ws_reserve(ws, d, n_cols, n_cols, n_faces + n_cols + 1, 0));
    cudaStream_t s = ws->stream;
    std::vector<double> seg(3 * d);
    double ee = 0.0;
    for (int k = 0; k < d; ++k) {
        seg[k] = h_v1[k];
        seg[d + k] = h_v2[k] - h_v1[k];
        seg[2 * d + k] = h_v2[k];
        ee = ee + seg[d + k] * seg[d + k];
    }
    std::vector<int32_t> iota(n_cols);
    for (int i = 0; i < n_cols; ++i) iota[i] = i;
    int32_t rec0[kRecInts] = {0};
    rec0[kFaces] = n_faces;
    rec0[slot_offset(0) + kNumCand] = n_cols;
    EZ_CUDA(cudaMemcpyAsync(ws->seg, seg.data(), sizeof(double) * 3 * d, cudaMemcpyHostToDevice, s));
    EZ_CUDA(cudaMemcpyAsync(ws->A, h_A, sizeof(double) * n_faces * d, cudaMemcpyHostToDevice, s));
    EZ_CUDA(cudaMemcpyAsync(ws->b, h_b, sizeof(double) * n_faces, cudaMemcpyHostToDevice, s));
    EZ_CUDA(cudaMemcpyAsync(ws->X, h_cols, sizeof(double) * n_cols * d, cudaMemcpyHostToDevice, s));
    EZ_CUDA(cudaMemcpyAsync(ws->col, iota.data(), sizeof(int32_t) * n_cols, cudaMemcpyHostToDevice, s));
    EZ_CUDA(cudaMemcpyAsync(ws->rec, rec0, sizeof(rec0), cudaMemcpyHostToDevice, s));
    const int32_t* it = ws->rec + slot_offset(0);
    if (d <= 4) EZ_TRY(launch_bisect<4>(w, ws, precision, s, it, n_cols, d, ee, n_b, t_col));
    else if (d <= 8) EZ_TRY(launch_bisect<8>(w, ws, precision, s, it, n_cols, d, ee, n_b, t_col));
    else if (d <= 16) EZ_TRY(launch_bisect<16>(w, ws, precision, s, it, n_cols, d, ee, n_b, t_col));
    else EZ_TRY(launch_bisect<32>(w, ws, precision, s, it, n_cols, d, ee, n_b, t_col));
    if (n_cols > 200 * 1024) return fail(EZ_UNSUPPORTED, "more than 204800 collisions in one repair");
    const int place_dcap = place_dist_cap(static_cast<int>(n_cols));
    const size_t place_smem = place_smem_bytes(static_cast<int>(n_cols), place_dcap);
    if (place_smem > 48 * 1024)
        EZ_TRY(allow_max_dyn_smem(k_place));
    k_place<<<1, 1024, place_smem, s>>>(ws->A, ws->b, ws->rec, ws->rec + slot_offset(0), d, ws->star, ws->pstar,
                                        ws->dstar, ws->seg, delta_max, n_cols, ws->X, place_dcap);
    EZ_CUDA(cudaGetLastError());
    EZ_CUDA(cudaMemcpyAsync(ws->h_rec, ws->rec, kRecInts * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    EZ_CUDA(cudaStreamSynchronize(s));
    const int32_t* g = ws->h_rec;
    if (g[kStatus] == EZ_SEGMENT_IN_COLLISION)
        return fail(EZ_SEGMENT_IN_COLLISION, "seed segment projection in collision, or a collision within t_col, during repair");
    if (g[kStatus] == EZ_GRADIENT_UNDEFINED) return fail(EZ_GRADIENT_UNDEFINED, "candidate collapsed onto the segment");
    if (g[kStatus] != EZ_OK) return fail(g[kStatus], "repair device failure");
    const int F = g[kFaces];
    if (F > face_cap) return fail(EZ_CAPACITY, "face_cap smaller than the repaired polytope");
    EZ_CUDA(cudaMemcpyAsync(h_A_out, ws->A, sizeof(double) * F * d, cudaMemcpyDeviceToHost, s));
    EZ_CUDA(cudaMemcpyAsync(h_b_out, ws->b, sizeof(double) * F, cudaMemcpyDeviceToHost, s));
    EZ_CUDA(cudaStreamSynchronize(s));
    *n_faces_out = F;
    if (collision_checks) *collision_checks = static_cast<int64_t>(n_cols) * (1 + n_b);
    return EZ_OK;
}

#include "ez_eizo_session.inc"
