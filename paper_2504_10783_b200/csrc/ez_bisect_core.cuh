// ez_bisect_core.cuh — the EI-ZO bisection on the run-time specialised check
// (ez_jit.cu compiles it with the model's JitPolicy).  Replaces
// inflation.py:191-200 (_bisection_batch) with the fail-fast projection check
// (:302-305) and the t_col guard (:307-310), like k_bisect2 in ez_eizo.cu.
//
// 2^L threads per candidate, one checked point each: thread 0 the projection
// (first round only), threads 1 .. 2^L - 1 the nodes of the next L binary
// steps (node 1 = the midpoint of [lo, hi]; node n's children 2n and 2n + 1
// are the midpoints after "collides" (hi = mid) and "free" (lo = mid)).  A
// round then takes the L steps the group's ballot decides.  Every node's point is
// formed from the current ends by the same operations as the one-step loop's
// next midpoints, so the checked points, decisions and star/pstar rows are
// those of k_bisect and k_bisect2 — in ceil(N_b / L) dependent rounds of
// single-thread checks instead of N_b (k_bisect) or ceil(N_b / 2) (k_bisect2)
// rounds of 8-lane cooperative ones — wherever the specialised and the generic
// fp32 checks agree.  They can disagree only inside the fp32 contact band
// (tests/test_gpu_jit.py: |fp64 clearance| < 1e-7 measured on 5M boundary
// points, 0.3% of them), where either decision honours the fp32 contract.
#pragma once

#include "ez_device.cuh"

namespace ez {

// project_batch for one point held whole by the thread (inflation.py:124-137):
// the serial dot products of ez_eizo.cu's project_group, operation for
// operation.
template <int D>
__device__ __forceinline__ double project_point(const double (&c)[D], const double* __restrict__ v1,
                                                const double* __restrict__ e, double ee, double (&p)[D]) {
    double alpha = 0.0;
    if (ee != 0.0) {
        double dot = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) dot = fma(c[k] - v1[k], e[k], dot);
        alpha = fmin(fmax(dot / ee, 0.0), 1.0);
    }
    double ss = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        p[k] = __dadd_rn(v1[k], __dmul_rn(alpha, e[k]));
        const double r = c[k] - p[k];
        ss = fma(r, r, ss);
    }
    return sqrt(ss);
}

// rec[0] status, rec[1] stop (ez_eizo.cu kStatus / kStop); *n_cand = C.  A
// CTA of CTA threads; each group's bracket [lo, hi] lives in shared memory
// (thread t owns components t, t + 2^L, ...), so only the thread's own point is
// live in registers across the check (14-DOF: 28 instead of 84 registers).
// L trades dependent rounds for speculative checks (2^L per L steps);
// measured per region (7-DOF / 14-DOF): L = 2 473 us / 53.7 ms, L = 3 336 us
// / 37.7 ms, L = 4 348 us / 30.8 ms (4 wins once the candidates fit in one
// wave), against k_bisect2's 534 us / 24.0 ms: the 14-DOF model keeps
// k_bisect2 (ez_eizo.cu launch_bisect).  Each point runs the policy's full()
// (one FK; a() then b() computed it three times for a free point): 7-DOF
// 289 -> 234 us per region, 14-DOF 29.8 ms.
//
// L is chosen per launch from the device-side C: 4 when C * 16 threads fit in
// `resident` (the GPU's resident threads for this kernel), else 3; forced_l in
// 1..4 overrides.  Launch grids cover n_p * 16 threads.
template <class P, int D, int CTA>
__device__ __forceinline__ void bisect_points(const P& pol, const double* __restrict__ X, const int32_t* __restrict__ col,
                                              int32_t* __restrict__ rec, const int32_t* __restrict__ n_cand,
                                              const double* __restrict__ seg, double ee, int n_b, double t_col,
                                              double* __restrict__ star, double* __restrict__ pstar,
                                              double* __restrict__ dstar, int64_t resident, int forced_l) {
    __shared__ double s_lo[CTA / 2][D], s_hi[CTA / 2][D];
    const int C = *n_cand;
    if (rec[0] != EZ_OK || rec[1]) return;
    const int L = forced_l >= 1 && forced_l <= 4 ? forced_l : ((static_cast<int64_t>(C) << 4) <= resident ? 4 : 3);
    const int G = 1 << L;  // threads per candidate: the projection + 2^L - 1 tree nodes
    const unsigned kGroup = G == 32 ? 0xffffffffu : (1u << G) - 1u;
    const int64_t gt = static_cast<int64_t>(blockIdx.x) * CTA + threadIdx.x;
    const int i = static_cast<int>(gt >> L), t = static_cast<int>(gt & (G - 1));
    if (i >= C) return;  // whole groups leave together
    const int sh = (threadIdx.x & 31) & ~(G - 1);
    const unsigned gm = kGroup << sh;
    double* lo = s_lo[threadIdx.x >> L];
    double* hi = s_hi[threadIdx.x >> L];
    const double* v1 = seg;
    const double* e = seg + D;
    if (t == 0) {
        double c[D], p[D];
        const double* xc = X + static_cast<int64_t>(col[i]) * D;
#pragma unroll
        for (int k = 0; k < D; ++k) c[k] = xc[k];
        project_point<D>(c, v1, e, ee, p);
#pragma unroll
        for (int k = 0; k < D; ++k) {
            lo[k] = p[k];
            hi[k] = c[k];
        }
    }
    __syncwarp(gm);
    const int depth = t ? 31 - __clz(t) : 0;  // of node t (t >= 1)
    bool first = true;
    for (int done = 0; first || done < n_b;) {
        const int lv = min(L, n_b - done);  // binary steps taken this round
        const bool active = t == 0 ? first : depth < lv;
        bool fr = true;
        if (active) {
            double pt[D];
#pragma unroll
            for (int k = 0; k < D; ++k) {
                double a = lo[k], b = hi[k];
                if (t != 0) {
                    for (int l = depth - 1; l >= 0; --l) {  // the path to node t, root first
                        const double m = 0.5 * (a + b);
                        if ((t >> l) & 1) a = m;
                        else b = m;
                    }
                }
                pt[k] = t == 0 ? a : 0.5 * (a + b);
            }
#ifdef EZ_BISECT_AB
            fr = !pol.a(pt, static_cast<float*>(nullptr)) && !pol.b(pt, static_cast<float*>(nullptr));
#else
            fr = !pol.full(pt, static_cast<float*>(nullptr));  // one FK per point
#endif
        }
        const unsigned bal = (__ballot_sync(gm, fr) >> sh) & kGroup;
        if (first) {
            if (!(bal & 1u)) {
                if (t == 0) atomicCAS(rec, 0, static_cast<int32_t>(EZ_SEGMENT_IN_COLLISION));  // inflation.py:303-305
                return;
            }
            first = false;
        }
        __syncwarp(gm);  // every point of this round is read
        for (int k = t; k < D; k += G) {
            double a = lo[k], b = hi[k];
            int node = 1;
            for (int l = 0; l < lv; ++l) {
                const bool f = (bal >> node) & 1u;
                const double m = 0.5 * (a + b);
                if (f) a = m;
                else b = m;
                node = 2 * node + (f ? 1 : 0);
            }
            lo[k] = a;
            hi[k] = b;
        }
        __syncwarp(gm);
        done += lv;
    }
    if (t != 0) return;
    double h[D], ps[D];
#pragma unroll
    for (int k = 0; k < D; ++k) h[k] = hi[k];
    const double ds = project_point<D>(h, v1, e, ee, ps);
    if (ds <= t_col) atomicCAS(rec, 0, static_cast<int32_t>(EZ_SEGMENT_IN_COLLISION));  // inflation.py:307-310
#pragma unroll
    for (int k = 0; k < D; ++k) {
        star[static_cast<int64_t>(i) * D + k] = h[k];
        pstar[static_cast<int64_t>(i) * D + k] = ps[k];
    }
    dstar[i] = ds;
}

}  // namespace ez
