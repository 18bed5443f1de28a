// ez_device.cuh — device building blocks of the fused FK + collision check.
//
// Reference semantics (corridor/world.py):
//   fk_batch            195-223   per-joint T_child = T_parent * Origin * Motion(q)
//   _check_chunk        505-517   OR over robot-vs-obstacle tests and self pairs
//   _sphere_vs_obstacles 519-536  static spheres, voxel spheres (nearest centre), static boxes
//   _pair               554-557   sphere-sphere self pairs
// Touching counts as collision everywhere (<=), the margin enters every
// radius sum.  T = float (default; parity outside a 1e-5 contact band) or
// double (the reference's FP64 arithmetic).
#pragma once

#include "ez_common.h"

namespace ez {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// One elected thread moves `bytes` (multiple of 16, 16-B aligned) from global
// to shared memory with the TMA bulk-copy engine (cp.async.bulk + mbarrier
// transaction count); every thread of the CTA waits on the barrier.
__device__ __forceinline__ void tma_stage(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                     ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
    }
    __syncthreads();
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done) : "r"(smem_u32(bar)) : "memory");
    }
}

// ---------------------------------------------------------------------------
// scalar helpers
// ---------------------------------------------------------------------------
template <typename T> __device__ __forceinline__ T tsqrt(T x);
template <> __device__ __forceinline__ float tsqrt<float>(float x) { return sqrtf(x); }
template <> __device__ __forceinline__ double tsqrt<double>(double x) { return sqrt(x); }

// fp32 sin and cos of a joint value: a two-constant reduction by 2 pi into
// [-pi, pi] and the SFU's sin / cos (MUFU.SIN / MUFU.COS, absolute error
// about 2^-21.4 there).  Near contact this moves the fp32 decisions by at most
// 2.8e-7 in fp64 clearance (tools/diag_fp32_contact.py, 27k boundary points
// per model; 1.3e-7 with the 1.5-ulp minimax polynomials used before, at
// about 4x the instructions), far inside the 1e-5 contact band of the fp32
// contract (tests/test_gpu_check.py::test_fp32_disagreements_hug_contact).
// Config 2: 87.8 -> 81.1 us per 2^20.  Beyond |x| = 128 rad the library
// routine takes over.
__device__ __forceinline__ void sincos_f32(float x, float& s, float& c) {
    if (!(fabsf(x) <= 128.0f)) {
        sincosf(x, &s, &c);
        return;
    }
    const float k = rintf(x * 0.159154943091895336f);
    float r = fmaf(k, -6.28318548202514648f, x);  // 2 pi rounded to fp32
    r = fmaf(k, 1.74845553e-7f, r);                 // minus its rounding error
    s = __sinf(r);
    c = __cosf(r);
}

// sin/cos of a joint value.  fp32 arithmetic on an fp64 input keeps the
// residual q - float(q) as a first-order correction, so rounding the sample
// to fp32 costs no accuracy.
template <typename T, typename Q> struct Angle;
template <> struct Angle<float, float> {
    __device__ static __forceinline__ void sc(float q, float& s, float& c) { sincos_f32(q, s, c); }
};
template <> struct Angle<float, double> {
    __device__ static __forceinline__ void sc(double q, float& s, float& c) {
        const float hi = static_cast<float>(q);
        const float lo = static_cast<float>(q - static_cast<double>(hi));
        float s0, c0;
        sincos_f32(hi, s0, c0);
        s = fmaf(c0, lo, s0);
        c = fmaf(-s0, lo, c0);
    }
};
template <> struct Angle<double, double> {
    __device__ static __forceinline__ void sc(double q, double& s, double& c) { sincos(q, &s, &c); }
};
template <> struct Angle<double, float> {
    __device__ static __forceinline__ void sc(float q, double& s, double& c) {
        sincos(static_cast<double>(q), &s, &c);
    }
};

// voxel centre origin + (idx + 0.5) * side, rounded exactly like the
// reference's numpy expression (world.py:311-312) in fp64 mode.
__device__ __forceinline__ float lattice_centre(float org, int idx, float side) {
    return fmaf(static_cast<float>(idx) + 0.5f, side, org);
}
__device__ __forceinline__ double lattice_centre(double org, int idx, double side) {
    return __dadd_rn(org, __dmul_rn(static_cast<double>(idx) + 0.5, side));
}

// ---------------------------------------------------------------------------
// forward kinematics: all sphere centres of one configuration
// ---------------------------------------------------------------------------
// q: the configuration (dof values, any stride 1 memory), cen: sphere centre
// store, element (s, k) at cen[(3 s + k) * stride].
// Boxes: the world rotation (9) and translation (3) of box b are stored at
// words box_base + 12 b + k of the same store.
template <typename T, typename Q>
__device__ __forceinline__ void fk_sphere_centres(const JointRec<T>* __restrict__ J, int nj,
                                                  const SphereRec<T>* __restrict__ S,
                                                  const Q* __restrict__ q, T* __restrict__ cen,
                                                  int stride, const BoxRec<T>* __restrict__ BX = nullptr,
                                                  int box_base = 0) {
    T R[9] = {T(1), T(0), T(0), T(0), T(1), T(0), T(0), T(0), T(1)};
    T t[3] = {T(0), T(0), T(0)};
    T store[kMaxStore][12];
    for (int j = 0; j < nj; ++j) {
        const JointRec<T>& jr = J[j];
        if (jr.parent != j - 1) {
            if (jr.parent < 0) {
#pragma unroll
                for (int k = 0; k < 9; ++k) R[k] = (k % 4 == 0) ? T(1) : T(0);
                t[0] = t[1] = t[2] = T(0);
            } else {
#pragma unroll
                for (int k = 0; k < 9; ++k) R[k] = store[jr.parent_slot][k];
#pragma unroll
                for (int k = 0; k < 3; ++k) t[k] = store[jr.parent_slot][9 + k];
            }
        }
        T N[9], tn[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
#pragma unroll
            for (int c = 0; c < 3; ++c)
                N[3 * r + c] = R[3 * r] * jr.R[c] + R[3 * r + 1] * jr.R[3 + c] + R[3 * r + 2] * jr.R[6 + c];
            tn[r] = t[r] + (R[3 * r] * jr.t[0] + R[3 * r + 1] * jr.t[1] + R[3 * r + 2] * jr.t[2]);
        }
        if (jr.kind == EZ_JOINT_REVOLUTE) {
            T s, c;
            Angle<T, Q>::sc(q[jr.qidx], s, c);
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                const T n0 = N[3 * r], n1 = N[3 * r + 1];
                N[3 * r] = n0 * c + n1 * s;
                N[3 * r + 1] = n1 * c - n0 * s;
            }
        } else if (jr.kind == EZ_JOINT_PRISMATIC) {
            const T qq = static_cast<T>(q[jr.qidx]);
#pragma unroll
            for (int r = 0; r < 3; ++r)
                tn[r] += (N[3 * r] * jr.ax[0] + N[3 * r + 1] * jr.ax[1] + N[3 * r + 2] * jr.ax[2]) * qq;
        }
#pragma unroll
        for (int k = 0; k < 9; ++k) R[k] = N[k];
#pragma unroll
        for (int k = 0; k < 3; ++k) t[k] = tn[k];
        if (jr.store_slot >= 0) {
#pragma unroll
            for (int k = 0; k < 9; ++k) store[jr.store_slot][k] = R[k];
#pragma unroll
            for (int k = 0; k < 3; ++k) store[jr.store_slot][9 + k] = t[k];
        }
        for (int s = jr.sph_begin; s < jr.sph_end; ++s) {
            const SphereRec<T>& sp = S[s];
#pragma unroll
            for (int r = 0; r < 3; ++r)
                cen[(3 * s + r) * stride] =
                    t[r] + (R[3 * r] * sp.p[0] + R[3 * r + 1] * sp.p[1] + R[3 * r + 2] * sp.p[2]);
        }
        for (int bx = jr.box_begin; bx < jr.box_end; ++bx) {
            const BoxRec<T>& br = BX[bx];
            T* o = cen + (box_base + 12 * bx) * stride;
#pragma unroll
            for (int r = 0; r < 3; ++r) {
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    o[(3 * r + c) * stride] = R[3 * r] * br.R[c] + R[3 * r + 1] * br.R[3 + c] + R[3 * r + 2] * br.R[6 + c];
                o[(9 + r) * stride] = t[r] + (R[3 * r] * br.t[0] + R[3 * r + 1] * br.t[1] + R[3 * r + 2] * br.t[2]);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// boxes (world.py:394-427, 538-565)
// ---------------------------------------------------------------------------
// squared distance from p to the box (rotation R row-major, centre t, half extents he)
template <typename T>
__device__ __forceinline__ T point_box_d2(const T (&R)[9], const T (&t)[3], const T* he, T px, T py, T pz) {
    const T dx = px - t[0], dy = py - t[1], dz = pz - t[2];
    T d2 = T(0);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const T l = R[i] * dx + R[3 + i] * dy + R[6 + i] * dz;  // (R^T (p - t))_i
        const T cl = fmin(fmax(l, -he[i]), he[i]);
        d2 += (l - cl) * (l - cl);
    }
    return d2;
}

// separating-axis test, touching = colliding (world.py:401-427); axes with
// norm <= 1e-12 give no separation evidence.  Ra/Rb row-major, columns = box axes.
template <typename T>
__device__ __forceinline__ bool boxes_collide(const T (&Ra)[9], const T (&ta)[3], const T* hea, const T (&Rb)[9],
                                              const T (&tb)[3], const T* heb, T margin) {
    const T diff[3] = {tb[0] - ta[0], tb[1] - ta[1], tb[2] - ta[2]};
    auto separated = [&](T ux, T uy, T uz) -> bool {
        const T n = tsqrt<T>(ux * ux + uy * uy + uz * uz);
        if (!(n > T(1e-12))) return false;
        ux /= n;
        uy /= n;
        uz /= n;
        const T dist = fabs(ux * diff[0] + uy * diff[1] + uz * diff[2]);
        T ra = T(0), rb = T(0);
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            ra += fabs(ux * Ra[j] + uy * Ra[3 + j] + uz * Ra[6 + j]) * hea[j];
            rb += fabs(ux * Rb[j] + uy * Rb[3 + j] + uz * Rb[6 + j]) * heb[j];
        }
        return dist > ra + rb + margin;
    };
#pragma unroll
    for (int i = 0; i < 3; ++i)
        if (separated(Ra[i], Ra[3 + i], Ra[6 + i])) return false;
#pragma unroll
    for (int i = 0; i < 3; ++i)
        if (separated(Rb[i], Rb[3 + i], Rb[6 + i])) return false;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const T ax = Ra[3 + i] * Rb[6 + j] - Ra[6 + i] * Rb[3 + j];
            const T ay = Ra[6 + i] * Rb[j] - Ra[i] * Rb[6 + j];
            const T az = Ra[i] * Rb[3 + j] - Ra[3 + i] * Rb[j];
            if (separated(ax, ay, az)) return false;
        }
    }
    return true;
}

template <typename T>
__device__ __forceinline__ void load_box(const T* __restrict__ cen, int stride, int word, T (&R)[9], T (&t)[3]) {
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = cen[(word + k) * stride];
#pragma unroll
    for (int k = 0; k < 3; ++k) t[k] = cen[(word + 9 + k) * stride];
}

// Robot box vs static spheres, voxel spheres (occupied lattice cells inside
// the box's dilated bounding box, exact point-box test) and static boxes.
template <typename T>
__device__ __forceinline__ bool box_hits_obstacles(const ModelDev<T>& M, const uint8_t* blob, const T (&R)[9],
                                                   const T (&t)[3], const T* he, T margin) {
    const StaticSphereRec<T>* SS = reinterpret_cast<const StaticSphereRec<T>*>(blob + M.off_ssph);
    for (int i = 0; i < M.n_ssph; ++i) {
        const StaticSphereRec<T> o = SS[i];
        const T rr = o.r + margin;
        if (point_box_d2<T>(R, t, he, o.c[0], o.c[1], o.c[2]) <= rr * rr) return true;
    }
    const StaticBoxRec<T>* SB = reinterpret_cast<const StaticBoxRec<T>*>(blob + M.off_sbox);
    for (int i = 0; i < M.n_sbox; ++i) {
        const StaticBoxRec<T>& b = SB[i];
        T Rb[9], tb[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
#pragma unroll
            for (int c = 0; c < 3; ++c) Rb[3 * r + c] = b.Rt[3 * c + r];
            tb[r] = b.t[r];
        }
        if (boxes_collide<T>(R, t, he, Rb, tb, b.he, margin)) return true;
    }
    const VoxGrid<T>& V = M.vox;
    if (!V.present) return false;
    const T Rr = V.rvox + margin;  // r_vox + margin (world.py:542-547)
    const T R2 = Rr * Rr;
    int lo[3], hi[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const T ext = fabs(R[3 * k]) * he[0] + fabs(R[3 * k + 1]) * he[1] + fabs(R[3 * k + 2]) * he[2] + Rr;
        const T a = (t[k] - ext - V.vorg[k]) / V.vside - T(0.5);
        const T b = (t[k] + ext - V.vorg[k]) / V.vside - T(0.5);
        lo[k] = max(V.lbase[k], static_cast<int>(floor(a)) - 1);
        hi[k] = min(V.lbase[k] + V.L[k] - 1, static_cast<int>(floor(b)) + 1);
    }
    // rows of the x-range, 32 lattice cells per bitmap word: empty words (most
    // of a sparse cloud) are skipped whole, set bits visited by ffs
    if (lo[0] > hi[0]) return false;
    for (int z = lo[2]; z <= hi[2]; ++z)
        for (int y = lo[1]; y <= hi[1]; ++y) {
            const int64_t row = (static_cast<int64_t>(z - V.lbase[2]) * V.L[1] + (y - V.lbase[1])) * V.L[0] - V.lbase[0];
            const int64_t b0 = row + lo[0], b1 = row + hi[0];
            for (int64_t wi = b0 >> 5; wi <= (b1 >> 5); ++wi) {
                uint32_t word = __ldg(V.occ + wi);
                if (wi == (b0 >> 5)) word &= ~0u << (b0 & 31);
                if (wi == (b1 >> 5)) word &= ~0u >> (31 - (b1 & 31));
                while (word) {
                    const int bpos = __ffs(word) - 1;
                    word &= word - 1;
                    const int x = static_cast<int>((wi << 5) + bpos - row);
                    if (point_box_d2<T>(R, t, he, lattice_centre(V.vorg[0], x, V.vside),
                                        lattice_centre(V.vorg[1], y, V.vside), lattice_centre(V.vorg[2], z, V.vside)) <= R2)
                        return true;
                }
            }
        }
    return false;
}

// all box tests of one configuration: boxes vs obstacles, then mixed self pairs
template <typename T>
__device__ __forceinline__ bool boxes_collide_all(const ModelDev<T>& M, const uint8_t* blob,
                                                  const T* __restrict__ cen, int stride, T margin) {
    const BoxRec<T>* BX = reinterpret_cast<const BoxRec<T>*>(blob + M.off_boxes);
    const int base = M.box_base;
    for (int b = 0; b < M.n_boxes; ++b) {
        T R[9], t[3];
        load_box<T>(cen, stride, base + 12 * b, R, t);
        if (box_hits_obstacles<T>(M, blob, R, t, BX[b].he, margin)) return true;
    }
    const MixPairRec<T>* MP = reinterpret_cast<const MixPairRec<T>*>(blob + M.off_mix);
    for (int p = 0; p < M.n_mix; ++p) {
        const MixPairRec<T> mp = MP[p];
        T Rb[9], tb[3];
        load_box<T>(cen, stride, base + 12 * mp.b_slot, Rb, tb);
        if (mp.a_kind == 0) {
            const T rr = mp.ra + margin;
            if (point_box_d2<T>(Rb, tb, BX[mp.b_slot].he, cen[(3 * mp.a_slot) * stride], cen[(3 * mp.a_slot + 1) * stride],
                                cen[(3 * mp.a_slot + 2) * stride]) <= rr * rr)
                return true;
        } else {
            T Ra[9], ta[3];
            load_box<T>(cen, stride, base + 12 * mp.a_slot, Ra, ta);
            if (boxes_collide<T>(Ra, ta, BX[mp.a_slot].he, Rb, tb, BX[mp.b_slot].he, margin)) return true;
        }
    }
    return false;
}

// ---------------------------------------------------------------------------
// self pairs (world.py:514-516, 554-557)
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ bool pair_hits(const HotRec<T>& h, const T* __restrict__ cen, int stride) {
    const T dx = cen[(3 * h.a) * stride] - cen[(3 * h.b) * stride];
    const T dy = cen[(3 * h.a + 1) * stride] - cen[(3 * h.b + 1) * stride];
    const T dz = cen[(3 * h.a + 2) * stride] - cen[(3 * h.b + 2) * stride];
    return dx * dx + dy * dy + dz * dz <= h.thr2;
}

// Non-hot self pairs, block by link pair: the bounding-sphere test skips
// whole blocks (see BlockRec); inside a block four independent pair tests run
// per branch so their loads and math overlap.
template <typename T>
__device__ __forceinline__ bool blocks_collide(const ModelDev<T>& M, const uint8_t* blob,
                                               const T* __restrict__ cen, int stride) {
    const BlockRec<T>* B = reinterpret_cast<const BlockRec<T>*>(blob + M.off_blocks);
    const HotRec<T>* P = reinterpret_cast<const HotRec<T>*>(blob + M.off_rest);
    for (int k = 0; k < M.n_blocks; ++k) {
        const BlockRec<T> bk = B[k];
        const T bx = cen[(3 * bk.ba) * stride] - cen[(3 * bk.bb) * stride];
        const T by = cen[(3 * bk.ba + 1) * stride] - cen[(3 * bk.bb + 1) * stride];
        const T bz = cen[(3 * bk.ba + 2) * stride] - cen[(3 * bk.bb + 2) * stride];
        if (bx * bx + by * by + bz * bz > bk.thr2) continue;
        int p = bk.begin;
        for (; p + 4 <= bk.end; p += 4) {
            bool hit = false;
#pragma unroll
            for (int u = 0; u < 4; ++u) hit |= pair_hits<T>(P[p + u], cen, stride);
            if (hit) return true;
        }
        for (; p < bk.end; ++p)
            if (pair_hits<T>(P[p], cen, stride)) return true;
    }
    return false;
}

// ---------------------------------------------------------------------------
// voxel spheres: "nearest voxel centre within r + r_vox + margin"
// (world.py:529-532), answered exactly through the quantised distance grid
// ---------------------------------------------------------------------------
// sqrt(x) or an upper bound of it: every use of the point-to-cell-centre
// distance e below stays exact with any e' >= e (the tests only get more
// conservative), so fp32 takes x * rsqrt(x) raised by 2^-20 (> its error).
template <typename T> __device__ __forceinline__ T dist_ub(T x);
template <> __device__ __forceinline__ float dist_ub<float>(float x) {
    return x > 0.0f ? x * rsqrtf(x) * 1.00000095367431640625f : 0.0f;
}
template <> __device__ __forceinline__ double dist_ub<double>(double x) { return sqrt(x); }

// Cell of the distance grid holding p (-1 outside the grid: farther than the
// list radius from every voxel) and an upper bound e of the distance from p
// to the cell centre (dist_ub).
template <typename T>
__device__ __forceinline__ int64_t voxel_cell(const VoxGrid<T>& V, T px, T py, T pz, T& e) {
    const T fx = (px - V.org[0]) * V.inv_h;
    const T fy = (py - V.org[1]) * V.inv_h;
    const T fz = (pz - V.org[2]) * V.inv_h;
    e = T(0);
    if (!(fx >= T(0) && fy >= T(0) && fz >= T(0) && fx < T(V.n[0]) && fy < T(V.n[1]) && fz < T(V.n[2])))
        return -1;
    const int ix = static_cast<int>(fx), iy = static_cast<int>(fy), iz = static_cast<int>(fz);
    const T ex = px - (V.org[0] + (T(ix) + T(0.5)) * V.h);
    const T ey = py - (V.org[1] + (T(iy) + T(0.5)) * V.h);
    const T ez_ = pz - (V.org[2] + (T(iz) + T(0.5)) * V.h);
    e = dist_ub<T>(ex * ex + ey * ey + ez_ * ez_);
    return (static_cast<int64_t>(iz) * V.n[1] + iy) * V.n[0] + ix;
}

constexpr uint32_t kFarCell = 0xFF000000u;  // q = 255: no voxel within the list radius

// List walk for a cell the quantised distance does not decide (rare: the
// point is within one quantisation step of R).
#ifndef EZ_VOXEL_WALK_ATTR
#define EZ_VOXEL_WALK_ATTR __forceinline__
#endif
template <typename T>
__device__ EZ_VOXEL_WALK_ATTR bool voxel_walk(const VoxGrid<T>& V, uint32_t w, T e, T px, T py, T pz, T R) {
    const int4* __restrict__ L = V.lists + (w & 0x00FFFFFFu);
    const T lim = R + e + V.eps;
    const T R2 = R * R;
    for (;;) {
        const int4 E = __ldg(L);
        ++L;
        if (static_cast<T>(__int_as_float(E.w)) > lim) return false;
        const T dx = px - lattice_centre(V.vorg[0], E.x, V.vside);
        const T dy = py - lattice_centre(V.vorg[1], E.y, V.vside);
        const T dz = pz - lattice_centre(V.vorg[2], E.z, V.vside);
        if (dx * dx + dy * dy + dz * dz <= R2) return true;
    }
}

// Decide "some voxel centre within R of p" from the cell word w.
template <typename T>
__device__ __forceinline__ bool voxel_decide(const VoxGrid<T>& V, uint32_t w, T e, T px, T py, T pz, T R) {
    const uint32_t qc = w >> 24;
    const T lo = T(qc) * V.dq;
    if (lo - e > R + V.eps) return false;                          // certainly free
    if (qc < 255u && lo + V.dq + e <= R - V.eps) return true;      // certainly hit
    return voxel_walk<T>(V, w, e, px, py, pz, R);
}

template <typename T>
__device__ __forceinline__ bool voxel_hit(const VoxGrid<T>& V, T px, T py, T pz, T R) {
    T e;
    const int64_t c = voxel_cell<T>(V, px, py, pz, e);
    if (c < 0) return false;
    return voxel_decide<T>(V, __ldg(V.cells + c), e, px, py, pz, R);
}

template <typename T>
__device__ __forceinline__ bool static_hits(const ModelDev<T>& M, const SphereRec<T>& sp,
                                            const StaticSphereRec<T>* __restrict__ SS,
                                            const StaticBoxRec<T>* __restrict__ SB, T margin, T px, T py, T pz) {
    for (int i = 0; i < M.n_ssph; ++i) {
        const StaticSphereRec<T> o = SS[i];
        const T dx = px - o.c[0], dy = py - o.c[1], dz = pz - o.c[2];
        const T rr = (o.r + sp.r) + margin;
        if (dx * dx + dy * dy + dz * dz <= rr * rr) return true;
    }
    for (int i = 0; i < M.n_sbox; ++i) {
        const StaticBoxRec<T>& b = SB[i];
        const T dx = px - b.t[0], dy = py - b.t[1], dz = pz - b.t[2];
        T d2 = T(0);
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const T l = b.Rt[3 * r] * dx + b.Rt[3 * r + 1] * dy + b.Rt[3 * r + 2] * dz;
            const T cl = fmin(fmax(l, -b.he[r]), b.he[r]);
            d2 += (l - cl) * (l - cl);
        }
        if (d2 <= sp.rmar * sp.rmar) return true;
    }
    return false;
}

template <typename T>
__device__ __forceinline__ bool sphere_hits_obstacles(const ModelDev<T>& M,
                                                      const SphereRec<T>& sp,
                                                      const StaticSphereRec<T>* __restrict__ SS,
                                                      const StaticBoxRec<T>* __restrict__ SB,
                                                      T margin, T px, T py, T pz) {
    if (static_hits<T>(M, sp, SS, SB, margin, px, py, pz)) return true;
    return M.vox.present && voxel_hit<T>(M.vox, px, py, pz, sp.rvox);
}

// Phase A: the calibrated hot self pairs (flat list, most frequent first).
template <typename T>
__device__ __forceinline__ bool hot_pairs_collide(const ModelDev<T>& M, const uint8_t* blob,
                                                  const T* __restrict__ cen, int stride) {
    const HotRec<T>* H = reinterpret_cast<const HotRec<T>*>(blob + M.off_hot);
    for (int p = 0; p < M.n_hot; ++p) {
        const HotRec<T> h = H[p];
        const T dx = cen[(3 * h.a) * stride] - cen[(3 * h.b) * stride];
        const T dy = cen[(3 * h.a + 1) * stride] - cen[(3 * h.b + 1) * stride];
        const T dz = cen[(3 * h.a + 2) * stride] - cen[(3 * h.b + 2) * stride];
        if (dx * dx + dy * dy + dz * dz <= h.thr2) return true;
    }
    return false;
}

// Phase B: obstacles (spheres in calibrated hit-frequency order, distance-
// grid cells fetched kVoxBatch at a time so their L2 latencies overlap), then
// the remaining self pairs grouped by first sphere.
constexpr int kVoxBatch = 4;

template <typename T>
__device__ __forceinline__ bool rest_collides(const ModelDev<T>& M, const uint8_t* blob,
                                              const T* __restrict__ cen, int stride, T margin) {
    const SphereRec<T>* S = reinterpret_cast<const SphereRec<T>*>(blob + M.off_spheres);
    const int32_t* order = reinterpret_cast<const int32_t*>(blob + M.off_order);
    const StaticSphereRec<T>* SS = reinterpret_cast<const StaticSphereRec<T>*>(blob + M.off_ssph);
    const StaticBoxRec<T>* SB = reinterpret_cast<const StaticBoxRec<T>*>(blob + M.off_sbox);
    const bool vox = M.vox.present;
    for (int k0 = 0; k0 < M.n_spheres; k0 += kVoxBatch) {
        T px[kVoxBatch], py[kVoxBatch], pz[kVoxBatch], e[kVoxBatch];
        uint32_t w[kVoxBatch];
        int sid[kVoxBatch];
#pragma unroll
        for (int j = 0; j < kVoxBatch; ++j) {
            const int k = min(k0 + j, M.n_spheres - 1);
            const int s = order[k];
            sid[j] = s;
            px[j] = cen[(3 * s) * stride];
            py[j] = cen[(3 * s + 1) * stride];
            pz[j] = cen[(3 * s + 2) * stride];
            w[j] = kFarCell;
            e[j] = T(0);
            if (vox) {
                const int64_t c = voxel_cell<T>(M.vox, px[j], py[j], pz[j], e[j]);
                if (c >= 0) w[j] = __ldg(M.vox.cells + c);
            }
        }
#pragma unroll
        for (int j = 0; j < kVoxBatch; ++j) {
            if (k0 + j >= M.n_spheres) break;
            const SphereRec<T>& sp = S[sid[j]];
            if (static_hits<T>(M, sp, SS, SB, margin, px[j], py[j], pz[j])) return true;
            if (vox && w[j] != kFarCell && voxel_decide<T>(M.vox, w[j], e[j], px[j], py[j], pz[j], sp.rvox))
                return true;
        }
    }
    if (blocks_collide<T>(M, blob, cen, stride)) return true;
    return (M.n_boxes > 0) && boxes_collide_all<T>(M, blob, cen, stride, margin);
}

// Everything about one configuration whose sphere centres are in `cen`.
template <typename T>
__device__ __forceinline__ bool config_collides(const ModelDev<T>& M, const uint8_t* blob,
                                                const T* __restrict__ cen, int stride, T margin) {
    return hot_pairs_collide<T>(M, blob, cen, stride) || rest_collides<T>(M, blob, cen, stride, margin);
}

// Full check of one configuration q (dof values).  Returns true if free.
template <typename T, typename Q>
__device__ __forceinline__ bool config_free(const ModelDev<T>& M, const uint8_t* blob,
                                            const Q* q, T* cen, int stride, T margin) {
    const JointRec<T>* J = reinterpret_cast<const JointRec<T>*>(blob);
    const SphereRec<T>* S = reinterpret_cast<const SphereRec<T>*>(blob + M.off_spheres);
    fk_sphere_centres<T, Q>(J, M.n_joints, S, q, cen, stride, reinterpret_cast<const BoxRec<T>*>(blob + M.off_boxes),
                            M.box_base);
    return !config_collides<T>(M, blob, cen, stride, margin);
}

// ---------------------------------------------------------------------------
// cooperative check: G lanes of a warp evaluate one configuration.  Used on
// latency-bound paths (bisection rounds) where there are only ~1e4
// configurations in flight.  Every lane runs the (cheap, serial) joint chain;
// sphere centres, pair tests and obstacle tests are split across the lanes
// and joined with a group ballot.  All loop trip counts are group-uniform.
// Centres live in a per-configuration store cen[3 s + k].
// ---------------------------------------------------------------------------
template <int G>
__device__ __forceinline__ unsigned coop_mask() {
    if (G == 32) return 0xffffffffu;
    return ((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1));
}

template <typename T, typename Q, int G>
__device__ __forceinline__ void fk_centres_coop(const JointRec<T>* __restrict__ J, int nj,
                                                const SphereRec<T>* __restrict__ S, const Q* __restrict__ q,
                                                T* __restrict__ cen, int lane,
                                                const BoxRec<T>* __restrict__ BX = nullptr, int box_base = 0) {
    T R[9] = {T(1), T(0), T(0), T(0), T(1), T(0), T(0), T(0), T(1)};
    T t[3] = {T(0), T(0), T(0)};
    T store[kMaxStore][12];
    for (int j = 0; j < nj; ++j) {
        const JointRec<T>& jr = J[j];
        if (jr.parent != j - 1) {
            if (jr.parent < 0) {
#pragma unroll
                for (int k = 0; k < 9; ++k) R[k] = (k % 4 == 0) ? T(1) : T(0);
                t[0] = t[1] = t[2] = T(0);
            } else {
#pragma unroll
                for (int k = 0; k < 9; ++k) R[k] = store[jr.parent_slot][k];
#pragma unroll
                for (int k = 0; k < 3; ++k) t[k] = store[jr.parent_slot][9 + k];
            }
        }
        T N[9], tn[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
#pragma unroll
            for (int c = 0; c < 3; ++c)
                N[3 * r + c] = R[3 * r] * jr.R[c] + R[3 * r + 1] * jr.R[3 + c] + R[3 * r + 2] * jr.R[6 + c];
            tn[r] = t[r] + (R[3 * r] * jr.t[0] + R[3 * r + 1] * jr.t[1] + R[3 * r + 2] * jr.t[2]);
        }
        if (jr.kind == EZ_JOINT_REVOLUTE) {
            T sn, cs;
            Angle<T, Q>::sc(q[jr.qidx], sn, cs);
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                const T n0 = N[3 * r], n1 = N[3 * r + 1];
                N[3 * r] = n0 * cs + n1 * sn;
                N[3 * r + 1] = n1 * cs - n0 * sn;
            }
        } else if (jr.kind == EZ_JOINT_PRISMATIC) {
            const T qq = static_cast<T>(q[jr.qidx]);
#pragma unroll
            for (int r = 0; r < 3; ++r)
                tn[r] += (N[3 * r] * jr.ax[0] + N[3 * r + 1] * jr.ax[1] + N[3 * r + 2] * jr.ax[2]) * qq;
        }
#pragma unroll
        for (int k = 0; k < 9; ++k) R[k] = N[k];
#pragma unroll
        for (int k = 0; k < 3; ++k) t[k] = tn[k];
        if (jr.store_slot >= 0) {
#pragma unroll
            for (int k = 0; k < 9; ++k) store[jr.store_slot][k] = R[k];
#pragma unroll
            for (int k = 0; k < 3; ++k) store[jr.store_slot][9 + k] = t[k];
        }
        for (int s = jr.sph_begin + lane; s < jr.sph_end; s += G) {
            const SphereRec<T>& sp = S[s];
#pragma unroll
            for (int r = 0; r < 3; ++r)
                cen[3 * s + r] = t[r] + (R[3 * r] * sp.p[0] + R[3 * r + 1] * sp.p[1] + R[3 * r + 2] * sp.p[2]);
        }
        for (int bx = jr.box_begin + lane; bx < jr.box_end; bx += G) {
            const BoxRec<T>& br = BX[bx];
            T* o = cen + box_base + 12 * bx;
#pragma unroll
            for (int r = 0; r < 3; ++r) {
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    o[3 * r + c] = R[3 * r] * br.R[c] + R[3 * r + 1] * br.R[3 + c] + R[3 * r + 2] * br.R[6 + c];
                o[9 + r] = t[r] + (R[3 * r] * br.t[0] + R[3 * r + 1] * br.t[1] + R[3 * r + 2] * br.t[2]);
            }
        }
    }
}

template <typename T, typename Q, int G>
__device__ __forceinline__ bool config_free_coop(const ModelDev<T>& M, const uint8_t* blob, const Q* q,
                                                 T* __restrict__ cen, T margin) {
    const unsigned gm = coop_mask<G>();
    const int lane = threadIdx.x & (G - 1);
    const JointRec<T>* J = reinterpret_cast<const JointRec<T>*>(blob);
    const SphereRec<T>* S = reinterpret_cast<const SphereRec<T>*>(blob + M.off_spheres);
    const BoxRec<T>* BX = reinterpret_cast<const BoxRec<T>*>(blob + M.off_boxes);
    fk_centres_coop<T, Q, G>(J, M.n_joints, S, q, cen, lane, BX, M.box_base);
    __syncwarp(gm);
    const HotRec<T>* H = reinterpret_cast<const HotRec<T>*>(blob + M.off_hot);
    for (int p0 = 0; p0 < M.n_hot; p0 += G) {
        const int p = p0 + lane;
        bool hit = false;
        if (p < M.n_hot) {
            const HotRec<T> h = H[p];
            const T dx = cen[3 * h.a] - cen[3 * h.b], dy = cen[3 * h.a + 1] - cen[3 * h.b + 1],
                    dz = cen[3 * h.a + 2] - cen[3 * h.b + 2];
            hit = dx * dx + dy * dy + dz * dz <= h.thr2;
        }
        if (__ballot_sync(gm, hit)) return false;
    }
    const int32_t* order = reinterpret_cast<const int32_t*>(blob + M.off_order);
    const StaticSphereRec<T>* SS = reinterpret_cast<const StaticSphereRec<T>*>(blob + M.off_ssph);
    const StaticBoxRec<T>* SB = reinterpret_cast<const StaticBoxRec<T>*>(blob + M.off_sbox);
    // kVoxBatch spheres per lane per round: their distance-grid cells are
    // fetched together (independent L2 loads in flight), then decided
    const bool vox = M.vox.present;
    for (int k0 = 0; k0 < M.n_spheres; k0 += kVoxBatch * G) {
        T px[kVoxBatch], py[kVoxBatch], pz[kVoxBatch], e[kVoxBatch];
        uint32_t w[kVoxBatch];
        int sid[kVoxBatch];
#pragma unroll
        for (int j = 0; j < kVoxBatch; ++j) {
            const int k = k0 + j * G + lane;
            sid[j] = (k < M.n_spheres) ? order[k] : -1;
            w[j] = kFarCell;
            e[j] = T(0);
            if (sid[j] >= 0) {
                px[j] = cen[3 * sid[j]];
                py[j] = cen[3 * sid[j] + 1];
                pz[j] = cen[3 * sid[j] + 2];
                if (vox) {
                    const int64_t c = voxel_cell<T>(M.vox, px[j], py[j], pz[j], e[j]);
                    if (c >= 0) w[j] = __ldg(M.vox.cells + c);
                }
            }
        }
        bool hit = false;
#pragma unroll
        for (int j = 0; j < kVoxBatch; ++j) {
            if (sid[j] < 0 || hit) continue;
            const SphereRec<T>& sp = S[sid[j]];
            hit = static_hits<T>(M, sp, SS, SB, margin, px[j], py[j], pz[j]) ||
                  (w[j] != kFarCell && voxel_decide<T>(M.vox, w[j], e[j], px[j], py[j], pz[j], sp.rvox));
        }
        if (__ballot_sync(gm, hit)) return false;
    }
    const BlockRec<T>* Bk = reinterpret_cast<const BlockRec<T>*>(blob + M.off_blocks);
    const HotRec<T>* P = reinterpret_cast<const HotRec<T>*>(blob + M.off_rest);
    for (int k = 0; k < M.n_blocks; ++k) {
        const BlockRec<T> bk = Bk[k];
        const T bx = cen[3 * bk.ba] - cen[3 * bk.bb], by = cen[3 * bk.ba + 1] - cen[3 * bk.bb + 1],
                bz = cen[3 * bk.ba + 2] - cen[3 * bk.bb + 2];
        if (bx * bx + by * by + bz * bz > bk.thr2) continue;  // group-uniform
        for (int p0 = bk.begin; p0 < bk.end; p0 += G) {
            const int p = p0 + lane;
            const bool hit = p < bk.end && pair_hits<T>(P[p], cen, 1);
            if (__ballot_sync(gm, hit)) return false;
        }
    }
    if (M.n_boxes == 0) return true;
    const int base = M.box_base;
    for (int b0 = 0; b0 < M.n_boxes; b0 += G) {
        const int b = b0 + lane;
        bool hit = false;
        if (b < M.n_boxes) {
            T Rb[9], tb[3];
            load_box<T>(cen, 1, base + 12 * b, Rb, tb);
            hit = box_hits_obstacles<T>(M, blob, Rb, tb, BX[b].he, margin);
        }
        if (__ballot_sync(gm, hit)) return false;
    }
    const MixPairRec<T>* MP = reinterpret_cast<const MixPairRec<T>*>(blob + M.off_mix);
    for (int p0 = 0; p0 < M.n_mix; p0 += G) {
        const int p = p0 + lane;
        bool hit = false;
        if (p < M.n_mix) {
            const MixPairRec<T> mp = MP[p];
            T Rb[9], tb[3];
            load_box<T>(cen, 1, base + 12 * mp.b_slot, Rb, tb);
            if (mp.a_kind == 0) {
                const T rr = mp.ra + margin;
                hit = point_box_d2<T>(Rb, tb, BX[mp.b_slot].he, cen[3 * mp.a_slot], cen[3 * mp.a_slot + 1],
                                      cen[3 * mp.a_slot + 2]) <= rr * rr;
            } else {
                T Ra[9], ta[3];
                load_box<T>(cen, 1, base + 12 * mp.a_slot, Ra, ta);
                hit = boxes_collide<T>(Ra, ta, BX[mp.a_slot].he, Rb, tb, BX[mp.b_slot].he, margin);
            }
        }
        if (__ballot_sync(gm, hit)) return false;
    }
    return true;
}

}  // namespace ez
