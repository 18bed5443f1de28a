// ez_common.h — host+device shared definitions for the corridor_b200 library.
#pragma once

#ifdef __CUDACC_RTC__
// run-time compiled kernels (ez_jit.cu): no host headers
typedef signed char int8_t;
typedef unsigned char uint8_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
#else
#include <cstdint>
#include <cstdio>
#include <functional>
#include <string>

#include <cuda_runtime.h>
#endif

#include "../../include/corridor_b200.h"

namespace ez {

// ---------------------------------------------------------------------------
// error plumbing: thread-local last error + status propagation
// ---------------------------------------------------------------------------
#ifndef __CUDACC_RTC__
void set_error(const std::string& msg);
int32_t fail(int32_t status, const std::string& msg);
int32_t cuda_fail(cudaError_t err, const char* what, const char* file, int line);
int32_t retain_async_pool();  // keep the current device's default mem pool cached
// fn(lo, hi) over [0, n) split across a persistent host thread pool (parts of
// at least min_per_part items); returns when every part is done
void host_parallel(int64_t n, int64_t min_per_part, const std::function<void(int64_t, int64_t)>& fn);
// n bytes into (write-combined) pinned staging memory with streaming stores
void copy_to_staging(void* dst, const void* src, size_t n);
#endif

#define EZ_CUDA(call)                                                        \
    do {                                                                     \
        cudaError_t _e = (call);                                             \
        if (_e != cudaSuccess) return ::ez::cuda_fail(_e, #call, __FILE__, __LINE__); \
    } while (0)

#define EZ_TRY(call)                                                         \
    do {                                                                     \
        int32_t _s = (call);                                                 \
        if (_s != EZ_OK) return _s;                                          \
    } while (0)

#ifndef __CUDACC_RTC__
// Every C entry point runs on its object's device and leaves the caller's
// current device as it found it.
struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int device) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != device) err = cudaSetDevice(device);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};
#define EZ_ON_DEVICE(dev)                                                    \
    ::ez::DeviceGuard _ez_dg(dev);                                           \
    EZ_CUDA(_ez_dg.err)

// Allow a kernel the current device's whole opt-in dynamic shared memory.
// Launch sizes differ by call (faces, candidates, models, grids) and calls run
// on several host threads: setting the attribute to each launch's own size
// let another thread lower it between that set and this launch.  The maximum
// is the same for every caller, so concurrent sets agree.
template <typename K>
inline int32_t allow_max_dyn_smem(K kern) {
    int dev = 0, optin = 0;
    EZ_CUDA(cudaGetDevice(&dev));
    EZ_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa{};
    EZ_CUDA(cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(kern)));
    EZ_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(kern), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 optin - static_cast<int>(fa.sharedSizeBytes)));
    return EZ_OK;
}
#endif

// ---------------------------------------------------------------------------
// device-side model records.  All kinematics are embedded in 3-D; a planar
// model is the z = 0 slice (revolute about z, boxes with zero z half-extent).
//
// Frames are "modified" frames G_j = (Rg_j, t_j) with the true link frame
// F_j = (Rg_j * Q_j^T, t_j), where Q_j maps e_z onto joint j's revolute axis.
// Every child constant is pre-rotated by Q^T on the host, so a revolute
// motion is always a right-multiplication by Rz(q) (world.py:64-69 Rodrigues
// rewritten as P Rz(q) P^T).
// ---------------------------------------------------------------------------
constexpr int kMaxJoints = 64;
constexpr int kMaxSpheres = 1024;
constexpr int kMaxStore = 8;   // links whose frame is reused by a non-consecutive child

template <typename T>
struct alignas(16) JointRec {
    T R[9];     // Q_parent^T * R_origin * P_j
    T t[3];     // Q_parent^T * t_origin
    T ax[3];    // prismatic axis (joint frame), zeros otherwise
    int32_t kind;        // EZ_JOINT_*
    int32_t parent;      // parent link, -1 = world
    int32_t qidx;        // configuration column, -1 for fixed
    int32_t store_slot;  // >= 0: save this link's frame for a later child
    int32_t parent_slot; // >= 0: parent frame comes from this slot
    int32_t sph_begin, sph_end;  // spheres attached to this link
    int32_t box_begin, box_end;  // boxes attached to this link
    int32_t pad_[3];
};

// Self pairs outside the hot list are tested in blocks, one per pair of
// links: each link is bounded by a ball around one of its spheres (the
// anchor) enclosing all the link's spheres; if the anchors are farther apart
// than R_a + R_b + margin, no pair of the block can touch and the block is
// skipped.  thr2 carries a small upward
// slack, so the skip is conservative in fp32.
template <typename T>
struct alignas(16) BlockRec {
    int32_t ba, bb;       // anchor sphere indices
    int32_t begin, end;   // range in the rest-pair list (HotRec layout)
    T thr2;               // (R_a + R_b + margin)^2 (+ slack)
    T pad_[3];
};

// Robot box geometry (world.py:538-565).  World pose = link frame * local.
template <typename T>
struct alignas(16) BoxRec {
    T R[9];     // Q_link^T * local rotation
    T t[3];     // Q_link^T * local translation
    T he[3];    // half extents (planar boxes: z = 0)
    T pad_;
};

// Self pair with at least one box: a sphere-box (point-box distance against
// r + margin) or box-box (separating axes with margin) test.  kind 0 = sphere
// (slot = sphere index), 1 = box (slot = box index); a is the sphere if any.
template <typename T>
struct alignas(16) MixPairRec {
    int32_t a_kind, a_slot, b_kind, b_slot;
    T ra;       // sphere radius of a (sphere-box)
    T pad_[3];
};

template <typename T>
struct alignas(16) SphereRec {
    T p[3];     // Q_link^T * local translation
    T r;        // radius
    T rvox;     // (r + r_vox) + margin  (world.py:532)
    T rmar;     // r + margin            (world.py:535)
    T pad_[2];
};

// The self pairs most likely to collide (calibrated on uniform samples at
// world creation) are tested first, flat, so most colliding configurations
// leave after one or two pairs; the rest are tested in link-pair blocks.
template <typename T>
struct alignas(16) HotRec {
    int32_t a, b;
    T thr2;
    T pad_;
};

template <typename T>
struct alignas(16) StaticSphereRec {  // world.py:449-451, 522-528
    T c[3];
    T r;
};

template <typename T>
struct alignas(16) StaticBoxRec {     // world.py:394-398, 533-535
    T Rt[9];    // transposed world rotation
    T t[3];
    T he[3];
    T pad_;
};

// Voxel-sphere obstacle structure: a uint32 word per cell of a grid of side
// h = voxel_side / sub aligned with the voxel lattice.  Bits 31..24 hold a
// floor-quantised nearest-voxel-centre distance q (d(g) in [q dq, (q+1) dq),
// 255 = farther than the list radius); bits 23..0 the offset of the cell's
// candidate list (voxel lattice indices sorted by distance to the cell
// centre, terminated by a +inf sentinel).
template <typename T>
struct VoxGrid {
    const uint32_t* cells;
    const int4* lists;
    int32_t n[3];
    int32_t present;
    T org[3];       // corner of cell (0,0,0)
    T h, inv_h;
    T dq;           // quantisation step
    T eps;          // rounding guard of the filter (precision dependent)
    T vorg[3];      // voxel lattice origin
    T vside;
    T rvox;         // voxel sphere radius 0.5 * side * sqrt(dim)
    // dense occupancy bitmap of the padded voxel lattice (robot boxes scan it)
    const uint32_t* occ;
    int32_t lbase[3];  // lattice index of bit 0 along each axis
    int32_t L[3];      // lattice extent of the bitmap
};

template <typename T>
struct ModelDev {
    const uint8_t* blob;      // device: joints | spheres | hot | blocks | rest | order | ssph | sbox | boxes | mix
    uint32_t blob_bytes;      // multiple of 16
    int32_t n_joints, dof, n_spheres, n_hot, n_blocks, n_rest, n_ssph, n_sbox, n_store, n_boxes, n_mix;
    int32_t cen_words;        // per-configuration store: 3 per sphere + 12 per box
    int32_t box_base;         // first word of the box frames: 3 * n_spheres
    uint32_t off_spheres, off_hot, off_blocks, off_rest, off_order, off_ssph, off_sbox, off_boxes, off_mix;
    VoxGrid<T> vox;
};

}  // namespace ez
