/*
 * corridor_b200.h — C ABI of the B200-native EI-ZO hot path.
 *
 * One shared library (paper_2504_10783_b200/_lib/libcorridor_b200.so) exports
 * the entry points below.  Signatures use plain pointers, sizes and enums
 * only (no torch types).  Every call returns an ez_status; nothing is thrown
 * across the ABI.  ez_last_error() returns a thread-local message for the
 * last non-OK status.
 *
 * Each entry point replaces one interface of the reference Python package
 * (`corridor`, /root/reference/pkg/src/corridor).  The reference binds no
 * native code; the ctypes binding a maintainer would add is shown in
 * INTEGRATION.md and implemented in paper_2504_10783_b200/_native.py.
 *
 * Pointer conventions: arguments named d_* are CUDA device pointers (the
 * Python shim passes torch.Tensor.data_ptr()); h_* are host pointers;
 * plain structs are read on the host during the call.  `stream` is a
 * cudaStream_t (NULL = legacy default stream).
 */
#ifndef CORRIDOR_B200_H
#define CORRIDOR_B200_H

#ifndef __CUDACC_RTC__
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define EZ_ABI_VERSION 3

/* ---- status codes: mapped 1:1 onto corridor.errors (errors.py:4-64) ---- */
typedef enum ez_status {
    EZ_OK = 0,
    EZ_DIMENSION_MISMATCH = 1,   /* DimensionMismatch                       */
    EZ_EMPTY_CHORD = 2,          /* EmptyChord       (cpoly.py:167-168)      */
    EZ_SEED_OUTSIDE = 3,         /* SeedOutside      (cpoly.py:158-159)      */
    EZ_GRADIENT_UNDEFINED = 4,   /* GradientUndefined (inflation.py:423-424) */
    EZ_SEGMENT_IN_COLLISION = 5, /* SegmentInCollision (inflation.py:303-310)*/
    EZ_SEED_OUTSIDE_DOMAIN = 6,  /* SeedOutsideDomain (inflation.py:276-277) */
    EZ_GRID_MISMATCH = 7,        /* GridMismatch     (drm.py:269-270)        */
    EZ_INVALID_ARGUMENT = 8,     /* ValueError                               */
    EZ_CUDA_ERROR = 9,           /* CUDA runtime/driver failure              */
    EZ_UNSUPPORTED = 10,         /* model feature not implemented natively   */
    EZ_CAPACITY = 11             /* a device capacity limit was exceeded     */
} ez_status;

enum { EZ_JOINT_FIXED = 0, EZ_JOINT_REVOLUTE = 1, EZ_JOINT_PRISMATIC = 2 };
enum { EZ_GEOM_SPHERE = 0, EZ_GEOM_BOX = 1 };
enum { EZ_F32 = 0, EZ_F64 = 1 };          /* element type / arithmetic precision */
enum { EZ_RNG_COUNTER = 0, EZ_RNG_PHILOX = 1 };

typedef struct ez_world ez_world;          /* opaque, device-resident */
typedef struct ez_roadmap ez_roadmap;      /* opaque, device-resident */
typedef struct ez_eizo_session ez_eizo_session;  /* opaque: one rank's share of a sharded EI-ZO */

/* Robot description (host arrays, read during ez_world_create).
 * Mirrors world.RobotModel (world.py:122-167): joints in chain order with
 * joint j's child link j, geometries in link-major global order. */
typedef struct ez_robot_desc {
    int32_t dim;                  /* task-space dimension: 2 or 3            */
    int32_t n_joints;             /* == number of links                      */
    const int32_t* joint_kind;    /* [n_joints] EZ_JOINT_*                   */
    const int32_t* joint_parent;  /* [n_joints] parent link, -1 = world      */
    const double* joint_rot;      /* [n_joints][dim][dim] origin rotation    */
    const double* joint_trans;    /* [n_joints][dim]      origin translation */
    const double* joint_axis;     /* [n_joints][dim] axis (zeros if unused)  */
    int32_t n_geoms;
    const int32_t* geom_link;     /* [n_geoms] owning link                   */
    const int32_t* geom_kind;     /* [n_geoms] EZ_GEOM_*                     */
    const double* geom_rot;       /* [n_geoms][dim][dim] local rotation      */
    const double* geom_trans;     /* [n_geoms][dim]      local translation   */
    const double* geom_radius;    /* [n_geoms] sphere radius                 */
    const double* geom_half;      /* [n_geoms][dim] box half extents         */
    int32_t n_pairs;
    const int32_t* pairs;         /* [n_pairs][2] global geometry indices    */
    const double* joint_lower;    /* [dof] joint limits (optional: used to   */
    const double* joint_upper;    /* order the tests by hit frequency)       */
} ez_robot_desc;

/* Obstacles: static geometry posed in the world plus one voxel map
 * (world.py:369-391, 441-463).  Voxel i is the sphere of radius
 * 0.5*side*sqrt(dim) centred at origin + (idx_i + 0.5)*side. */
typedef struct ez_scene_desc {
    int32_t n_static;
    const int32_t* static_kind;   /* [n_static] EZ_GEOM_*                    */
    const double* static_rot;     /* [n_static][dim][dim]                    */
    const double* static_trans;   /* [n_static][dim]                         */
    const double* static_radius;  /* [n_static]                              */
    const double* static_half;    /* [n_static][dim]                         */
    int64_t n_voxels;             /* 0 = no voxel map                        */
    const int32_t* h_voxel_idx;   /* [n_voxels][dim] occupied lattice cells  */
    const double* voxel_origin;   /* [dim]                                   */
    double voxel_side;
} ez_scene_desc;

/* Summary of the device obstacle structure (for tests and benchmarks). */
typedef struct ez_world_info {
    int32_t dof, n_links, n_spheres, n_pairs, n_static, n_hot_pairs;
    int64_t n_voxels;
    int32_t grid_dims[3];         /* cells of the voxel distance grid        */
    double cell_side;             /* h = voxel side / subdivision            */
    int64_t list_entries;         /* candidate-list entries (incl. sentinels)*/
    int64_t device_bytes;         /* bytes held on the device                */
    int32_t check_cta;            /* CTA size of the specialised check kernel */
                                  /* for large batches, 0 = generic kernel   */
    int32_t check_variant;        /* voxel-code variant of the specialised   */
                                  /* kernel (0 literal grid, 1 generic), -1  */
} ez_world_info;

/* EI-ZO parameters: inflation.InflationParams (inflation.py:55-95). */
typedef struct ez_eizo_params {
    double delta, eps, tau, delta_max, t_col;
    int32_t n_p, n_f, n_b, n_ms;  /* n_b resolved by the caller (>= 1)      */
    int32_t n_it;                 /* 0 = unlimited                           */
} ez_eizo_params;

/* inflation.InflationReport (inflation.py:99-108) + timing. */
typedef struct ez_eizo_report {
    int32_t iterations;
    int32_t hyperplanes_added;
    int64_t collision_checks;
    int32_t terminated_by;        /* 0 = test_accepted, 1 = max_iterations   */
    int32_t n_faces;              /* rows written to A_out/b_out             */
    double device_ms;             /* GPU time of the whole inflation         */
} ez_eizo_report;

#ifndef __CUDACC_RTC__ /* the run-time compiled kernels need the types only */
/* ---------------- library ---------------- */
int32_t ez_abi_version(void);
const char* ez_last_error(void);
int32_t ez_device_count(void);
/* FP32 FMA throughput of `device` (TFLOP/s), the roofline denominator of the
 * FP32-bound checker; measured with a dependent-chain-free FMA kernel. */
int32_t ez_fp32_peak(int32_t device, double* tflops, double* ms);
/* FP64 tensor-core (DMMA m8n8k4) throughput of `device` (TFLOP/s), the
 * roofline denominator of the hit-and-run walk (FP64 chord GEMMs). */
int32_t ez_fp64_tc_peak(int32_t device, double* tflops, double* ms);

/* ---------------- world / collision checker ----------------
 * ez_world_create  replaces CollisionChecker.__init__   (world.py:441-463)
 * ez_check_batch   replaces CollisionChecker.check_batch (world.py:483-495)
 * ez_fk_batch      replaces fk_batch                     (world.py:195-223)
 */
int32_t ez_world_create(const ez_robot_desc* robot, const ez_scene_desc* scene,
                        double margin, int32_t device, ez_world** out);
int32_t ez_world_destroy(ez_world* world);
int32_t ez_world_get_info(const ez_world* world, ez_world_info* out);

/* Model-specialised fp32 check kernel (no reference counterpart: the
 * reference's _check_chunk, world.py:505-517, interprets the model per call).
 * mode 1: generate CUDA for this world's robot model (literal constants,
 * straight-line FK and pair tests), compile it with NVRTC for sm_100a and use
 * it for fp32 batches; mode 0: query only; mode -1: go back to the generic
 * kernel for good.  Returns EZ_OK if the specialised kernel is in use,
 * EZ_UNSUPPORTED if it is not (robot boxes, NVRTC missing, disabled).
 * Never compiled implicitly by a check call; the kernel is published
 * atomically after its CTA size is tuned, so concurrent checks on the world
 * see either the generic or the finished specialised kernel. */
int32_t ez_world_specialize(ez_world* world, int32_t mode);

/* Free mask (1 = collision-free) for n configurations.  d_q points at n rows
 * of `dof` values of type q_dtype with row stride ld (elements).  precision
 * selects the arithmetic (EZ_F32: parity outside a 1e-5 contact band;
 * EZ_F64: the reference's FP64 arithmetic). */
int32_t ez_check_batch(ez_world* world, const void* d_q, int32_t q_dtype, int64_t n,
                       int64_t ld, uint8_t* d_free, int32_t precision, void* stream);
/* Same, from host memory (rows of type q_dtype, pinned or pageable):
 * pipelined H2D / kernel / D2H over an internal pinned ring, synchronous on
 * return.  This is what a ctypes binding of the numpy-facing check_batch
 * calls; fp32 rows cross PCIe at 4 B per value. */
int32_t ez_check_batch_host(ez_world* world, const void* h_q, int32_t q_dtype, int64_t n, int64_t ld,
                            uint8_t* h_free, int32_t precision);
/* Link frames: d_frames[n][n_links][12] = row-major R (9) then t (3),
 * embedded in 3-D for planar models. */
int32_t ez_fk_batch(ez_world* world, const double* d_q, int64_t n, double* d_frames,
                    void* stream);

/* ---------------- hit-and-run (cpoly.py:127-173) ----------------
 * count walks of n_ms steps inside {x | A x <= b}; walk i starts at
 * d_seeds[i % n_seeds] and uses stream (seed, walk_offset + i). */
int32_t ez_hit_and_run(const double* d_A, const double* d_b, int32_t n_faces, int32_t dim,
                       const double* d_seeds, int64_t n_seeds, int64_t count, int32_t n_ms,
                       uint64_t seed, uint64_t walk_offset, int32_t rng, double* d_out,
                       void* stream);

/* ---------------- EI-ZO (inflation.py:262-325) ----------------
 * Host inputs: segment endpoints h_v1/h_v2 [dim], domain h_A0 [n_faces0][dim],
 * h_b0 [n_faces0].  Writes the result polytope to h_A_out/h_b_out (capacity
 * face_cap rows) and the report.  Samples never leave the device. */
int32_t ez_inflate_edge(ez_world* world, const double* h_v1, const double* h_v2, int32_t dim,
                        const double* h_A0, const double* h_b0, int32_t n_faces0,
                        const ez_eizo_params* params, uint64_t seed, int32_t precision,
                        int32_t rng, ez_eizo_report* report, double* h_A_out, double* h_b_out,
                        int32_t face_cap);

/* If the polytope has more than face_cap rows, ez_inflate_edge fills the
 * report (n_faces included), keeps the rows for the calling thread and returns
 * EZ_CAPACITY; ez_inflate_edge_result copies them out (count, then copy). */
int32_t ez_inflate_edge_result(double* h_A_out, double* h_b_out, int32_t face_cap, int32_t* n_faces);

/* In-segment batch sharding: EI-ZO as resumable steps.  Each
 * rank runs a session over the same segment/domain/seed; per iteration k the
 * caller (torch.distributed over NCCL) all-reduces the first-m collision
 * counts returned by _sample, all-gathers the candidate counts, bisects its
 * share of the global first n_p (_bisect, rows copied to caller device
 * buffers), all-gathers (star, pstar, dstar) and places the same faces on every rank
 * (_place).  Samples are keyed by global walk index, so the result equals
 * ez_inflate_edge for any number of ranks. */
int32_t ez_eizo_session_begin(ez_world* world, const double* h_v1, const double* h_v2, int32_t dim,
                              const double* h_A0, const double* h_b0, int32_t n_faces0,
                              const ez_eizo_params* params, uint64_t seed, int32_t precision, int32_t rng,
                              ez_eizo_session** out);
int32_t ez_eizo_session_end(ez_eizo_session* session);
int32_t ez_eizo_session_sample(ez_eizo_session* session, int32_t k, uint64_t walk_begin, int64_t count,
                               int64_t m_local, int32_t* n_col_m, int32_t* n_cand);
/* Optional hint: make the draws of iteration k's walks [walk_begin, +count)
 * ahead on the session's side stream (overlapping the current iteration). */
int32_t ez_eizo_session_prefetch(ez_eizo_session* session, int32_t k, uint64_t walk_begin, int64_t count);
int32_t ez_eizo_session_bisect(ez_eizo_session* session, int32_t k, int32_t n_take, double* d_star,
                               double* d_pstar, double* d_dstar);
int32_t ez_eizo_session_place(ez_eizo_session* session, int32_t k, const double* d_star, const double* d_pstar,
                              const double* d_dstar, int32_t n_total, int32_t* placed, int32_t* n_faces);
int32_t ez_eizo_session_result(ez_eizo_session* session, double* h_A_out, double* h_b_out, int32_t face_cap,
                               int32_t* n_faces);

/* Set repair, the device part of refine_sets (planner.py:159-224): project
 * n_cols host collisions onto the seed segment, fail-fast check, N_b
 * bisection rounds, then uncapped step-back faces discarding candidates whose
 * ORIGINAL collision leaves the set (planner.py:191-192).  Appends faces to
 * (h_A, h_b) and writes the result to h_A_out/h_b_out (capacity face_cap). */
int32_t ez_refine_set(ez_world* world, const double* h_v1, const double* h_v2, int32_t dim,
                      const double* h_A, const double* h_b, int32_t n_faces, const double* h_cols,
                      int32_t n_cols, double delta_max, double t_col, int32_t n_b, int32_t precision,
                      double* h_A_out, double* h_b_out, int32_t face_cap, int32_t* n_faces_out,
                      int64_t* collision_checks);

/* ---------------- DRM online phase ----------------
 * ez_voxelize        replaces voxelize_point_cloud (world.py:315-328): unique
 *                    occupied bins floor((p - origin)/side), lexicographically
 *                    sorted, written to d_idx_out[*n_out][dim] (capacity = n).
 * ez_roadmap_create  uploads the CSR voxel->node map (drm.py:108-131).
 * ez_collision_set   replaces collision_set (drm.py:262-296): d_blocked_bits
 *                    receives the node bitmap (ceil(n_nodes/32) words),
 *                    *n_blocked its popcount (synchronises); with
 *                    n_blocked = NULL the call stays asynchronous on stream. */
int32_t ez_voxelize(const double* d_points, int64_t n, int32_t dim, const double* h_origin,
                    double side, int32_t* d_idx_out, int64_t* n_out, void* stream);
int32_t ez_roadmap_create(const int64_t* h_cmap_offsets, const int32_t* h_cmap_ids,
                          int64_t n_voxels, int64_t n_nodes, int32_t dim,
                          const double* h_origin, double side, const int32_t* h_extents,
                          int32_t device, ez_roadmap** out);
int32_t ez_roadmap_destroy(ez_roadmap* roadmap);
/* Offline collision map on the GPU (replaces drm.py:170-204 _node_voxel_pairs
 * + the CSR assembly of build_drm, drm.py:250-251): voxel v lists every node
 * whose robot spheres touch v's circumscribing sphere, (r + r_vox)^2 test in
 * fp64, node ids ascending.  d_nodes: [n_nodes][dof] fp64 device rows. */
int32_t ez_roadmap_build(ez_world* world, const double* d_nodes, int64_t n_nodes, int32_t dim,
                         const double* h_origin, double side, const int32_t* h_extents, void* stream,
                         ez_roadmap** out);
/* Roadmap adjacency on the GPU (replaces build_drm's edge construction,
 * drm.py:219-248): for each node its nearest min(n, 4k+1) nodes in fp64
 * configuration distance (cKDTree order), the first skipped, stop at the
 * first distance > d_cs, skip end-effector distance > d_ts (d_ee:
 * [n_nodes][ee_dim] end-effector positions), keep at most k; symmetrised and
 * returned as CSR in d_adj_offsets[n_nodes + 1] (int64) and d_adj_ids
 * (int32, capacity 2 * k * n_nodes, ids ascending per row), *nnz entries.
 * Synchronises on `stream`. */
int32_t ez_roadmap_adjacency(const double* d_nodes, int64_t n_nodes, int32_t dof, const double* d_ee,
                             int32_t ee_dim, int32_t k, double d_cs, double d_ts, int64_t* d_adj_offsets,
                             int32_t* d_adj_ids, int64_t* nnz, void* stream);
int32_t ez_roadmap_info(const ez_roadmap* roadmap, int64_t* n_voxels, int64_t* n_nodes, int64_t* nnz);
int32_t ez_roadmap_export(const ez_roadmap* roadmap, int64_t* h_offsets, int32_t* h_ids);
int32_t ez_collision_set(ez_roadmap* roadmap, const int32_t* d_vox_idx, int64_t n_vox,
                         const double* h_vmap_origin, double vmap_side, int32_t same_grid,
                         uint32_t* d_blocked_bits, int64_t* n_blocked, void* stream);
/* Same, plus the blocked node ids in ascending order in d_ids (capacity
 * n_nodes) and their count in *n_ids (synchronises).  What the Python
 * collision_set returns, without unpacking the bitmap on the host. */
int32_t ez_collision_set_ids(ez_roadmap* roadmap, const int32_t* d_vox_idx, int64_t n_vox,
                             const double* h_vmap_origin, double vmap_side, int32_t same_grid,
                             uint32_t* d_blocked_bits, int32_t* d_ids, int64_t* n_ids, void* stream);
#endif /* __CUDACC_RTC__ */

#ifdef __cplusplus
}
#endif
#endif /* CORRIDOR_B200_H */
