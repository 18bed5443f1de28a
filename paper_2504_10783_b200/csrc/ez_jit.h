// ez_jit.h — run-time specialised check kernels (ez_jit.cu).
#pragma once

#include <string>

#include "ez_common.h"

struct ez_world;

namespace ez {

// CTA sizes the specialised kernels launch at (ez_world::jit_occ columns)
constexpr int kJitSizeCount = 5;  // 64, 128, 256, 512, 1024

// The check kernels for one robot model (and margin), one library each:
// k[rows f32/f64][0: 64..256 threads, 1: 512 threads, 2: 1024 threads].  Kept
// for the life of the process.
struct JitCheck {
    cudaLibrary_t lib[2][3] = {};
    cudaKernel_t k[2][3] = {};
    // the EI-ZO bisection on the same model code (ez_bisect_core.cuh)
    cudaLibrary_t blib = nullptr;
    cudaKernel_t bk = nullptr;
    int b_occ = 0;  // its resident CTAs per SM
    ~JitCheck();
};

// Generate, compile (NVRTC, sm_100a) and load the world's specialised check
// kernels, then pick the CTA size for large batches by timing 256, 512 and
// 1024 threads on random configurations; EZ_UNSUPPORTED if the model has robot
// boxes or NVRTC is missing.
int32_t jit_specialize(ez_world* w);  // published with std::atomic_store
// CUDA source of the specialised kernel (for inspection and tests)
std::string jit_source(const ez_world* w, int variant = 0);
// Launch it over n rows (fp32 arithmetic); jc is the caller's snapshot of ez_world::jit.
int32_t jit_launch(ez_world* w, const JitCheck& jc, const void* d_q, bool q64, int64_t n, int64_t ld,
                   uint8_t* d_free, cudaStream_t stream, int64_t count_lim, int32_t* n_col);

// The EI-ZO bisection of the first *n_cand (<= n_p) candidates on the
// specialised check (ez_bisect_core.cuh; same arguments as ez_eizo.cu's
// k_bisect2, rec = status / stop words, d = the world's dof).
int32_t jit_bisect_launch(ez_world* w, const JitCheck& jc, const double* X, const int32_t* col, int32_t* rec,
                          const int32_t* n_cand, int n_p, const double* seg, double ee, int n_b, double t_col,
                          double* star, double* pstar, double* dstar, cudaStream_t stream);

}  // namespace ez
