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

}  // namespace ez
