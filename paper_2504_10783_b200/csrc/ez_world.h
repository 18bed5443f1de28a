// ez_world.h — host-side state of one device-resident world (robot + obstacles
// for one checker margin), shared by the check, FK and EI-ZO translation units.
#pragma once

#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "ez_common.h"
#include "ez_jit.h"

struct ez_eizo_ws;  // EI-ZO device workspace (ez_eizo.cu)

struct ez_world {
    int32_t device = 0;
    int32_t num_sms = 148;
    int32_t smem_optin = 232448;  // max dynamic shared memory per CTA
    int32_t dim = 3, dof = 0, n_joints = 0, n_spheres = 0, n_pairs = 0, n_blocks = 0;
    int32_t n_ssph = 0, n_sbox = 0, n_store = 0, n_hot = 0;
    int64_t n_voxels = 0;
    double margin = 0.0;

    // per-link Q_j^T (fp64, row-major) to turn modified frames back into link frames
    double* d_linkQt = nullptr;

    // model blobs and views, [0] = fp32, [1] = fp64
    uint8_t* d_blob[2] = {nullptr, nullptr};
    ez::ModelDev<float> mf{};
    ez::ModelDev<double> md{};

    // voxel obstacle structure (shared by both precisions)
    uint32_t* d_cells = nullptr;
    int4* d_lists = nullptr;
    uint32_t* d_occ_bits = nullptr;  // dense occupancy bitmap of the padded voxel lattice
    int64_t n_list = 0;
    int32_t grid_n[3] = {0, 0, 0};
    double cell_h = 0.0;
    int64_t device_bytes = 0;

    // host-buffer check pipeline
    std::mutex mu;
    // kHostLanes lanes (a host thread and a stream each) with two stages per
    // lane: pinned/device row and flag buffers plus a reuse event per stage
    static constexpr int kHostLanes = 16;
    static constexpr int kHostStages = 2 * kHostLanes;
    cudaStream_t hstream[kHostLanes] = {};
    cudaEvent_t stage_done[kHostStages] = {};
    void* h_stage_in[kHostStages] = {};
    uint8_t* h_stage_out[kHostStages] = {};
    void* d_stage_in[kHostStages] = {};
    uint8_t* d_stage_out[kHostStages] = {};
    // capacities in rows (buffers grow on demand; all idle between calls)
    int64_t h_in_rows[kHostStages] = {}, h_out_rows[kHostStages] = {}, d_rows[kHostStages] = {};

    ez_eizo_ws* eizo = nullptr;

    // run-time specialised fp32 check kernel (ez_jit.cu) and the host copy of
    // the fp32 model blob it is generated from
    std::vector<uint8_t> h_blob_f;
    std::vector<double> q_lo, q_hi;  // joint box (the specialised kernel's CTA size is tuned on it)
    // published (std::atomic_store) only after tuning; launches take a
    // std::atomic_load snapshot, so concurrent checks never race its writer
    std::shared_ptr<const ez::JitCheck> jit;
    bool jit_failed = false;
    std::string jit_error;
    int32_t jit_bt = 512;            // CTA size for large batches
    int32_t jit_variant = -1;        // voxel-code variant in use (ez_jit.cu Gen::variant)
    int32_t jit_occ[2][ez::kJitSizeCount] = {};  // [rows f32/f64][CTA size 64..1024] resident CTAs per SM

    // cached launch shapes of k_check, [T fp64][Q fp64]; set once under cfg_mu
    // (EI-ZO calls of several threads may race to the first launch)
    std::mutex cfg_mu;
    int32_t launch_threads[4] = {0, 0, 0, 0};
    size_t launch_smem[4] = {0, 0, 0, 0};
    int32_t launch_occ[4] = {0, 0, 0, 0};
};

namespace ez {

// launch the fused check over n rows; q_dtype EZ_F32/EZ_F64, precision EZ_F32/EZ_F64.
// If n_col != nullptr, atomically adds the number of colliding rows with index < count_lim.
int32_t launch_check(ez_world* w, const void* d_q, int32_t q_dtype, int64_t n, int64_t ld,
                     uint8_t* d_free, int32_t precision, cudaStream_t stream,
                     int64_t count_lim = 0, int32_t* n_col = nullptr);

void eizo_ws_free(ez_eizo_ws* ws);

// CTA size (max_threads, halved down to 32) whose per-thread sphere-centre
// store fits in shared memory; writes the dynamic smem bytes.  0 if even 32
// threads do not fit.
template <typename T>
inline int check_block_threads(const ez_world* w, uint32_t blob_bytes, int cen_words, int row_bytes, size_t* smem,
                               int max_threads = 128) {
    for (int t = max_threads; t >= 32; t /= 2) {
        size_t b = blob_bytes + static_cast<size_t>(cen_words) * t * sizeof(T);
        b = (b + 15) & ~static_cast<size_t>(15);
        b += static_cast<size_t>(t) * row_bytes;
        b = (b + 15) & ~static_cast<size_t>(15);
        if (b + 64 <= static_cast<size_t>(w->smem_optin)) {
            *smem = b;
            return t;
        }
    }
    return 0;
}

}  // namespace ez
