// ez_roadmap.h — device-resident DRM collision map (CSR voxel -> node ids).
#pragma once

#include <mutex>

#include "ez_common.h"

struct ez_roadmap {
    int32_t device = 0;
    int32_t dim = 3;
    int64_t n_voxels = 0, n_nodes = 0, nnz = 0;
    double origin[3] = {0, 0, 0};
    double side = 0.0;
    int32_t ext[3] = {1, 1, 1};
    int64_t* d_off = nullptr;        // [n_voxels + 1]
    int32_t* d_ids = nullptr;        // [nnz], node ids sorted per voxel
    uint32_t* d_vox_bits = nullptr;  // scratch: active roadmap voxels
    unsigned long long* d_count = nullptr;
    unsigned long long* h_count = nullptr;
    // The scratch above is shared by every prune on this roadmap.  A prune
    // holds `mu` while it enqueues, waits on `scratch_free` (recorded by the
    // previous prune on its stream after its last scratch use) and records it
    // again, so asynchronous prunes on different streams use it in turn.
    std::mutex mu;
    cudaEvent_t scratch_free = nullptr;
};
