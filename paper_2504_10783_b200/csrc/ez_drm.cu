// ez_drm.cu — DRM online phase: point-cloud voxelisation and the voxel->node
// collision-set prune.  Replaces
//   voxelize_point_cloud  corridor/world.py:315-328   (ez_voxelize)
//   Drm CSR collision map corridor/drm.py:108-131     (ez_roadmap_create)
//   collision_set         corridor/drm.py:262-296     (ez_collision_set)
// Both kernels are HBM/latency bound integer work: occupancy and blocked-node
// sets are bitmaps, the CSR gather is one warp per active voxel.
#include <algorithm>
#include <climits>
#include <cmath>

#include <cub/device/device_scan.cuh>

#include "ez_common.h"

#include "ez_roadmap.h"

namespace ez {

struct VoxParams {
    double org[3];
    double inv_side_unused;
    double side;
    int32_t dim;
};

// bounding box of the indices: warp-reduced first, one atomic pair per warp
// and axis (a per-point atomic on six addresses serialised 1e5 updates)
__global__ void k_vox_index(const double* __restrict__ pts, int64_t n, VoxParams vp, int32_t* __restrict__ idx,
                            int32_t* __restrict__ bbox, int32_t* __restrict__ overflow) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool in = i < n;
    for (int k = 0; k < vp.dim; ++k) {
        int32_t v = 0;
        bool ok = in;
        if (in) {
            // floor((p - origin) / side), fp64 as numpy (world.py:327)
            const double f = floor((pts[i * vp.dim + k] - vp.org[k]) / vp.side);
            if (!(f >= -2147483648.0 && f <= 2147483647.0)) {
                atomicExch(overflow, 1);
                ok = false;
            } else {
                v = static_cast<int32_t>(f);
                idx[i * vp.dim + k] = v;
            }
        }
        const int32_t mn = __reduce_min_sync(0xffffffffu, ok ? v : INT_MAX);
        const int32_t mx = __reduce_max_sync(0xffffffffu, ok ? v : INT_MIN);
        if ((threadIdx.x & 31) == 0) {
            if (mn != INT_MAX) atomicMin(bbox + 2 * k, mn);
            if (mx != INT_MIN) atomicMax(bbox + 2 * k + 1, mx);
        }
    }
}

struct BoxDims {
    int32_t lo[3];
    int64_t n[3];
};

__device__ __forceinline__ int64_t lex_index(const int32_t* v, int dim, const BoxDims& bd) {
    int64_t r = 0;
    for (int k = 0; k < dim; ++k) r = r * bd.n[k] + (v[k] - bd.lo[k]);
    return r;
}

// occupancy bits; lanes hitting the same word (clustered clouds) merge their
// bits first, one atomic per distinct word per warp
__global__ void k_vox_mark(const int32_t* __restrict__ idx, int64_t n, int dim, BoxDims bd, uint32_t* __restrict__ bits) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool in = i < n;
    const int64_t li = in ? lex_index(idx + i * dim, dim, bd) : 0;
    const unsigned long long word = in ? static_cast<unsigned long long>(li >> 5) : ~0ull;
    const unsigned grp = __match_any_sync(0xffffffffu, word);
    const unsigned orv = __reduce_or_sync(grp, in ? (1u << (li & 31)) : 0u);
    if (in && static_cast<int>(threadIdx.x & 31) == __ffs(grp) - 1) atomicOr(bits + word, orv);
}

__global__ void k_popc(const uint32_t* __restrict__ bits, int64_t nw, uint32_t* __restrict__ cnt) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < nw) cnt[i] = __popc(bits[i]);
}

// emit occupied cells in lexicographic order (== sorted(tuple) order)
__global__ void k_vox_emit(const uint32_t* __restrict__ bits, const uint32_t* __restrict__ offs, int64_t nw, int dim,
                           BoxDims bd, int32_t* __restrict__ out) {
    const int64_t wi = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (wi >= nw) return;
    uint32_t w = bits[wi];
    uint32_t o = offs[wi];
    while (w) {
        const int bpos = __ffs(w) - 1;
        w &= w - 1;
        int64_t li = (wi << 5) + bpos;
        int32_t v[3];
        for (int k = dim - 1; k >= 0; --k) {
            v[k] = static_cast<int32_t>(li % bd.n[k]) + bd.lo[k];
            li /= bd.n[k];
        }
        for (int k = 0; k < dim; ++k) out[static_cast<int64_t>(o) * dim + k] = v[k];
        ++o;
    }
}

// ---- collision_set ----
struct PruneParams {
    double vorg[3], vside;   // voxel map
    double gorg[3], gside;   // roadmap grid
    int32_t ext[3];
    int32_t dim;
    int32_t same;
};

// activate roadmap voxels: identical grid -> the index itself, otherwise every
// roadmap voxel the occupied cube overlaps (+-1e-12 floor guards, drm.py:277-288)
__global__ void k_activate(const int32_t* __restrict__ vidx, int64_t n, PruneParams pp, uint32_t* __restrict__ vbits) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int k = 0; k < pp.dim; ++k) {
        const int32_t c = vidx[i * pp.dim + k];
        if (pp.same) {
            lo[k] = hi[k] = c;
        } else {
            const double clo = __dadd_rn(__dmul_rn(static_cast<double>(c), pp.vside), pp.vorg[k]);
            const double chi = __dadd_rn(clo, pp.vside);
            const double fl = floor(__dadd_rn((clo - pp.gorg[k]) / pp.gside, 1e-12));
            const double fh = floor(__dsub_rn((chi - pp.gorg[k]) / pp.gside, 1e-12));
            lo[k] = static_cast<int>(fmax(fl, -1.0));
            hi[k] = static_cast<int>(fmin(fh, static_cast<double>(pp.ext[k])));
        }
    }
    for (int z = lo[2]; z <= hi[2]; ++z) {
        if (pp.dim == 3 && (z < 0 || z >= pp.ext[2])) continue;
        for (int y = lo[1]; y <= hi[1]; ++y) {
            if (y < 0 || y >= pp.ext[1]) continue;
            for (int x = lo[0]; x <= hi[0]; ++x) {
                if (x < 0 || x >= pp.ext[0]) continue;
                // Grid.ids_of: row-major with x fastest (drm.py:59-64)
                const int64_t vid = (pp.dim == 3 ? (static_cast<int64_t>(z) * pp.ext[1] + y) * pp.ext[0]
                                                 : static_cast<int64_t>(y) * pp.ext[0]) + x;
                atomicOr(vbits + (vid >> 5), 1u << (vid & 31));
            }
        }
    }
}

// one warp per roadmap voxel: OR its node list into the blocked bitmap
__global__ void k_gather(const uint32_t* __restrict__ vbits, int64_t n_vox, const int64_t* __restrict__ off,
                         const int32_t* __restrict__ ids, uint32_t* __restrict__ nbits) {
    const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t v = warp; v < n_vox; v += nwarps) {
        if (!((vbits[v >> 5] >> (v & 31)) & 1u)) continue;
        const int64_t b = off[v], e = off[v + 1];
        for (int64_t j = b + lane; j < e; j += 32) {
            const int32_t node = __ldg(ids + j);
            atomicOr(nbits + (node >> 5), 1u << (node & 31));
        }
    }
}

__global__ void k_count_bits(const uint32_t* __restrict__ bits, int64_t nw, unsigned long long* __restrict__ out) {
    unsigned long long c = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nw;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        c += __popc(bits[i]);
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// Blocked-node ids, ascending, from the node bitmap: one CTA walks the words in
// chunks of 1024, a block-wide exclusive scan of the popcounts places each
// word's ids (the host no longer unpacks 1e5 bits).  ids[n_out] = count.
__global__ void __launch_bounds__(1024) k_bits_to_ids(const uint32_t* __restrict__ bits, int64_t nw,
                                                      int32_t* __restrict__ ids, int64_t* __restrict__ n_out) {
    __shared__ int s_warp[32];
    __shared__ int64_t s_base;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    for (int64_t w0 = 0; w0 < nw; w0 += 1024) {
        const int64_t wi = w0 + threadIdx.x;
        const uint32_t w = wi < nw ? bits[wi] : 0u;
        const int c = __popc(w);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_warp[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            const int v = s_warp[lane];
            int wincl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, wincl, o);
                if (lane >= o) wincl += y;
            }
            s_warp[lane] = wincl - v;  // exclusive prefix of the warps
        }
        __syncthreads();
        int64_t pos = s_base + s_warp[wid] + (incl - c);
        uint32_t m = w;
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            ids[pos++] = static_cast<int32_t>((wi << 5) + b);
        }
        __syncthreads();
        if (threadIdx.x == 1023) s_base = pos;  // the last thread ends the chunk
        __syncthreads();
    }
    if (threadIdx.x == 0) *n_out = s_base;
}

}  // namespace ez

using namespace ez;

extern "C" int32_t ez_voxelize(const double* d_points, int64_t n, int32_t dim, const double* h_origin, double side,
                               int32_t* d_idx_out, int64_t* n_out, void* stream) {
    if (!n_out) return fail(EZ_INVALID_ARGUMENT, "null n_out");
    *n_out = 0;
    if (!(side > 0.0)) return fail(EZ_INVALID_ARGUMENT, "bin side must be positive");
    if (dim < 1 || dim > 3) return fail(EZ_INVALID_ARGUMENT, "dimension must be 1..3");
    if (n == 0) return EZ_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    VoxParams vp{};
    for (int k = 0; k < dim; ++k) vp.org[k] = h_origin[k];
    vp.side = side;
    vp.dim = dim;
    int32_t* d_tmp = nullptr;   // bbox[6] + overflow
    int32_t* d_idx = nullptr;
    EZ_TRY(retain_async_pool());
    EZ_CUDA(cudaMallocAsync(&d_tmp, sizeof(int32_t) * 8, s));
    EZ_CUDA(cudaMallocAsync(&d_idx, sizeof(int32_t) * n * dim, s));
    int32_t init[8] = {INT_MAX, INT_MIN, INT_MAX, INT_MIN, INT_MAX, INT_MIN, 0, 0};
    EZ_CUDA(cudaMemcpyAsync(d_tmp, init, sizeof(init), cudaMemcpyHostToDevice, s));
    k_vox_index<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(d_points, n, vp, d_idx, d_tmp, d_tmp + 6);
    EZ_CUDA(cudaGetLastError());
    int32_t hb[8];
    EZ_CUDA(cudaMemcpyAsync(hb, d_tmp, sizeof(hb), cudaMemcpyDeviceToHost, s));
    EZ_CUDA(cudaStreamSynchronize(s));
    if (hb[6]) {
        cudaFreeAsync(d_tmp, s);
        cudaFreeAsync(d_idx, s);
        return fail(EZ_INVALID_ARGUMENT, "point cloud index outside the int32 range");
    }
    BoxDims bd{};
    int64_t vol = 1;
    for (int k = 0; k < 3; ++k) {
        bd.lo[k] = k < dim ? hb[2 * k] : 0;
        bd.n[k] = k < dim ? static_cast<int64_t>(hb[2 * k + 1]) - hb[2 * k] + 1 : 1;
        vol *= bd.n[k];
        if (vol > (int64_t(1) << 34)) break;
    }
    if (vol > (int64_t(1) << 34)) {
        cudaFreeAsync(d_tmp, s);
        cudaFreeAsync(d_idx, s);
        return fail(EZ_CAPACITY, "point cloud extent too large for the occupancy bitmap");
    }
    const int64_t nw = (vol + 31) / 32;
    uint32_t *d_bits = nullptr, *d_cnt = nullptr, *d_off = nullptr;
    void* d_scan = nullptr;
    size_t scan_bytes = 0;
    EZ_CUDA(cudaMallocAsync(&d_bits, sizeof(uint32_t) * nw, s));
    EZ_CUDA(cudaMallocAsync(&d_cnt, sizeof(uint32_t) * nw, s));
    EZ_CUDA(cudaMallocAsync(&d_off, sizeof(uint32_t) * nw, s));
    EZ_CUDA(cudaMemsetAsync(d_bits, 0, sizeof(uint32_t) * nw, s));
    k_vox_mark<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(d_idx, n, dim, bd, d_bits);
    k_popc<<<static_cast<unsigned>((nw + 255) / 256), 256, 0, s>>>(d_bits, nw, d_cnt);
    EZ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, d_cnt, d_off, static_cast<int>(nw), s));
    EZ_CUDA(cudaMallocAsync(&d_scan, scan_bytes, s));
    EZ_CUDA(cub::DeviceScan::ExclusiveSum(d_scan, scan_bytes, d_cnt, d_off, static_cast<int>(nw), s));
    k_vox_emit<<<static_cast<unsigned>((nw + 255) / 256), 256, 0, s>>>(d_bits, d_off, nw, dim, bd, d_idx_out);
    EZ_CUDA(cudaGetLastError());
    uint32_t last[2];
    EZ_CUDA(cudaMemcpyAsync(&last[0], d_off + nw - 1, 4, cudaMemcpyDeviceToHost, s));
    EZ_CUDA(cudaMemcpyAsync(&last[1], d_cnt + nw - 1, 4, cudaMemcpyDeviceToHost, s));
    EZ_CUDA(cudaStreamSynchronize(s));
    *n_out = static_cast<int64_t>(last[0]) + last[1];
    cudaFreeAsync(d_tmp, s);
    cudaFreeAsync(d_idx, s);
    cudaFreeAsync(d_bits, s);
    cudaFreeAsync(d_cnt, s);
    cudaFreeAsync(d_off, s);
    cudaFreeAsync(d_scan, s);
    return EZ_OK;
}

extern "C" int32_t ez_roadmap_create(const int64_t* h_off, const int32_t* h_ids, int64_t n_voxels, int64_t n_nodes,
                                     int32_t dim, const double* h_origin, double side, const int32_t* h_extents,
                                     int32_t device, ez_roadmap** out) {
    if (!out || !h_off || !h_extents || !h_origin) return fail(EZ_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    if (dim < 2 || dim > 3) return fail(EZ_INVALID_ARGUMENT, "grid dimension must be 2 or 3");
    int64_t prod = 1;
    for (int k = 0; k < dim; ++k) prod *= h_extents[k];
    if (prod != n_voxels) return fail(EZ_INVALID_ARGUMENT, "grid extents disagree with the voxel count");
    EZ_ON_DEVICE(device);
    ez_roadmap* r = new ez_roadmap();
    r->device = device;
    r->dim = dim;
    r->n_voxels = n_voxels;
    r->n_nodes = n_nodes;
    r->nnz = h_off[n_voxels];
    r->side = side;
    for (int k = 0; k < dim; ++k) {
        r->origin[k] = h_origin[k];
        r->ext[k] = h_extents[k];
    }
    auto cleanup = [&](int32_t st) {
        cudaFree(r->d_off);
        cudaFree(r->d_ids);
        cudaFree(r->d_vox_bits);
        cudaFree(r->d_count);
        cudaFreeHost(r->h_count);
        delete r;
        return st;
    };
    cudaError_t e = cudaMalloc(&r->d_off, sizeof(int64_t) * (n_voxels + 1));
    if (e == cudaSuccess) e = cudaMemcpy(r->d_off, h_off, sizeof(int64_t) * (n_voxels + 1), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&r->d_ids, sizeof(int32_t) * std::max<int64_t>(1, r->nnz));
    if (e == cudaSuccess && r->nnz > 0) e = cudaMemcpy(r->d_ids, h_ids, sizeof(int32_t) * r->nnz, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&r->d_vox_bits, sizeof(uint32_t) * ((n_voxels + 31) / 32));
    if (e == cudaSuccess) e = cudaMalloc(&r->d_count, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMallocHost(&r->h_count, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r->scratch_free, cudaEventDisableTiming);
    if (e != cudaSuccess) return cleanup(cuda_fail(e, "roadmap upload", __FILE__, __LINE__));
    *out = r;
    return EZ_OK;
}

extern "C" int32_t ez_roadmap_destroy(ez_roadmap* r) {
    if (!r) return EZ_OK;
    ::ez::DeviceGuard dg(r->device);
    cudaFree(r->d_off);
    cudaFree(r->d_ids);
    cudaFree(r->d_vox_bits);
    cudaFree(r->d_count);
    cudaFreeHost(r->h_count);
    if (r->scratch_free) cudaEventDestroy(r->scratch_free);
    delete r;
    return EZ_OK;
}

// caller holds r->mu and is on r's device; leaves scratch_free recorded on s
static int32_t prune_locked(ez_roadmap* r, const int32_t* d_vox_idx, int64_t n_vox, const double* h_vmap_origin,
                            double vmap_side, int32_t same_grid, uint32_t* d_blocked_bits, int64_t* n_blocked,
                            cudaStream_t s) {
    const int64_t nbw = (r->n_nodes + 31) / 32;
    EZ_CUDA(cudaMemsetAsync(d_blocked_bits, 0, sizeof(uint32_t) * std::max<int64_t>(1, nbw), s));
    if (n_vox == 0) return EZ_OK;
    EZ_CUDA(cudaStreamWaitEvent(s, r->scratch_free, 0));  // the previous prune is done with the scratch
    const int64_t vbw = (r->n_voxels + 31) / 32;
    EZ_CUDA(cudaMemsetAsync(r->d_vox_bits, 0, sizeof(uint32_t) * vbw, s));
    if (n_blocked) EZ_CUDA(cudaMemsetAsync(r->d_count, 0, sizeof(unsigned long long), s));
    PruneParams pp{};
    for (int k = 0; k < r->dim; ++k) {
        pp.vorg[k] = h_vmap_origin[k];
        pp.gorg[k] = r->origin[k];
        pp.ext[k] = r->ext[k];
    }
    if (r->dim == 2) pp.ext[2] = 1;
    pp.vside = vmap_side;
    pp.gside = r->side;
    pp.dim = r->dim;
    pp.same = same_grid;
    k_activate<<<static_cast<unsigned>((n_vox + 255) / 256), 256, 0, s>>>(d_vox_idx, n_vox, pp, r->d_vox_bits);
    const int64_t want = std::min<int64_t>((r->n_voxels * 32 + 255) / 256, 148 * 16);
    k_gather<<<static_cast<unsigned>(std::max<int64_t>(1, want)), 256, 0, s>>>(r->d_vox_bits, r->n_voxels, r->d_off, r->d_ids,
                                                                            d_blocked_bits);
    EZ_CUDA(cudaGetLastError());
    if (!n_blocked) return EZ_OK;  // no count wanted: stays asynchronous on `stream`
    k_count_bits<<<static_cast<unsigned>(std::min<int64_t>(std::max<int64_t>(1, (nbw + 255) / 256), 296)), 256, 0, s>>>(
        d_blocked_bits, nbw, r->d_count);
    EZ_CUDA(cudaGetLastError());
    EZ_CUDA(cudaMemcpyAsync(r->h_count, r->d_count, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    EZ_CUDA(cudaStreamSynchronize(s));
    *n_blocked = static_cast<int64_t>(*r->h_count);
    return EZ_OK;
}

extern "C" int32_t ez_collision_set(ez_roadmap* r, const int32_t* d_vox_idx, int64_t n_vox, const double* h_vmap_origin,
                                    double vmap_side, int32_t same_grid, uint32_t* d_blocked_bits, int64_t* n_blocked,
                                    void* stream) {
    if (!r) return fail(EZ_INVALID_ARGUMENT, "null roadmap");
    if (n_blocked) *n_blocked = 0;
    EZ_ON_DEVICE(r->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lk(r->mu);
    const int32_t st = prune_locked(r, d_vox_idx, n_vox, h_vmap_origin, vmap_side, same_grid, d_blocked_bits,
                                    n_blocked, s);
    if (st == EZ_OK) EZ_CUDA(cudaEventRecord(r->scratch_free, s));
    return st;
}


extern "C" int32_t ez_collision_set_ids(ez_roadmap* r, const int32_t* d_vox_idx, int64_t n_vox,
                                        const double* h_vmap_origin, double vmap_side, int32_t same_grid,
                                        uint32_t* d_blocked_bits, int32_t* d_ids, int64_t* n_ids, void* stream) {
    if (!r || !n_ids) return fail(EZ_INVALID_ARGUMENT, "null argument");
    *n_ids = 0;
    EZ_ON_DEVICE(r->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lk(r->mu);  // d_count is scratch too
    EZ_TRY(prune_locked(r, d_vox_idx, n_vox, h_vmap_origin, vmap_side, same_grid, d_blocked_bits, nullptr, s));
    if (n_vox == 0) return EZ_OK;
    const int64_t nbw = (r->n_nodes + 31) / 32;
    int64_t* d_n = reinterpret_cast<int64_t*>(r->d_count);
    k_bits_to_ids<<<1, 1024, 0, s>>>(d_blocked_bits, nbw, d_ids, d_n);
    EZ_CUDA(cudaGetLastError());
    EZ_CUDA(cudaMemcpyAsync(r->h_count, d_n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    EZ_CUDA(cudaEventRecord(r->scratch_free, s));
    EZ_CUDA(cudaStreamSynchronize(s));
    *n_ids = static_cast<int64_t>(*r->h_count);
    return EZ_OK;
}
