// ez_drm_build.cu — the DRM collision map built on the GPU.
//
// Replaces corridor/drm.py:170-204 (_node_voxel_pairs) and the CSR assembly of
// drm.py:138-144/250-251: voxel v lists every node whose sphere geometry
// touches the voxel's circumscribing sphere, |t - c_v|^2 <= (r + r_vox)^2 in
// fp64 (no margin), node ids sorted per voxel.
//
// One warp per node: the joint chain runs in every lane, lane l places
// spheres l, l+32, ...; each lane scans the lattice box around its spheres and
// marks hits in the warp's shared-memory voxel bitmap (dedupes nodes that hit
// a voxel through several spheres).  Set bits become 64-bit keys
// (voxel << 32 | node); a device radix sort yields the CSR.
#include <algorithm>
#include <cmath>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "ez_device.cuh"
#include "ez_roadmap.h"
#include "ez_world.h"

namespace ez {

struct MapGrid {
    double org[3];
    double side;
    double r_vox;
    int32_t ext[3];
    int32_t dim;
    int32_t words;  // bitmap words per node
};

template <bool kEmit>
__global__ void __launch_bounds__(256)
k_node_voxels(const __grid_constant__ ModelDev<double> M, const double* __restrict__ nodes, int64_t n, MapGrid g,
              unsigned long long* __restrict__ keys, unsigned long long* __restrict__ n_keys) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint64_t bar;
    tma_stage(smem, M.blob, M.blob_bytes, &bar);
    const int warps = blockDim.x >> 5;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    size_t off = (M.blob_bytes + 15) & ~static_cast<size_t>(15);
    double* cen = reinterpret_cast<double*>(smem + off) + static_cast<size_t>(wid) * M.cen_words;
    off += static_cast<size_t>(warps) * M.cen_words * sizeof(double);
    double* row = reinterpret_cast<double*>(smem + off) + static_cast<size_t>(wid) * 32;
    off += static_cast<size_t>(warps) * 32 * sizeof(double);
    uint32_t* bits = reinterpret_cast<uint32_t*>(smem + off) + static_cast<size_t>(wid) * g.words;
    const JointRec<double>* J = reinterpret_cast<const JointRec<double>*>(smem);
    const SphereRec<double>* S = reinterpret_cast<const SphereRec<double>*>(smem + M.off_spheres);
    const BoxRec<double>* BX = reinterpret_cast<const BoxRec<double>*>(smem + M.off_boxes);
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * warps;
    for (int64_t node = static_cast<int64_t>(blockIdx.x) * warps + wid; node < n; node += nwarps) {
        if (lane < M.dof) row[lane] = nodes[node * M.dof + lane];
        for (int w = lane; w < g.words; w += 32) bits[w] = 0u;
        __syncwarp();
        fk_centres_coop<double, double, 32>(J, M.n_joints, S, row, cen, lane, BX, M.box_base);
        __syncwarp();
        for (int s = lane; s < M.n_spheres; s += 32) {
            const double R = S[s].r + g.r_vox;
            const double thr = R * R;  // (g.radius + r_vox) ** 2
            int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
            for (int k = 0; k < g.dim; ++k) {
                const double c = cen[3 * s + k];
                lo[k] = max(0, static_cast<int>(floor((c - R - g.org[k]) / g.side - 0.5)) - 1);
                hi[k] = min(g.ext[k] - 1, static_cast<int>(floor((c + R - g.org[k]) / g.side - 0.5)) + 1);
            }
            for (int z = lo[2]; z <= hi[2]; ++z) {
                double dz2 = 0.0;
                if (g.dim == 3) {
                    const double dz = __dsub_rn(cen[3 * s + 2], lattice_centre(g.org[2], z, g.side));
                    dz2 = __dmul_rn(dz, dz);
                }
                for (int y = lo[1]; y <= hi[1]; ++y) {
                    const double dy = __dsub_rn(cen[3 * s + 1], lattice_centre(g.org[1], y, g.side));
                    const double dy2 = __dmul_rn(dy, dy);
                    for (int x = lo[0]; x <= hi[0]; ++x) {
                        const double dx = __dsub_rn(cen[3 * s], lattice_centre(g.org[0], x, g.side));
                        // numpy: ((dx^2 + dy^2) + dz^2) <= (r + r_vox)^2
                        const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), dy2), dz2);
                        if (d2 <= thr) {
                            const int64_t vid = (static_cast<int64_t>(z) * g.ext[1] + y) * g.ext[0] + x;
                            atomicOr(bits + (vid >> 5), 1u << (vid & 31));
                        }
                    }
                }
            }
        }
        // boxes: |local - clip(local)|^2 <= r_vox^2 with local = R^T (c_v - t) (drm.py:186-189)
        for (int b = lane; b < M.n_boxes; b += 32) {
            double Rb[9], tb[3];
            load_box<double>(cen, 1, M.box_base + 12 * b, Rb, tb);
            const double* he = BX[b].he;
            const double thr = g.r_vox * g.r_vox;
            int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
            for (int k = 0; k < g.dim; ++k) {
                const double ext = fabs(Rb[3 * k]) * he[0] + fabs(Rb[3 * k + 1]) * he[1] + fabs(Rb[3 * k + 2]) * he[2] + g.r_vox;
                lo[k] = max(0, static_cast<int>(floor((tb[k] - ext - g.org[k]) / g.side - 0.5)) - 1);
                hi[k] = min(g.ext[k] - 1, static_cast<int>(floor((tb[k] + ext - g.org[k]) / g.side - 0.5)) + 1);
            }
            for (int z = lo[2]; z <= hi[2]; ++z)
                for (int y = lo[1]; y <= hi[1]; ++y)
                    for (int x = lo[0]; x <= hi[0]; ++x) {
                        const double d2 = point_box_d2<double>(Rb, tb, he, lattice_centre(g.org[0], x, g.side),
                                                               lattice_centre(g.org[1], y, g.side),
                                                               g.dim == 3 ? lattice_centre(g.org[2], z, g.side) : 0.0);
                        if (d2 <= thr) {
                            const int64_t vid = (static_cast<int64_t>(z) * g.ext[1] + y) * g.ext[0] + x;
                            atomicOr(bits + (vid >> 5), 1u << (vid & 31));
                        }
                    }
        }
        __syncwarp();
        // emit the set bits of this node's bitmap
        int cnt = 0;
        for (int w = lane; w < g.words; w += 32) cnt += __popc(bits[w]);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        unsigned long long base = 0;
        if (lane == 31 && total) base = atomicAdd(n_keys, static_cast<unsigned long long>(total));
        base = __shfl_sync(0xffffffffu, base, 31);
        if (kEmit) {
            unsigned long long o = base + static_cast<unsigned long long>(incl - cnt);
            for (int w = lane; w < g.words; w += 32) {
                uint32_t b = bits[w];
                while (b) {
                    const int p = __ffs(b) - 1;
                    b &= b - 1;
                    const unsigned long long vid = static_cast<unsigned long long>(w) * 32 + p;
                    keys[o++] = (vid << 32) | static_cast<unsigned long long>(node);
                }
            }
        }
        __syncwarp();
    }
}

__global__ void k_key_split(const unsigned long long* __restrict__ keys, int64_t nnz, int32_t* __restrict__ ids,
                            unsigned long long* __restrict__ counts) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nnz) return;
    const unsigned long long k = keys[i];
    ids[i] = static_cast<int32_t>(k & 0xffffffffull);
    atomicAdd(counts + (k >> 32), 1ull);
}

__global__ void k_offsets_finish(const unsigned long long* __restrict__ excl, int64_t n_vox, int64_t nnz,
                                 int64_t* __restrict__ off) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n_vox) off[i] = static_cast<int64_t>(excl[i]);
    if (i == 0) off[n_vox] = nnz;
}

}  // namespace ez

using namespace ez;

extern "C" int32_t ez_roadmap_build(ez_world* w, const double* d_nodes, int64_t n_nodes, int32_t dim,
                                    const double* h_origin, double side, const int32_t* h_extents, void* stream,
                                    ez_roadmap** out) {
    if (!w || !out || !h_origin || !h_extents) return fail(EZ_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    if (dim != w->dim) return fail(EZ_DIMENSION_MISMATCH, "grid dimension differs from the robot's task space");
    if (!(side > 0.0)) return fail(EZ_INVALID_ARGUMENT, "grid side must be positive");
    if (w->dof > 32) return fail(EZ_UNSUPPORTED, "more than 32 degrees of freedom");
    EZ_ON_DEVICE(w->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    MapGrid g{};
    int64_t n_vox = 1;
    for (int k = 0; k < 3; ++k) {
        g.ext[k] = k < dim ? h_extents[k] : 1;
        g.org[k] = k < dim ? h_origin[k] : 0.0;
        n_vox *= g.ext[k];
    }
    if (dim == 2) g.org[2] = -0.5 * side;  // planar voxels at z = 0
    g.side = side;
    g.dim = dim;
    g.r_vox = 0.5 * side * std::sqrt(static_cast<double>(dim));  // Grid.sphere_radius (drm.py:50-51)
    g.words = static_cast<int32_t>((n_vox + 31) / 32);
    if (n_vox >= (int64_t(1) << 31)) return fail(EZ_CAPACITY, "roadmap grid too large");
    const ModelDev<double>& M = w->md;
    int warps = 8;
    auto smem_for = [&](int wps) {
        size_t b = (M.blob_bytes + 15) & ~static_cast<size_t>(15);
        b += static_cast<size_t>(wps) * M.cen_words * sizeof(double);
        b += static_cast<size_t>(wps) * 32 * sizeof(double);
        b += static_cast<size_t>(wps) * g.words * sizeof(uint32_t);
        return b;
    };
    while (warps > 1 && smem_for(warps) > 160 * 1024) warps /= 2;
    const size_t smem = smem_for(warps);
    if (smem > static_cast<size_t>(w->smem_optin) - 2048) return fail(EZ_CAPACITY, "roadmap grid bitmap exceeds shared memory");
    EZ_TRY(allow_max_dyn_smem(k_node_voxels<false>));
    EZ_TRY(allow_max_dyn_smem(k_node_voxels<true>));
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>((n_nodes + warps - 1) / warps, 148 * 8));
    // temporaries come from the stream-ordered pool (kept mapped between builds)
    EZ_TRY(retain_async_pool());
    unsigned long long* d_cnt = nullptr;
    EZ_CUDA(cudaMallocAsync(&d_cnt, sizeof(unsigned long long), s));
    EZ_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), s));
    if (n_nodes > 0)
        k_node_voxels<false><<<grid, warps * 32, smem, s>>>(M, d_nodes, n_nodes, g, nullptr, d_cnt);
    EZ_CUDA(cudaGetLastError());
    unsigned long long nnz = 0;
    EZ_CUDA(cudaMemcpyAsync(&nnz, d_cnt, sizeof(nnz), cudaMemcpyDeviceToHost, s));
    EZ_CUDA(cudaStreamSynchronize(s));

    ez_roadmap* r = new ez_roadmap();
    r->device = w->device;
    r->dim = dim;
    r->n_voxels = n_vox;
    r->n_nodes = n_nodes;
    r->nnz = static_cast<int64_t>(nnz);
    r->side = side;
    for (int k = 0; k < dim; ++k) {
        r->origin[k] = h_origin[k];
        r->ext[k] = h_extents[k];
    }
    unsigned long long *keys = nullptr, *keys_sorted = nullptr, *counts = nullptr, *excl = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0, scan_bytes = 0;
    auto cleanup = [&]() {
        cudaFreeAsync(keys, s);
        cudaFreeAsync(keys_sorted, s);
        cudaFreeAsync(counts, s);
        cudaFreeAsync(excl, s);
        cudaFreeAsync(tmp, s);
        cudaFreeAsync(d_cnt, s);
        cudaStreamSynchronize(s);
    };
    cudaError_t e = cudaSuccess;
    const size_t nk = std::max<unsigned long long>(1, nnz);
    if (e == cudaSuccess) e = cudaMallocAsync(&keys, sizeof(unsigned long long) * nk, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&keys_sorted, sizeof(unsigned long long) * nk, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&counts, sizeof(unsigned long long) * n_vox, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&excl, sizeof(unsigned long long) * n_vox, s);
    if (e == cudaSuccess) e = cudaMalloc(&r->d_off, sizeof(int64_t) * (n_vox + 1));
    if (e == cudaSuccess) e = cudaMalloc(&r->d_ids, sizeof(int32_t) * nk);
    if (e == cudaSuccess) e = cudaMalloc(&r->d_vox_bits, sizeof(uint32_t) * ((n_vox + 31) / 32));
    if (e == cudaSuccess) e = cudaMalloc(&r->d_count, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMallocHost(&r->h_count, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r->scratch_free, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * n_vox, s);
    if (e == cudaSuccess && n_nodes > 0) {
        k_node_voxels<true><<<grid, warps * 32, smem, s>>>(M, d_nodes, n_nodes, g, keys, d_cnt);
        e = cudaGetLastError();
    }
    // sort (voxel, node) keys: CSR by voxel with node ids ascending
    int end_bit = 32;
    while ((int64_t(1) << (end_bit - 32)) < n_vox && end_bit < 64) ++end_bit;
    if (e == cudaSuccess)
        e = cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys, keys_sorted, static_cast<int64_t>(nnz), 0, end_bit, s);
    if (e == cudaSuccess)
        e = cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, counts, excl, static_cast<int>(n_vox), s);
    if (e == cudaSuccess) e = cudaMallocAsync(&tmp, std::max(tmp_bytes, scan_bytes), s);
    if (e == cudaSuccess && nnz > 0)
        e = cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, keys, keys_sorted, static_cast<int64_t>(nnz), 0, end_bit, s);
    if (e == cudaSuccess && nnz > 0) {
        k_key_split<<<static_cast<unsigned>((nnz + 255) / 256), 256, 0, s>>>(keys_sorted, static_cast<int64_t>(nnz),
                                                                           r->d_ids, counts);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, counts, excl, static_cast<int>(n_vox), s);
    if (e == cudaSuccess) {
        k_offsets_finish<<<static_cast<unsigned>((n_vox + 256) / 256), 256, 0, s>>>(excl, n_vox, static_cast<int64_t>(nnz),
                                                                                  r->d_off);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cleanup();
    if (e != cudaSuccess) {
        ez_roadmap_destroy(r);
        return cuda_fail(e, "roadmap build", __FILE__, __LINE__);
    }
    *out = r;
    return EZ_OK;
}

extern "C" int32_t ez_roadmap_info(const ez_roadmap* r, int64_t* n_voxels, int64_t* n_nodes, int64_t* nnz) {
    if (!r) return fail(EZ_INVALID_ARGUMENT, "null roadmap");
    if (n_voxels) *n_voxels = r->n_voxels;
    if (n_nodes) *n_nodes = r->n_nodes;
    if (nnz) *nnz = r->nnz;
    return EZ_OK;
}

extern "C" int32_t ez_roadmap_export(const ez_roadmap* r, int64_t* h_offsets, int32_t* h_ids) {
    if (!r) return fail(EZ_INVALID_ARGUMENT, "null roadmap");
    EZ_ON_DEVICE(r->device);
    if (h_offsets) EZ_CUDA(cudaMemcpy(h_offsets, r->d_off, sizeof(int64_t) * (r->n_voxels + 1), cudaMemcpyDeviceToHost));
    if (h_ids && r->nnz) EZ_CUDA(cudaMemcpy(h_ids, r->d_ids, sizeof(int32_t) * r->nnz, cudaMemcpyDeviceToHost));
    return EZ_OK;
}
