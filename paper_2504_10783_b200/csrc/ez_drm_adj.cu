// ez_drm_adj.cu — DRM roadmap adjacency built on the GPU.
//
// Replaces the edge construction of corridor/drm.py:build_drm (219-248):
//   cKDTree.query(nodes, k = min(n, 4k + 1)) -> for each node i, its
//   neighbours in ascending configuration distance, position 0 (the node
//   itself) skipped; stop at the first distance > d_cs; skip j whose
//   end-effector distance exceeds d_ts; keep at most k -> symmetrise
//   (unique (i, j) and (j, i)) -> CSR rows sorted by neighbour id.
//
// k_knn_edges: one warp per node.  Lane l scans the candidates j = l, l + 32,
// ... and keeps its own ascending top-K list (distance^2, index) in shared
// memory (insertion only when a candidate beats the lane's K-th, rare after
// the first few hundred).  The 32 lists are merged by K rounds of a warp
// arg-min; the merged order is lexicographic (distance, index), which is
// cKDTree's order for distinct distances.  Distances are fp64 sums of
// squares in coordinate order without FMA contraction (scipy's kernel
// arithmetic), then sqrt, as the d_cs test compares cKDTree's distances.
// Emitted edges become 64-bit keys (row << 32 | col) in both directions; a
// radix sort, a unique pass and a row count give the CSR.
#include <algorithm>
#include <cmath>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "ez_common.h"

namespace ez {
namespace {

constexpr int kKnnWarps = 8;     // warps (query nodes) per CTA
constexpr int kKnnMaxK = 64;     // top-K capacity per lane
constexpr int kKnnMaxDof = 32;

constexpr int kKnnTile = 256;  // candidates staged per CTA round

__global__ void __launch_bounds__(32 * kKnnWarps)
k_knn_edges(const double* __restrict__ X, int64_t n, int d, const double* __restrict__ E, int de, int K, int k_keep,
            double d_cs, double d_ts, unsigned long long* __restrict__ keys, unsigned long long* __restrict__ n_keys) {
    // shared: the candidate tile [kKnnTile][d], then per lane K (d2, idx)
    // entries (struct of arrays); every warp of the CTA scans the same tiles
    extern __shared__ __align__(16) uint8_t smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* s_x = reinterpret_cast<double*>(smem);
    double* s_d = s_x + static_cast<size_t>(kKnnTile) * d + (static_cast<size_t>(wid) * 32 + lane) * K;
    int32_t* s_i = reinterpret_cast<int32_t*>(s_x + static_cast<size_t>(kKnnTile) * d +
                                              static_cast<size_t>(kKnnWarps) * 32 * K) +
                   (static_cast<size_t>(wid) * 32 + lane) * K;
    for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * kKnnWarps; i0 < n;
         i0 += static_cast<int64_t>(gridDim.x) * kKnnWarps) {
        const int64_t i = i0 + wid;
        const bool active = i < n;
        double xi[kKnnMaxDof];
#pragma unroll
        for (int k = 0; k < kKnnMaxDof; ++k)
            if (k < d) xi[k] = active ? X[i * d + k] : 0.0;
        int cnt = 0;
        double kth = INFINITY;  // the lane's K-th smallest once it holds K
        for (int64_t t0 = 0; t0 < n; t0 += kKnnTile) {
            const int tn = static_cast<int>(n - t0 < kKnnTile ? n - t0 : kKnnTile);
            __syncthreads();
            for (int e = threadIdx.x; e < tn * d; e += blockDim.x) s_x[e] = X[t0 * d + e];
            __syncthreads();
            if (!active) continue;
            for (int jj = lane; jj < tn; jj += 32) {
                const double* xj = s_x + static_cast<size_t>(jj) * d;
                double s = 0.0;
#pragma unroll
                for (int k = 0; k < kKnnMaxDof; ++k)
                    if (k < d) {
                        const double t = __dsub_rn(xi[k], xj[k]);
                        s = __dadd_rn(s, __dmul_rn(t, t));
                    }
                if (cnt == K && !(s < kth)) continue;  // ties keep the lower index (scan order is ascending)
                int p = cnt < K ? cnt : K - 1;
                while (p > 0 && s_d[p - 1] > s) {  // strictly greater: equal distances stay in index order
                    s_d[p] = s_d[p - 1];
                    s_i[p] = s_i[p - 1];
                    --p;
                }
                s_d[p] = s;
                s_i[p] = static_cast<int32_t>(t0 + jj);
                if (cnt < K) ++cnt;
                if (cnt == K) kth = s_d[K - 1];
            }
        }
        if (!active) continue;
        // merge the 32 sorted lists: K rounds of a warp arg-min on (d2, index)
        int head = 0, picked = 0;
        bool stop = false;
        for (int pos = 0; pos < K && !stop; ++pos) {
            double hd = head < cnt ? s_d[head] : INFINITY;
            int32_t hi = head < cnt ? s_i[head] : INT32_MAX;
            double bd = hd;
            int32_t bi = hi;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double od = __shfl_xor_sync(0xffffffffu, bd, o);
                const int32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (od < bd || (od == bd && oi < bi)) {
                    bd = od;
                    bi = oi;
                }
            }
            if (bi == INT32_MAX) break;  // fewer than K candidates in all
            if (hi == bi && hd == bd) ++head;
            if (pos == 0) continue;  // the query itself (drm.py:224, j_pos from 1)
            if (sqrt(bd) > d_cs) {   // ascending: nothing further qualifies (drm.py:226-227)
                stop = true;
                break;
            }
            // end-effector distance (drm.py:228-229), evaluated by every lane
            double e2 = 0.0;
            for (int k = 0; k < de; ++k) {
                const double t = __dsub_rn(E[i * de + k], E[static_cast<int64_t>(bi) * de + k]);
                e2 = __dadd_rn(e2, __dmul_rn(t, t));
            }
            if (sqrt(e2) > d_ts) continue;
            if (lane == 0) {
                const unsigned long long a = static_cast<unsigned long long>(i), b = static_cast<unsigned long long>(bi);
                const unsigned long long slot = atomicAdd(n_keys, 2ull);
                keys[slot] = (a << 32) | b;
                keys[slot + 1] = (b << 32) | a;
            }
            if (++picked >= k_keep) stop = true;
        }
        __syncwarp();
    }
}

// CSR offsets of unique sorted keys: row r starts at the first key with row >= r
__global__ void k_adj_offsets(const unsigned long long* __restrict__ keys, int64_t nnz, int64_t n,
                              int64_t* __restrict__ off) {
    for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r <= n;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int64_t lo = 0, hi = nnz;  // first index with (key >> 32) >= r
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (static_cast<int64_t>(keys[mid] >> 32) < r) lo = mid + 1;
            else hi = mid;
        }
        off[r] = lo;
    }
}

__global__ void k_adj_ids(const unsigned long long* __restrict__ keys, int64_t nnz, int32_t* __restrict__ ids) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x)
        ids[e] = static_cast<int32_t>(keys[e] & 0xFFFFFFFFull);
}

}  // namespace
}  // namespace ez

using namespace ez;

extern "C" int32_t ez_roadmap_adjacency(const double* d_nodes, int64_t n_nodes, int32_t dof, const double* d_ee,
                                        int32_t ee_dim, int32_t k, double d_cs, double d_ts, int64_t* d_adj_offsets,
                                        int32_t* d_adj_ids, int64_t* nnz, void* stream) {
    if (!d_nodes || !d_ee || !d_adj_offsets || !d_adj_ids || !nnz) return fail(EZ_INVALID_ARGUMENT, "null argument");
    *nnz = 0;
    if (n_nodes < 2) return fail(EZ_INVALID_ARGUMENT, "need at least two nodes");
    if (k < 1) return fail(EZ_INVALID_ARGUMENT, "k must be >= 1");
    if (dof < 1 || dof > kKnnMaxDof || ee_dim < 1) return fail(EZ_UNSUPPORTED, "1..32 degrees of freedom");
    if (n_nodes >= (int64_t(1) << 31)) return fail(EZ_CAPACITY, "too many roadmap nodes");
    const int K = static_cast<int>(std::min<int64_t>(n_nodes, 4 * static_cast<int64_t>(k) + 1));  // drm.py:222
    if (K > kKnnMaxK) return fail(EZ_UNSUPPORTED, "k above 15 (neighbour query of more than 64)");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    EZ_TRY(retain_async_pool());
    int dev = 0, optin = 0;
    EZ_CUDA(cudaGetDevice(&dev));
    EZ_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (static_cast<size_t>(kKnnTile) * dof * sizeof(double) +
            static_cast<size_t>(kKnnWarps) * 32 * K * (sizeof(double) + sizeof(int32_t)) > static_cast<size_t>(optin))
        return fail(EZ_UNSUPPORTED, "neighbour lists of this k and dof exceed shared memory");
    const int64_t cap = 2 * static_cast<int64_t>(k) * n_nodes;
    unsigned long long *keys = nullptr, *sorted = nullptr, *uniq = nullptr, *d_cnt = nullptr;
    int64_t* d_nuniq = nullptr;
    void* tmp = nullptr;
    int32_t st = EZ_OK;
    auto ck = [&](cudaError_t e, const char* what) {
        if (e != cudaSuccess && st == EZ_OK) st = cuda_fail(e, what, __FILE__, __LINE__);
        return st == EZ_OK;
    };
    const size_t smem = static_cast<size_t>(kKnnTile) * dof * sizeof(double) +
                        static_cast<size_t>(kKnnWarps) * 32 * K * (sizeof(double) + sizeof(int32_t));
    unsigned long long h_cnt = 0;
    int64_t h_uniq = 0;
    if (ck(cudaMallocAsync(&keys, sizeof(unsigned long long) * std::max<int64_t>(1, cap), s), "alloc keys") &&
        ck(cudaMallocAsync(&sorted, sizeof(unsigned long long) * std::max<int64_t>(1, cap), s), "alloc sorted") &&
        ck(cudaMallocAsync(&uniq, sizeof(unsigned long long) * std::max<int64_t>(1, cap), s), "alloc unique") &&
        ck(cudaMallocAsync(&d_cnt, sizeof(unsigned long long), s), "alloc count") &&
        ck(cudaMallocAsync(&d_nuniq, sizeof(int64_t), s), "alloc count") &&
        ck(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), s), "memset") &&
        (st = allow_max_dyn_smem(k_knn_edges)) == EZ_OK) {
        const unsigned grid = static_cast<unsigned>((n_nodes + kKnnWarps - 1) / kKnnWarps);
        k_knn_edges<<<grid, 32 * kKnnWarps, smem, s>>>(d_nodes, n_nodes, dof, d_ee, ee_dim, K, k, d_cs, d_ts, keys,
                                                       d_cnt);
        if (ck(cudaGetLastError(), "k_knn_edges") &&
            ck(cudaMemcpyAsync(&h_cnt, d_cnt, sizeof(h_cnt), cudaMemcpyDeviceToHost, s), "count") &&
            ck(cudaStreamSynchronize(s), "k_knn_edges")) {
            size_t sort_bytes = 0, uniq_bytes = 0;
            const int64_t m = static_cast<int64_t>(h_cnt);
            int end_bit = 32;
            while ((int64_t(1) << (end_bit - 32)) < n_nodes && end_bit < 64) ++end_bit;
            if (ck(cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, keys, sorted, m, 0, end_bit, s), "sort size") &&
                ck(cub::DeviceSelect::Unique(nullptr, uniq_bytes, sorted, uniq, d_nuniq, m, s), "unique size") &&
                ck(cudaMallocAsync(&tmp, std::max<size_t>(1, std::max(sort_bytes, uniq_bytes)), s), "alloc tmp") &&
                ck(cub::DeviceRadixSort::SortKeys(tmp, sort_bytes, keys, sorted, m, 0, end_bit, s), "sort") &&
                ck(cub::DeviceSelect::Unique(tmp, uniq_bytes, sorted, uniq, d_nuniq, m, s), "unique") &&
                ck(cudaMemcpyAsync(&h_uniq, d_nuniq, sizeof(h_uniq), cudaMemcpyDeviceToHost, s), "count") &&
                ck(cudaStreamSynchronize(s), "unique")) {
                k_adj_offsets<<<static_cast<unsigned>(std::min<int64_t>((n_nodes + 256) / 256, 4096)), 256, 0, s>>>(
                    uniq, h_uniq, n_nodes, d_adj_offsets);
                if (h_uniq > 0)
                    k_adj_ids<<<static_cast<unsigned>(std::min<int64_t>((h_uniq + 255) / 256, 4096)), 256, 0, s>>>(
                        uniq, h_uniq, d_adj_ids);
                if (ck(cudaGetLastError(), "adjacency CSR")) *nnz = h_uniq;
            }
        }
    }
    cudaFreeAsync(keys, s);
    cudaFreeAsync(sorted, s);
    cudaFreeAsync(uniq, s);
    cudaFreeAsync(d_cnt, s);
    cudaFreeAsync(d_nuniq, s);
    if (tmp) cudaFreeAsync(tmp, s);
    if (st == EZ_OK) ck(cudaStreamSynchronize(s), "adjacency");
    return st;
}
