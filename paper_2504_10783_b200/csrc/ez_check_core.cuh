// ez_check_core.cuh — the tile loop of the fused FK + collision check,
// shared by the generic kernel (model read from the staged blob) and the
// per-model kernels compiled at run time (ez_jit.cu).  Replaces
// corridor/world.py:483-517 (check_batch / _check_chunk).
//
// Two phases per tile of bt configurations (one CTA):
//   A) every thread: FK + the calibrated hot self pairs.  Most colliding
//      configurations are decided here.
//   B) survivors are appended (in index order) to a CTA ring buffer; whenever
//      a full CTA's worth is queued, every thread takes one, reloads its row,
//      recomputes FK and runs the obstacle tests and remaining pairs.  Phase
//      B therefore always runs on full warps and no warp idles at a barrier
//      while a few lanes finish the expensive tail.
//
// A policy P supplies the model:
//   bool a(const Q* row, T* cen) const   phase A, true = collides
//   bool b(const Q* row, T* cen) const   phase B, true = collides
//   static constexpr bool kRegRows
// `cen` is the thread's centre store (element k at cen[k * BT]).  With
// kRegRows (a policy whose joint count is a compile-time constant: the
// run-time compiled kernels) `row` is a register array loaded by the thread
// itself, the next tile's row prefetched, and the CTA meets at two barriers
// per tile; otherwise rows are staged through shared memory.
#pragma once

#include "ez_device.cuh"

namespace ez {

constexpr int kPrefetch = 8;  // registers per thread for the next tile's rows (dof*BT/BT <= 8)

template <typename T, typename Q, int BT, class P>
__device__ __forceinline__ void check_phase_b(const P& pol, int dof, const Q* __restrict__ q, int64_t ld, int64_t idx,
                                              Q* row, T* cen, uint8_t* __restrict__ out, int64_t count_lim,
                                              int32_t* n_col) {
    Q v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k)
        if (k < dof) v[k] = q[idx * ld + k];
#pragma unroll
    for (int k = 0; k < 32; ++k)
        if (k < dof) row[k] = v[k];
    const bool c2 = pol.b(row, cen);
    out[idx] = c2 ? 0 : 1;
    if (n_col != nullptr && c2 && idx < count_lim) atomicAdd(n_col, 1);
}

// Register-row variant (P::kRegRows): no shared-memory rows, so neither the
// staging barriers nor a barrier per phase-B round.  The two barriers left per
// tile publish the per-warp survivor counts and then the queue; a thread that
// passes the first one of the next tile knows every thread has finished this
// tile's rounds, so queue slots and s_warp are never overwritten early.
//
// s_pf (bt rows of dof, or nullptr): the next tile's row is prefetched with
// cp.async into the thread's own shared-memory slot, so it occupies no
// registers while this tile is checked.  (Held in registers across phase B
// at 64 registers, the prefetched row was spilled right after its load, and
// the spill store waited for the load: 4% of the stall samples.)
template <typename Q>
__device__ __forceinline__ void cp_async_elem(Q* dst, const Q* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"(sizeof(Q))
                 : "memory");
}

template <typename T, typename Q, int BT, class P>
__device__ __forceinline__ void check_tiles_reg(const P& pol, int dof, int32_t* s_queue, int* s_warp, Q* s_pf,
                                                const Q* __restrict__ q, int64_t n, int64_t ld,
                                                uint8_t* __restrict__ out, int64_t count_lim,
                                                int32_t* __restrict__ n_col) {
    const int bt = BT > 0 ? BT : static_cast<int>(blockDim.x);
    const int qcap = 2 * bt;
    auto wrap = [&](int x) { return BT > 0 ? x % qcap : (x & (qcap - 1)); };
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#ifdef EZ_CHECK_NO_PF
    const bool pre = false;
#else
    const bool pre = s_pf == nullptr && dof <= kPrefetch;  // prefetch the next tile's row in registers
#endif
    int qhead = 0, qn = 0;
    const int64_t tiles = (n + bt - 1) / bt;
    Q nxt[kPrefetch];
    auto prefetch = [&](int64_t tile) {
        const int64_t r = tile * bt + threadIdx.x;
        if (tile < tiles && r < n) {
#pragma unroll
            for (int k = 0; k < kPrefetch; ++k)
                if (k < dof) nxt[k] = q[r * ld + k];
        }
    };
    Q* my_pf = s_pf != nullptr ? s_pf + threadIdx.x * dof : nullptr;
    auto prefetch_sm = [&](int64_t tile) {
        const int64_t r = tile * bt + threadIdx.x;
        if (tile < tiles && r < n) {
#pragma unroll
            for (int k = 0; k < 32; ++k)
                if (k < dof) cp_async_elem(my_pf + k, q + r * ld + k);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (pre) prefetch(blockIdx.x);
    if (my_pf != nullptr) prefetch_sm(blockIdx.x);
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int64_t base = tile * bt;
        const int nr = static_cast<int>(min(static_cast<int64_t>(bt), n - base));
        const bool valid = threadIdx.x < nr;
        bool col = false;
        if (valid) {
            Q row[32];
            if (my_pf != nullptr) {
                asm volatile("cp.async.wait_group 0;" ::: "memory");  // this thread's own copies
#pragma unroll
                for (int k = 0; k < 32; ++k)
                    if (k < dof) row[k] = my_pf[k];
                prefetch_sm(tile + gridDim.x);  // lands while this tile is checked
            } else if (pre) {
#pragma unroll
                for (int k = 0; k < kPrefetch; ++k)
                    if (k < dof) row[k] = nxt[k];
                prefetch(tile + gridDim.x);  // lands while this tile is checked
            } else {
#pragma unroll
                for (int k = 0; k < 32; ++k)
                    if (k < dof) row[k] = q[(base + threadIdx.x) * ld + k];
            }
            col = pol.a(row, static_cast<T*>(nullptr));
            if (col) out[base + threadIdx.x] = 0;
        }
        if (n_col != nullptr) {
            const unsigned m = __ballot_sync(0xffffffffu, col && (base + threadIdx.x) < count_lim);
            if (lane == 0 && m) atomicAdd(n_col, __popc(m));
        }
        const bool surv = valid && !col;
        const unsigned sm = __ballot_sync(0xffffffffu, surv);
        if (lane == 0) s_warp[wid] = __popc(sm);
        __syncthreads();
        // survivors in earlier warps (off) and in the tile (add): lane l reads
        // warp l's count, two warp reductions (a per-thread loop over the 32
        // counts was ~95 instructions per thread per tile)
        const int wc = lane < bt / 32 ? s_warp[lane] : 0;
        const int off = static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(lane < wid ? wc : 0)));
        const int add = static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(wc)));
        if (surv)
            s_queue[wrap(qhead + qn + off + __popc(sm & ((1u << lane) - 1u)))] = static_cast<int32_t>(base + threadIdx.x);
        qn += add;
        __syncthreads();
        const bool last = tile + gridDim.x >= tiles;
        while (qn >= bt || (last && qn > 0)) {
            if (threadIdx.x < min(qn, bt)) {
                const int64_t idx = s_queue[wrap(qhead + threadIdx.x)];
                Q row[32];
#pragma unroll
                for (int k = 0; k < 32; ++k)
                    if (k < dof) row[k] = q[idx * ld + k];
                const bool c2 = pol.b(row, static_cast<T*>(nullptr));
                out[idx] = c2 ? 0 : 1;
                if (n_col != nullptr && c2 && idx < count_lim) atomicAdd(n_col, 1);
            }
            const int took = min(qn, bt);
            qhead = wrap(qhead + took);
            qn -= took;
        }
    }
}

// Small batches (the EI-ZO loop's 10-15k samples): one row per thread, the
// policy's full() check (one FK), no survivor queue.  The tile loop's phase B
// recomputes the FK (twice in the streamed variant) and meets at barriers,
// which costs latency when every thread has a single row.
template <typename Q, class P>
__device__ __forceinline__ void check_rows_full(const P& pol, int dof, const Q* __restrict__ q, int64_t n, int64_t ld,
                                                uint8_t* __restrict__ out, int64_t count_lim,
                                                int32_t* __restrict__ n_col) {
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        Q row[32];
#pragma unroll
        for (int k = 0; k < 32; ++k)
            if (k < dof) row[k] = q[r * ld + k];
        const bool col = pol.full(row, static_cast<float*>(nullptr));
        out[r] = col ? 0 : 1;
        if (n_col != nullptr && col && r < count_lim) atomicAdd(n_col, 1);
    }
}

// rows: bt * dof staging slots in shared memory; s_queue: 2 * bt entries;
// s_warp: bt / 32 entries; cen: this thread's centre store.  The CTA size bt
// is BT, or blockDim.x for BT = 0 (one kernel launched at several sizes).
template <typename T, typename Q, int BT, class P>
__device__ __forceinline__ void check_tiles(const P& pol, int dof, T* my_cen, Q* rows, int32_t* s_queue, int* s_warp,
                                            const Q* __restrict__ q, int64_t n, int64_t ld,
                                            uint8_t* __restrict__ out, int64_t count_lim, int32_t* __restrict__ n_col) {
    const int bt = BT > 0 ? BT : static_cast<int>(blockDim.x);
    const int qcap = 2 * bt;
    // ring index; a run-time CTA size is a power of two
    auto wrap = [&](int x) { return BT > 0 ? x % qcap : (x & (qcap - 1)); };
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    Q* my_row = rows + threadIdx.x * dof;
    const bool contiguous = (ld == dof) && (dof <= kPrefetch);
    int qhead = 0, qn = 0;  // ring buffer state (uniform across the CTA)
    const int64_t tiles = (n + bt - 1) / bt;
    Q pf[kPrefetch];
    auto prefetch = [&](int64_t tile) {
        if (tile >= tiles) return;
        const int64_t base = tile * bt;
        const int tot = static_cast<int>(min(static_cast<int64_t>(bt), n - base)) * dof;
        const Q* src = q + base * dof;
#pragma unroll
        for (int j = 0; j < kPrefetch; ++j) {
            const int i = threadIdx.x + j * bt;
            if (i < tot) pf[j] = src[i];
        }
    };
    if (contiguous) prefetch(blockIdx.x);
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int64_t base = tile * bt;
        const int nr = static_cast<int>(min(static_cast<int64_t>(bt), n - base));
        __syncthreads();
        if (contiguous) {
            const int tot = nr * dof;
#pragma unroll
            for (int j = 0; j < kPrefetch; ++j) {
                const int i = threadIdx.x + j * bt;
                if (i < tot) rows[i] = pf[j];
            }
        } else {
            for (int i = threadIdx.x; i < nr * dof; i += bt) {
                const int r = i / dof, k = i - r * dof;
                rows[i] = q[(base + r) * ld + k];
            }
        }
        __syncthreads();
        if (contiguous) prefetch(tile + gridDim.x);  // lands while this tile is checked
        // phase A
        const bool valid = threadIdx.x < nr;
        bool col = false;
        if (valid) {
            col = pol.a(my_row, my_cen);
            if (col) out[base + threadIdx.x] = 0;
        }
        if (n_col != nullptr) {
            const unsigned m = __ballot_sync(0xffffffffu, col && (base + threadIdx.x) < count_lim);
            if (lane == 0 && m) atomicAdd(n_col, __popc(m));
        }
        // append the survivors to the queue, in index order
        const bool surv = valid && !col;
        const unsigned sm = __ballot_sync(0xffffffffu, surv);
        if (lane == 0) s_warp[wid] = __popc(sm);
        __syncthreads();
        // (the generic kernels keep the per-thread loop over the warp counts:
        // with the two warp reductions of check_tiles_reg the fp64 kernel ran
        // 479 -> 614 us per 2^20)
        int off = 0, add = 0;
        for (int w = 0; w < bt / 32; ++w) {
            const int c = s_warp[w];
            off += (w < wid) ? c : 0;
            add += c;
        }
        if (surv)
            s_queue[wrap(qhead + qn + off + __popc(sm & ((1u << lane) - 1u)))] = static_cast<int32_t>(base + threadIdx.x);
        qn += add;
        __syncthreads();
        // phase B on full CTAs; after the last tile, the partial rest
        const bool last = tile + gridDim.x >= tiles;
        while (qn >= bt || (last && qn > 0)) {
            if (threadIdx.x < min(qn, bt))
                check_phase_b<T, Q, BT>(pol, dof, q, ld, s_queue[wrap(qhead + threadIdx.x)], my_row, my_cen, out,
                                        count_lim, n_col);
            const int took = min(qn, bt);
            qhead = wrap(qhead + took);
            qn -= took;
            __syncthreads();
        }
    }
}

// The generic policy: the model is the blob staged in shared memory.
template <typename T, int BT>
struct BlobPolicy {
    static constexpr bool kRegRows = false;  // run-time joint count: rows stay in shared memory
    const ModelDev<T>& M;
    const uint8_t* smem;
    T margin;
    template <typename Q>
    __device__ __forceinline__ void fk(const Q* row, T* cen) const {
        fk_sphere_centres<T, Q>(reinterpret_cast<const JointRec<T>*>(smem), M.n_joints,
                                reinterpret_cast<const SphereRec<T>*>(smem + M.off_spheres), row, cen, BT,
                                reinterpret_cast<const BoxRec<T>*>(smem + M.off_boxes), M.box_base);
    }
    template <typename Q>
    __device__ __forceinline__ bool a(const Q* row, T* cen) const {
        fk<Q>(row, cen);
        return hot_pairs_collide<T>(M, smem, cen, BT);
    }
    template <typename Q>
    __device__ __forceinline__ bool b(const Q* row, T* cen) const {
        fk<Q>(row, cen);
        return rest_collides<T>(M, smem, cen, BT, margin);
    }
};

}  // namespace ez
