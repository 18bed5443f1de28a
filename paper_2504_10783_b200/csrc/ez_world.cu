// ez_world.cu — world upload, voxel distance-grid build, fused FK + collision
// check kernel and batched FK.  Replaces corridor/world.py:
//   CollisionChecker.__init__   441-463 (ez_world_create)
//   CollisionChecker.check_batch 483-495 (ez_check_batch / ez_check_batch_host)
//   fk_batch                    195-223 (ez_fk_batch)
#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include <cub/device/device_scan.cuh>

#include "ez_check_core.cuh"
#include "ez_rng.cuh"
#include "ez_world.h"

namespace ez {


// ---------------------------------------------------------------------------
// host-side model folding
// ---------------------------------------------------------------------------
namespace {

struct M3 {
    double a[9];
};

M3 mat_eye() {
    M3 m{};
    m.a[0] = m.a[4] = m.a[8] = 1.0;
    return m;
}
M3 mat_mul(const M3& x, const M3& y) {
    M3 r{};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += x.a[3 * i + k] * y.a[3 * k + j];
            r.a[3 * i + j] = s;
        }
    return r;
}
M3 mat_T(const M3& x) {
    M3 r{};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.a[3 * i + j] = x.a[3 * j + i];
    return r;
}
void mat_vec(const M3& m, const double* v, double* out) {
    for (int i = 0; i < 3; ++i) out[i] = m.a[3 * i] * v[0] + m.a[3 * i + 1] * v[1] + m.a[3 * i + 2] * v[2];
}
// rotation/translation of a `dim`-dimensional rigid transform embedded in 3-D
M3 embed_rot(const double* r, int dim) {
    M3 m = mat_eye();
    for (int i = 0; i < dim; ++i)
        for (int j = 0; j < dim; ++j) m.a[3 * i + j] = r[dim * i + j];
    return m;
}
void embed_vec(const double* v, int dim, double* out) {
    out[0] = out[1] = out[2] = 0.0;
    for (int i = 0; i < dim; ++i) out[i] = v[i];
}
// rotation P = [u v a] with P e_z = a (unit), right handed
M3 axis_frame(const double* axis) {
    double a[3] = {axis[0], axis[1], axis[2]};
    const double n = std::sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
    for (double& x : a) x /= n;
    double h[3] = {1.0, 0.0, 0.0};
    if (std::fabs(a[0]) > 0.9) { h[0] = 0.0; h[1] = 1.0; }
    const double d = h[0] * a[0] + h[1] * a[1] + h[2] * a[2];
    double u[3] = {h[0] - d * a[0], h[1] - d * a[1], h[2] - d * a[2]};
    const double un = std::sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
    for (double& x : u) x /= un;
    const double v[3] = {a[1] * u[2] - a[2] * u[1], a[2] * u[0] - a[0] * u[2], a[0] * u[1] - a[1] * u[0]};
    M3 P{};
    for (int i = 0; i < 3; ++i) {
        P.a[3 * i + 0] = u[i];
        P.a[3 * i + 1] = v[i];
        P.a[3 * i + 2] = a[i];
    }
    return P;
}

struct HJoint {
    M3 R;
    double t[3], ax[3];
    int kind, parent, qidx, store_slot = -1, parent_slot = -1, sb = 0, se = 0, bb = 0, be = 0;
};
struct HSphere {
    double p[3], r, rvox, rmar;
};
struct HSelfPair {
    int a, b;
    double thr2;
};
struct HBlock {     // self pairs between two links
    int ba, bb, begin, end;
    double thr2;
};
struct HBox {
    M3 R;
    double t[3], he[3];
    int link;
};
struct HMix {
    int a_kind, a_slot, b_kind, b_slot;
    double ra;
};
struct HModel {
    std::vector<HJoint> joints;
    std::vector<M3> linkQt;
    std::vector<HSphere> spheres;
    std::vector<HSelfPair> all_pairs;
    std::vector<HSelfPair> hot;
    std::vector<HBlock> blocks;
    std::vector<HSelfPair> rest;    // non-hot pairs, block-major
    std::vector<int> pair_src;      // rest position -> index in all_pairs
    std::vector<int32_t> order;     // obstacle-test order of the spheres
    std::vector<double> ssph;  // c3, r
    std::vector<double> sbox;  // Rt9, t3, he3
    std::vector<HBox> boxes;   // robot boxes
    std::vector<HMix> mix;     // self pairs with a box
    double margin = 0.0;
    int dof = 0, n_store = 0;
};

// calibrated hot self pairs tested in phase A.  Measured with the round-2
// specialised kernels (2^20 rows, tools/time_check.py): the 7-DOF model (232
// pairs) is fastest at 4 (11.1e9 checks/s; 16: 10.6e9, 2: 8.0e9), the 14-DOF
// model (1,248 pairs) at 48 (5.13e9; 31: 5.05e9, 96: 3.9e9): 4 below 400
// pairs, else one per 26 pairs in [16, 48].  EZ_HOT_PAIRS overrides.
int hot_pairs(int n_pairs) {
    static const int v = [] {
        const char* e = getenv("EZ_HOT_PAIRS");
        const int x = e ? atoi(e) : -1;
        return (x >= 0 && x <= 256) ? x : -1;
    }();
    if (v >= 0) return v;
    return n_pairs < 400 ? 4 : std::max(16, std::min(48, n_pairs / 26));
}
constexpr int kMinBlock = 3;   // smaller link-pair blocks are tested without the bounding-sphere skip

// Pair/sphere layout.  Without statistics: no hot list, blocks in link order.
// With per-pair and per-sphere hit counts: the hot_pairs(np) most frequent self
// pairs first (flat), the rest in link-pair blocks ordered by hits, spheres
// tested against obstacles in decreasing hit frequency.
void layout_pairs(HModel& hm, const std::vector<uint32_t>* pair_hits, const std::vector<uint32_t>* sph_hits) {
    const int np = static_cast<int>(hm.all_pairs.size());
    auto hits = [&](int i) -> uint64_t { return pair_hits ? (*pair_hits)[i] : 0; };
    std::vector<int> rank(np);
    for (int i = 0; i < np; ++i) rank[i] = i;
    std::vector<char> is_hot(np, 0);
    hm.hot.clear();
    if (pair_hits) {
        std::stable_sort(rank.begin(), rank.end(), [&](int x, int y) { return hits(x) > hits(y); });
        for (int k = 0; k < std::min(hot_pairs(np), np); ++k) {
            if (hits(rank[k]) == 0) break;
            is_hot[rank[k]] = 1;
            hm.hot.push_back(hm.all_pairs[rank[k]]);
        }
    }
    const int ns = static_cast<int>(hm.spheres.size());
    const int nl = static_cast<int>(hm.joints.size());
    std::vector<int> link_of(ns, 0);
    for (int l = 0; l < nl; ++l) {
        for (int s = hm.joints[l].sb; s < hm.joints[l].se; ++s) link_of[s] = l;
    }
    // non-hot pairs by unordered link pair
    std::vector<std::vector<int>> by_key(static_cast<size_t>(nl) * nl);
    for (int i = 0; i < np; ++i) {
        if (is_hot[i]) continue;
        const int la = link_of[hm.all_pairs[i].a], lb = link_of[hm.all_pairs[i].b];
        by_key[static_cast<size_t>(std::min(la, lb)) * nl + std::max(la, lb)].push_back(i);
    }
    std::vector<int> keys;
    std::vector<uint64_t> key_hits(by_key.size(), 0);
    for (size_t k = 0; k < by_key.size(); ++k) {
        if (by_key[k].empty()) continue;
        keys.push_back(static_cast<int>(k));
        for (int i : by_key[k]) key_hits[k] += hits(i);
        std::stable_sort(by_key[k].begin(), by_key[k].end(), [&](int x, int y) { return hits(x) > hits(y); });
    }
    std::stable_sort(keys.begin(), keys.end(), [&](int x, int y) { return key_hits[x] > key_hits[y]; });
    // A link's bound is one of its own spheres (the anchor, chosen to minimise
    // the radius enclosing every sphere of the link around it): no extra FK
    // work or centre storage, at a slightly looser radius than a free centre.
    std::vector<int> anchor(nl, -1);
    std::vector<double> bound_r(nl, 0.0);
    auto bound_of = [&](int l) -> int {
        if (anchor[l] >= 0) return anchor[l];
        const HJoint& j = hm.joints[l];
        auto dist = [&](int s, const double* x) {
            const double dx = hm.spheres[s].p[0] - x[0], dy = hm.spheres[s].p[1] - x[1], dz = hm.spheres[s].p[2] - x[2];
            return std::sqrt(dx * dx + dy * dy + dz * dz);
        };
        double best = 1e300;
        for (int a = j.sb; a < j.se; ++a) {
            double R = 0.0;
            for (int s = j.sb; s < j.se; ++s) R = std::max(R, dist(s, hm.spheres[a].p) + hm.spheres[s].r);
            if (R < best) {
                best = R;
                anchor[l] = a;
            }
        }
        bound_r[l] = best;
        return anchor[l];
    };
    hm.blocks.clear();
    hm.rest.clear();
    hm.pair_src.clear();
    for (int k : keys) {
        const std::vector<int>& ps = by_key[k];
        HBlock b{0, 0, static_cast<int>(hm.rest.size()), 0, 1e30};  // small block: always tested
        if (static_cast<int>(ps.size()) >= kMinBlock) {
            const int la = k / nl, lb = k % nl;
            b.ba = bound_of(la);
            b.bb = bound_of(lb);
            const double Ra = bound_r[la], Rb = bound_r[lb];
            // conservative: fp32 FK error is far below the 1e-4 relative slack
            const double thr = (Ra + Rb + hm.margin) * (1.0 + 1e-4) + 1e-5;
            b.thr2 = thr * thr;
        }
        for (int i : ps) {
            hm.rest.push_back(hm.all_pairs[i]);
            hm.pair_src.push_back(i);
        }
        b.end = static_cast<int>(hm.rest.size());
        hm.blocks.push_back(b);
    }
    hm.order.resize(ns);
    for (int i = 0; i < ns; ++i) hm.order[i] = i;
    if (sph_hits)
        std::stable_sort(hm.order.begin(), hm.order.end(),
                         [&](int x, int y) { return (*sph_hits)[x] > (*sph_hits)[y]; });
}

size_t align16(size_t x) { return (x + 15) & ~static_cast<size_t>(15); }

template <typename T>
std::vector<uint8_t> pack_blob(const HModel& hm, ModelDev<T>& md) {
    const size_t sz_j = align16(hm.joints.size() * sizeof(JointRec<T>));
    const size_t n_sph = hm.spheres.size();
    const size_t sz_s = align16(n_sph * sizeof(SphereRec<T>));
    const size_t sz_h = align16(hm.hot.size() * sizeof(HotRec<T>));
    const size_t sz_g = align16(hm.blocks.size() * sizeof(BlockRec<T>));
    const size_t sz_p = align16(hm.rest.size() * sizeof(HotRec<T>));
    const size_t sz_o = align16(hm.order.size() * sizeof(int32_t));
    const size_t n_ss = hm.ssph.size() / 4, n_sb = hm.sbox.size() / 15;
    const size_t sz_ss = align16(n_ss * sizeof(StaticSphereRec<T>));
    const size_t sz_sb = align16(n_sb * sizeof(StaticBoxRec<T>));
    size_t off = sz_j;
    md.off_spheres = static_cast<uint32_t>(off); off += sz_s;
    md.off_hot = static_cast<uint32_t>(off); off += sz_h;
    md.off_blocks = static_cast<uint32_t>(off); off += sz_g;
    md.off_rest = static_cast<uint32_t>(off); off += sz_p;
    md.off_order = static_cast<uint32_t>(off); off += sz_o;
    md.off_ssph = static_cast<uint32_t>(off); off += sz_ss;
    md.off_sbox = static_cast<uint32_t>(off); off += sz_sb;
    md.off_boxes = static_cast<uint32_t>(off); off += align16(hm.boxes.size() * sizeof(BoxRec<T>));
    md.off_mix = static_cast<uint32_t>(off); off += align16(hm.mix.size() * sizeof(MixPairRec<T>));
    std::vector<uint8_t> blob(std::max<size_t>(16, off), 0);
    md.blob_bytes = static_cast<uint32_t>(blob.size());
    auto* BXR = reinterpret_cast<BoxRec<T>*>(blob.data() + md.off_boxes);
    for (size_t i = 0; i < hm.boxes.size(); ++i) {
        BoxRec<T> r{};
        for (int k = 0; k < 9; ++k) r.R[k] = static_cast<T>(hm.boxes[i].R.a[k]);
        for (int k = 0; k < 3; ++k) {
            r.t[k] = static_cast<T>(hm.boxes[i].t[k]);
            r.he[k] = static_cast<T>(hm.boxes[i].he[k]);
        }
        BXR[i] = r;
    }
    auto* MXR = reinterpret_cast<MixPairRec<T>*>(blob.data() + md.off_mix);
    for (size_t i = 0; i < hm.mix.size(); ++i) {
        MixPairRec<T> r{};
        r.a_kind = hm.mix[i].a_kind;
        r.a_slot = hm.mix[i].a_slot;
        r.b_kind = hm.mix[i].b_kind;
        r.b_slot = hm.mix[i].b_slot;
        r.ra = static_cast<T>(hm.mix[i].ra);
        MXR[i] = r;
    }
    md.n_boxes = static_cast<int32_t>(hm.boxes.size());
    md.n_mix = static_cast<int32_t>(hm.mix.size());
    md.box_base = static_cast<int32_t>(3 * n_sph);
    md.cen_words = static_cast<int32_t>(3 * n_sph + 12 * hm.boxes.size());
    auto put_pairs = [&](const std::vector<HSelfPair>& src, uint32_t off_) {
        auto* HR = reinterpret_cast<HotRec<T>*>(blob.data() + off_);
        for (size_t i = 0; i < src.size(); ++i) {
            HotRec<T> r{};
            r.a = src[i].a;
            r.b = src[i].b;
            r.thr2 = static_cast<T>(src[i].thr2);
            HR[i] = r;
        }
    };
    put_pairs(hm.hot, md.off_hot);
    put_pairs(hm.rest, md.off_rest);
    auto* BK = reinterpret_cast<BlockRec<T>*>(blob.data() + md.off_blocks);
    for (size_t i = 0; i < hm.blocks.size(); ++i) {
        BlockRec<T> r{};
        r.ba = hm.blocks[i].ba;
        r.bb = hm.blocks[i].bb;
        r.begin = hm.blocks[i].begin;
        r.end = hm.blocks[i].end;
        r.thr2 = static_cast<T>(hm.blocks[i].thr2);
        BK[i] = r;
    }
    auto* OR = reinterpret_cast<int32_t*>(blob.data() + md.off_order);
    for (size_t i = 0; i < hm.order.size(); ++i) OR[i] = hm.order[i];
    auto* J = reinterpret_cast<JointRec<T>*>(blob.data());
    for (size_t j = 0; j < hm.joints.size(); ++j) {
        const HJoint& h = hm.joints[j];
        JointRec<T> r{};
        for (int k = 0; k < 9; ++k) r.R[k] = static_cast<T>(h.R.a[k]);
        for (int k = 0; k < 3; ++k) {
            r.t[k] = static_cast<T>(h.t[k]);
            r.ax[k] = static_cast<T>(h.ax[k]);
        }
        r.kind = h.kind;
        r.parent = h.parent;
        r.qidx = h.qidx;
        r.store_slot = h.store_slot;
        r.parent_slot = h.parent_slot;
        r.sph_begin = h.sb;
        r.sph_end = h.se;
        r.box_begin = h.bb;
        r.box_end = h.be;
        J[j] = r;
    }
    auto* S = reinterpret_cast<SphereRec<T>*>(blob.data() + md.off_spheres);
    for (size_t s = 0; s < n_sph; ++s) {
        const HSphere& h = hm.spheres[s];
        SphereRec<T> r{};
        for (int k = 0; k < 3; ++k) r.p[k] = static_cast<T>(h.p[k]);
        r.r = static_cast<T>(h.r);
        r.rvox = static_cast<T>(h.rvox);
        r.rmar = static_cast<T>(h.rmar);
        S[s] = r;
    }
    auto* SS = reinterpret_cast<StaticSphereRec<T>*>(blob.data() + md.off_ssph);
    for (size_t i = 0; i < n_ss; ++i) {
        StaticSphereRec<T> r{};
        for (int k = 0; k < 3; ++k) r.c[k] = static_cast<T>(hm.ssph[4 * i + k]);
        r.r = static_cast<T>(hm.ssph[4 * i + 3]);
        SS[i] = r;
    }
    auto* SB = reinterpret_cast<StaticBoxRec<T>*>(blob.data() + md.off_sbox);
    for (size_t i = 0; i < n_sb; ++i) {
        StaticBoxRec<T> r{};
        for (int k = 0; k < 9; ++k) r.Rt[k] = static_cast<T>(hm.sbox[15 * i + k]);
        for (int k = 0; k < 3; ++k) {
            r.t[k] = static_cast<T>(hm.sbox[15 * i + 9 + k]);
            r.he[k] = static_cast<T>(hm.sbox[15 * i + 12 + k]);
        }
        SB[i] = r;
    }
    md.n_joints = static_cast<int32_t>(hm.joints.size());
    md.dof = hm.dof;
    md.n_spheres = static_cast<int32_t>(hm.spheres.size());
    md.n_hot = static_cast<int32_t>(hm.hot.size());
    md.n_blocks = static_cast<int32_t>(hm.blocks.size());
    md.n_rest = static_cast<int32_t>(hm.rest.size());
    md.n_ssph = static_cast<int32_t>(n_ss);
    md.n_sbox = static_cast<int32_t>(n_sb);
    md.n_store = hm.n_store;
    return blob;
}

}  // namespace

// ---------------------------------------------------------------------------
// voxel distance grid build (fp64, device)
// ---------------------------------------------------------------------------
struct GridBuild {
    int32_t L[3];        // dense lattice dims (padded)
    int32_t lbase[3];    // lattice index of dense cell 0
    int32_t n[3];        // cell dims
    int32_t sub[3];      // cells per voxel side per axis
    double dq, e_max, r_min, r_max, eps;
};

__global__ void k_occ_scatter(const int32_t* __restrict__ idx, int64_t n, int dim, GridBuild gb,
                              uint8_t* __restrict__ occ) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int c[3] = {0, 0, 0};
    for (int k = 0; k < dim; ++k) c[k] = idx[i * dim + k] - gb.lbase[k];
    occ[(static_cast<int64_t>(c[2]) * gb.L[1] + c[1]) * gb.L[0] + c[0]] = 1;
}

// one thread per cell: nearest occupied voxel (from the distance-sorted offset
// table of the cell's sub-position) and, where the filter can be ambiguous,
// the candidate list length.
template <bool kFill>
__global__ void k_cells(GridBuild gb, const uint8_t* __restrict__ occ, const int4* __restrict__ tab,
                        const int32_t* __restrict__ tab_off, uint32_t* __restrict__ cells,
                        uint32_t* __restrict__ counts, int4* __restrict__ lists) {
    const int64_t ncell = static_cast<int64_t>(gb.n[0]) * gb.n[1] * gb.n[2];
    const int64_t ci = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (ci >= ncell) return;
    const int cx = static_cast<int>(ci % gb.n[0]);
    const int cy = static_cast<int>((ci / gb.n[0]) % gb.n[1]);
    const int cz = static_cast<int>(ci / (static_cast<int64_t>(gb.n[0]) * gb.n[1]));
    const int lx = cx / gb.sub[0], ly = cy / gb.sub[1], lz = cz / gb.sub[2];
    const int mx = cx % gb.sub[0], my = cy % gb.sub[1], mz = cz % gb.sub[2];
    const int tsel = (mz * gb.sub[1] + my) * gb.sub[0] + mx;
    const int4* t = tab + tab_off[tsel];
    const int tn = tab_off[tsel + 1] - tab_off[tsel];
    uint32_t q = 255u;
    bool need = false, first = true;
    uint32_t cnt = 0;
    uint32_t out = 0;
    if (kFill) out = cells[ci] & 0x00FFFFFFu;  // list offset from the scan
    for (int k = 0; k < tn; ++k) {
        const int4 e = t[k];
        const int X = lx + e.x, Y = ly + e.y, Z = lz + e.z;
        if (X < 0 || Y < 0 || Z < 0 || X >= gb.L[0] || Y >= gb.L[1] || Z >= gb.L[2]) continue;
        if (!occ[(static_cast<int64_t>(Z) * gb.L[1] + Y) * gb.L[0] + X]) continue;
        const double d = static_cast<double>(__int_as_float(e.w));
        if (first) {
            first = false;
            const double qq = floor(d / gb.dq);
            q = qq >= 255.0 ? 255u : static_cast<uint32_t>(qq);
            const bool always_free = double(q) * gb.dq - gb.e_max > gb.r_max + gb.eps;
            const bool always_hit = q < 255u && (double(q) + 1.0) * gb.dq + gb.e_max <= gb.r_min - gb.eps;
            need = !(always_free || always_hit);
            if (!need) break;
        }
        if (kFill) lists[out + cnt] = make_int4(X + gb.lbase[0], Y + gb.lbase[1], Z + gb.lbase[2], e.w);
        ++cnt;
    }
    if (kFill) {
        if (need) lists[out + cnt] = make_int4(0, 0, 0, __float_as_int(INFINITY));
    } else {
        counts[ci] = need ? cnt + 1 : 0u;
        cells[ci] = q << 24;
    }
}

__global__ void k_pack_bits(const uint8_t* __restrict__ occ, int64_t n, uint32_t* __restrict__ bits) {
    const int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (w * 32 >= n) return;
    uint32_t v = 0;
    for (int b = 0; b < 32; ++b)
        if (w * 32 + b < n && occ[w * 32 + b]) v |= 1u << b;
    bits[w] = v;
}

__global__ void k_cells_merge(int64_t ncell, const uint32_t* __restrict__ offs, uint32_t* __restrict__ cells) {
    const int64_t ci = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (ci < ncell) cells[ci] = (cells[ci] & 0xFF000000u) | (offs[ci] & 0x00FFFFFFu);
}

static int32_t build_voxel_grid(ez_world* w, const ez_scene_desc* sc, const HModel& hm, int dim) {
    const int64_t nv = sc->n_voxels;
    const double s = sc->voxel_side;
    if (!(s > 0.0)) return fail(EZ_INVALID_ARGUMENT, "voxel side must be positive");
    if (hm.spheres.empty() && hm.boxes.empty()) return EZ_OK;  // no geometry can meet a voxel
    const double r_vox = 0.5 * s * std::sqrt(static_cast<double>(dim));
    double r_min = 1e300, r_max = -1e300;
    for (const HSphere& sp : hm.spheres) {
        r_min = std::min(r_min, sp.rvox);
        r_max = std::max(r_max, sp.rvox);
    }
    if (hm.spheres.empty()) r_min = r_max = r_vox + w->margin;  // boxes only: the bitmap is what matters
    int32_t lmin[3] = {0, 0, 0}, lmax[3] = {0, 0, 0};
    for (int k = 0; k < dim; ++k) {
        lmin[k] = INT32_MAX;
        lmax[k] = INT32_MIN;
    }
    for (int64_t i = 0; i < nv; ++i)
        for (int k = 0; k < dim; ++k) {
            lmin[k] = std::min(lmin[k], sc->h_voxel_idx[i * dim + k]);
            lmax[k] = std::max(lmax[k], sc->h_voxel_idx[i * dim + k]);
        }
    double vorg[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < dim; ++k) vorg[k] = sc->voxel_origin[k];
    if (dim == 2) vorg[2] = -0.5 * s;  // planar voxels sit at z = 0

    // cells per voxel side: finest of 4/3/2/1 that keeps the grid under budget
    const char* env = std::getenv("EZ_GRID_SUB");
    int sub_pref = env ? std::max(1, std::atoi(env)) : 2;
    double maxc = 0.0;
    for (int k = 0; k < 3; ++k)
        maxc = std::max({maxc, std::fabs(vorg[k] + (lmin[k] - 8.0) * s), std::fabs(vorg[k] + (lmax[k] + 8.0) * s)});
    const double eps_build = 8.0 * std::ldexp(1.0, -23) * (1.0 + maxc);

    for (int sub = sub_pref; sub >= 1; --sub) {
        const double h = s / sub;
        const double e_max = 0.5 * h * std::sqrt(3.0);
        const double list_r = r_max + e_max + 2.0 * eps_build;
        const int P = static_cast<int>(std::ceil(list_r / s)) + 1;
        GridBuild gb{};
        int64_t ncell = 1;
        for (int k = 0; k < 3; ++k) {
            const bool planar_z = (dim == 2 && k == 2);
            gb.sub[k] = planar_z ? 1 : sub;
            const int pad = planar_z ? 0 : P;
            gb.lbase[k] = lmin[k] - pad;
            gb.L[k] = lmax[k] - lmin[k] + 1 + 2 * pad;
            gb.n[k] = gb.L[k] * gb.sub[k];
            ncell *= gb.n[k];
        }
        if (ncell > (int64_t(1) << 28) && sub > 1) continue;
        if (ncell > (int64_t(1) << 28)) return fail(EZ_CAPACITY, "voxel map extent too large for the distance grid");
        gb.dq = list_r / 255.0;
        gb.e_max = e_max;
        gb.r_min = r_min;
        gb.r_max = r_max;
        gb.eps = eps_build;

        // distance-sorted lattice offsets for each sub-position of a cell centre
        const int K = P;
        std::vector<int4> tab;
        std::vector<int32_t> tab_off(1, 0);
        for (int mz = 0; mz < gb.sub[2]; ++mz)
            for (int my = 0; my < gb.sub[1]; ++my)
                for (int mx = 0; mx < gb.sub[0]; ++mx) {
                    const double dl[3] = {(mx + 0.5) / gb.sub[0] - 0.5, (my + 0.5) / gb.sub[1] - 0.5,
                                          (mz + 0.5) / gb.sub[2] - 0.5};
                    struct E { double d; int x, y, z; };
                    std::vector<E> es;
                    const int kz = (dim == 2) ? 0 : K;
                    for (int z = -kz; z <= kz; ++z)
                        for (int y = -K; y <= K; ++y)
                            for (int x = -K; x <= K; ++x) {
                                const double ddx = (x - dl[0]) * s, ddy = (y - dl[1]) * s, ddz = (z - dl[2]) * s;
                                const double d = std::sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
                                if (d <= list_r) es.push_back({d, x, y, z});
                            }
                    std::sort(es.begin(), es.end(), [](const E& a, const E& b) {
                        if (a.d != b.d) return a.d < b.d;
                        if (a.z != b.z) return a.z < b.z;
                        if (a.y != b.y) return a.y < b.y;
                        return a.x < b.x;
                    });
                    for (const E& e : es) {
                        // round the stored distance down: the query's break test stays exact
                        float fd = static_cast<float>(e.d);
                        if (static_cast<double>(fd) > e.d) fd = std::nextafter(fd, 0.0f);
                        int4 v;
                        v.x = e.x; v.y = e.y; v.z = e.z;
                        std::memcpy(&v.w, &fd, 4);
                        tab.push_back(v);
                    }
                    tab_off.push_back(static_cast<int32_t>(tab.size()));
                }

        const int64_t nl = static_cast<int64_t>(gb.L[0]) * gb.L[1] * gb.L[2];
        uint8_t* d_occ = nullptr;
        int32_t* d_idx = nullptr;
        int4* d_tab = nullptr;
        int32_t* d_tab_off = nullptr;
        uint32_t* d_counts = nullptr;
        uint32_t* d_offs = nullptr;
        void* d_tmp = nullptr;
        size_t tmp_bytes = 0;
        EZ_CUDA(cudaMalloc(&d_occ, nl));
        EZ_CUDA(cudaMemset(d_occ, 0, nl));
        EZ_CUDA(cudaMalloc(&d_idx, sizeof(int32_t) * std::max<int64_t>(1, nv * dim)));
        EZ_CUDA(cudaMemcpy(d_idx, sc->h_voxel_idx, sizeof(int32_t) * nv * dim, cudaMemcpyHostToDevice));
        EZ_CUDA(cudaMalloc(&d_tab, sizeof(int4) * std::max<size_t>(1, tab.size())));
        EZ_CUDA(cudaMemcpy(d_tab, tab.data(), sizeof(int4) * tab.size(), cudaMemcpyHostToDevice));
        EZ_CUDA(cudaMalloc(&d_tab_off, sizeof(int32_t) * tab_off.size()));
        EZ_CUDA(cudaMemcpy(d_tab_off, tab_off.data(), sizeof(int32_t) * tab_off.size(), cudaMemcpyHostToDevice));
        EZ_CUDA(cudaMalloc(&w->d_cells, sizeof(uint32_t) * ncell));
        EZ_CUDA(cudaMalloc(&d_counts, sizeof(uint32_t) * ncell));
        EZ_CUDA(cudaMalloc(&d_offs, sizeof(uint32_t) * ncell));

        k_occ_scatter<<<static_cast<unsigned>((nv + 255) / 256), 256>>>(d_idx, nv, dim, gb, d_occ);
        const unsigned nb = static_cast<unsigned>((ncell + 255) / 256);
        k_cells<false><<<nb, 256>>>(gb, d_occ, d_tab, d_tab_off, w->d_cells, d_counts, nullptr);
        EZ_CUDA(cudaGetLastError());
        EZ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_counts, d_offs, static_cast<int>(ncell)));
        EZ_CUDA(cudaMalloc(&d_tmp, tmp_bytes));
        EZ_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_counts, d_offs, static_cast<int>(ncell)));
        uint32_t last_off = 0, last_cnt = 0;
        EZ_CUDA(cudaMemcpy(&last_off, d_offs + ncell - 1, 4, cudaMemcpyDeviceToHost));
        EZ_CUDA(cudaMemcpy(&last_cnt, d_counts + ncell - 1, 4, cudaMemcpyDeviceToHost));
        const int64_t total = static_cast<int64_t>(last_off) + last_cnt;
        bool too_big = total >= (int64_t(1) << 24);
        if (!too_big) {
            k_cells_merge<<<nb, 256>>>(ncell, d_offs, w->d_cells);
            EZ_CUDA(cudaMalloc(&w->d_lists, sizeof(int4) * std::max<int64_t>(1, total)));
            k_cells<true><<<nb, 256>>>(gb, d_occ, d_tab, d_tab_off, w->d_cells, nullptr, w->d_lists);
            // the occupancy bitmap stays on the device for robot boxes (box vs voxel spheres)
            const int64_t words = (nl + 31) / 32;
            EZ_CUDA(cudaMalloc(&w->d_occ_bits, sizeof(uint32_t) * words));
            k_pack_bits<<<static_cast<unsigned>((words + 255) / 256), 256>>>(d_occ, nl, w->d_occ_bits);
            w->device_bytes += words * 4;
            EZ_CUDA(cudaGetLastError());
            EZ_CUDA(cudaDeviceSynchronize());
        }
        cudaFree(d_occ);
        cudaFree(d_idx);
        cudaFree(d_tab);
        cudaFree(d_tab_off);
        cudaFree(d_counts);
        cudaFree(d_offs);
        cudaFree(d_tmp);
        if (too_big) {
            cudaFree(w->d_cells);
            w->d_cells = nullptr;
            if (sub > 1) continue;
            return fail(EZ_CAPACITY, "voxel candidate lists exceed 2^24 entries");
        }
        w->n_list = total;
        w->cell_h = h;
        for (int k = 0; k < 3; ++k) w->grid_n[k] = gb.n[k];
        w->device_bytes += ncell * 4 + total * 16;

        // kernel-side views
        const double org[3] = {vorg[0] + gb.lbase[0] * s, vorg[1] + gb.lbase[1] * s,
                               dim == 2 ? -0.5 * h : vorg[2] + gb.lbase[2] * s};
        auto fill = [&](auto& V, double eps) {
            using TT = std::remove_reference_t<decltype(V.h)>;
            V.cells = w->d_cells;
            V.lists = w->d_lists;
            for (int k = 0; k < 3; ++k) {
                V.n[k] = gb.n[k];
                V.org[k] = static_cast<TT>(org[k]);
                V.vorg[k] = static_cast<TT>(vorg[k]);
            }
            V.present = 1;
            V.h = static_cast<TT>(h);
            V.inv_h = static_cast<TT>(1.0 / h);
            V.dq = static_cast<TT>(gb.dq);
            V.eps = static_cast<TT>(eps);
            V.vside = static_cast<TT>(s);
            V.rvox = static_cast<TT>(r_vox);
            V.occ = w->d_occ_bits;
            for (int k = 0; k < 3; ++k) {
                V.lbase[k] = gb.lbase[k];
                V.L[k] = gb.L[k];
            }
        };
        fill(w->mf.vox, eps_build);
        fill(w->md.vox, 1e-12 * (1.0 + maxc));
        return EZ_OK;
    }
    return fail(EZ_CAPACITY, "could not size the voxel distance grid");
}

// ---------------------------------------------------------------------------
// kernels: fused check, FK frames
// ---------------------------------------------------------------------------
template <typename T, typename Q, int BT>
__global__ void __launch_bounds__(BT)
k_check(const __grid_constant__ ModelDev<T> M, const Q* __restrict__ q, int64_t n, int64_t ld, uint8_t* __restrict__ out,
        T margin, int64_t count_lim, int32_t* __restrict__ n_col) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ int32_t s_queue[2 * BT];
    __shared__ int s_warp[BT / 32];
    tma_stage(smem, M.blob, M.blob_bytes, &bar);
    T* cen = reinterpret_cast<T*>(smem + M.blob_bytes);
    const size_t roff = (static_cast<size_t>(M.blob_bytes) + static_cast<size_t>(M.cen_words) * BT * sizeof(T) + 15) &
                        ~static_cast<size_t>(15);
    const BlobPolicy<T, BT> pol{M, smem, margin};
    check_tiles<T, Q, BT>(pol, M.dof, cen + threadIdx.x, reinterpret_cast<Q*>(smem + roff), s_queue, s_warp, q, n, ld,
                          out, count_lim, n_col);
}

// link frames (true frames, fp64) for fk_batch / forward_kinematics
__global__ void k_fk_frames(const __grid_constant__ ModelDev<double> M, const double* __restrict__ Qt, const double* __restrict__ q,
                            int64_t n, double* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const JointRec<double>* J = reinterpret_cast<const JointRec<double>*>(M.blob);
    const int dof = M.dof, nj = M.n_joints;
    double R[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, t[3] = {0, 0, 0};
    double* o = out + i * nj * 12;
    for (int j = 0; j < nj; ++j) {
        const JointRec<double> jr = J[j];
        if (jr.parent != j - 1) {
            if (jr.parent < 0) {
                for (int k = 0; k < 9; ++k) R[k] = (k % 4 == 0) ? 1.0 : 0.0;
                t[0] = t[1] = t[2] = 0.0;
            } else {
                // reload the parent's modified frame from the output (true frame * Q)
                const double* pf = out + i * nj * 12 + jr.parent * 12;
                const double* pq = Qt + jr.parent * 9;  // Q^T of parent
                for (int r = 0; r < 3; ++r)
                    for (int c = 0; c < 3; ++c)  // Rg = Rf * Q = Rf * (Q^T)^T
                        R[3 * r + c] = pf[3 * r] * pq[3 * c] + pf[3 * r + 1] * pq[3 * c + 1] + pf[3 * r + 2] * pq[3 * c + 2];
                for (int k = 0; k < 3; ++k) t[k] = pf[9 + k];
            }
        }
        double N[9], tn[3];
        for (int r = 0; r < 3; ++r) {
            for (int c = 0; c < 3; ++c)
                N[3 * r + c] = R[3 * r] * jr.R[c] + R[3 * r + 1] * jr.R[3 + c] + R[3 * r + 2] * jr.R[6 + c];
            tn[r] = t[r] + (R[3 * r] * jr.t[0] + R[3 * r + 1] * jr.t[1] + R[3 * r + 2] * jr.t[2]);
        }
        if (jr.kind == EZ_JOINT_REVOLUTE) {
            double s, c;
            sincos(q[i * dof + jr.qidx], &s, &c);
            for (int r = 0; r < 3; ++r) {
                const double n0 = N[3 * r], n1 = N[3 * r + 1];
                N[3 * r] = n0 * c + n1 * s;
                N[3 * r + 1] = n1 * c - n0 * s;
            }
        } else if (jr.kind == EZ_JOINT_PRISMATIC) {
            const double qq = q[i * dof + jr.qidx];
            for (int r = 0; r < 3; ++r) tn[r] += (N[3 * r] * jr.ax[0] + N[3 * r + 1] * jr.ax[1] + N[3 * r + 2] * jr.ax[2]) * qq;
        }
        for (int k = 0; k < 9; ++k) R[k] = N[k];
        for (int k = 0; k < 3; ++k) t[k] = tn[k];
        const double* Qtj = Qt + j * 9;
        double* f = o + j * 12;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)  // Rf = Rg * Q^T
                f[3 * r + c] = R[3 * r] * Qtj[c] + R[3 * r + 1] * Qtj[3 + c] + R[3 * r + 2] * Qtj[6 + c];
        for (int k = 0; k < 3; ++k) f[9 + k] = t[k];
    }
}

// Hit statistics of every self pair and every sphere-vs-obstacle test over
// uniform samples of the joint box; used only to order the tests.
__global__ void __launch_bounds__(128)
k_calibrate(const __grid_constant__ ModelDev<float> M, const float* __restrict__ lo, const float* __restrict__ hi, int n, uint64_t seed,
            float margin, uint32_t* __restrict__ pcount, uint32_t* __restrict__ sph_hits) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint64_t bar;
    tma_stage(smem, M.blob, M.blob_bytes, &bar);
    float* cen = reinterpret_cast<float*>(smem + M.blob_bytes);
    const size_t roff = (static_cast<size_t>(M.blob_bytes) + static_cast<size_t>(M.cen_words) * blockDim.x * 4 + 15) &
                        ~static_cast<size_t>(15);
    float* q = reinterpret_cast<float*>(smem + roff) + threadIdx.x * M.dof;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int k = 0; k < M.dof; ++k) {
        const Philox4 r = philox_draw(seed, static_cast<uint64_t>(i), static_cast<uint32_t>(k), 0u);
        const float u = (static_cast<float>(r.x >> 8) + 0.5f) * 0x1p-24f;
        q[k] = lo[k] + (hi[k] - lo[k]) * u;
    }
    const JointRec<float>* J = reinterpret_cast<const JointRec<float>*>(smem);
    const SphereRec<float>* S = reinterpret_cast<const SphereRec<float>*>(smem + M.off_spheres);
    float* c = cen + threadIdx.x;
    const int st = blockDim.x;
    fk_sphere_centres<float, float>(J, M.n_joints, S, q, c, st,
                                    reinterpret_cast<const BoxRec<float>*>(smem + M.off_boxes), M.box_base);
    const HotRec<float>* P = reinterpret_cast<const HotRec<float>*>(smem + M.off_rest);
    for (int p = 0; p < M.n_rest; ++p)
        if (pair_hits<float>(P[p], c, st)) atomicAdd(pcount + p, 1u);
    const StaticSphereRec<float>* SS = reinterpret_cast<const StaticSphereRec<float>*>(smem + M.off_ssph);
    const StaticBoxRec<float>* SB = reinterpret_cast<const StaticBoxRec<float>*>(smem + M.off_sbox);
    for (int s = 0; s < M.n_spheres; ++s)
        if (sphere_hits_obstacles<float>(M, S[s], SS, SB, margin, c[3 * s * st], c[(3 * s + 1) * st], c[(3 * s + 2) * st]))
            atomicAdd(sph_hits + s, 1u);
}

static int32_t calibrate_layout(ez_world* w, HModel& hm, const double* lower, const double* upper) {
    const int n = 1 << 15;
    const int dof = hm.dof;
    std::vector<float> lh(2 * dof);
    for (int k = 0; k < dof; ++k) {
        lh[k] = static_cast<float>(lower[k]);
        lh[dof + k] = static_cast<float>(upper[k]);
    }
    const size_t np = std::max<size_t>(1, hm.rest.size()), ns = std::max<size_t>(1, hm.spheres.size());
    float* d_lh = nullptr;
    uint32_t* d_cnt = nullptr;
    EZ_CUDA(cudaMalloc(&d_lh, sizeof(float) * 2 * dof));
    EZ_CUDA(cudaMemcpy(d_lh, lh.data(), sizeof(float) * 2 * dof, cudaMemcpyHostToDevice));
    EZ_CUDA(cudaMalloc(&d_cnt, sizeof(uint32_t) * (np + ns)));
    EZ_CUDA(cudaMemset(d_cnt, 0, sizeof(uint32_t) * (np + ns)));
    size_t smem = 0;
    const int threads = check_block_threads<float>(w, w->mf.blob_bytes, w->mf.cen_words, dof * 4, &smem);
    if (threads == 0) return fail(EZ_CAPACITY, "robot model too large for one checking CTA");
    if (smem > 48 * 1024)
        EZ_TRY(allow_max_dyn_smem(k_calibrate));
    k_calibrate<<<(n + threads - 1) / threads, threads, smem>>>(w->mf, d_lh, d_lh + dof, n, 0x5EEDC0DEull,
                                                                static_cast<float>(w->margin), d_cnt, d_cnt + np);
    EZ_CUDA(cudaGetLastError());
    std::vector<uint32_t> cnt(np + ns);
    EZ_CUDA(cudaMemcpy(cnt.data(), d_cnt, sizeof(uint32_t) * (np + ns), cudaMemcpyDeviceToHost));
    cudaFree(d_lh);
    cudaFree(d_cnt);
    std::vector<uint32_t> pair_hits(hm.all_pairs.size(), 0), sph_hits(hm.spheres.size(), 0);
    for (size_t p = 0; p < hm.pair_src.size(); ++p) pair_hits[hm.pair_src[p]] = cnt[p];
    for (size_t s = 0; s < hm.spheres.size(); ++s) sph_hits[s] = cnt[np + s];
    layout_pairs(hm, &pair_hits, &sph_hits);
    for (int i = 0; i < 2; ++i) {
        std::vector<uint8_t> blob = (i == 0) ? pack_blob<float>(hm, w->mf) : pack_blob<double>(hm, w->md);
        if (i == 0) w->h_blob_f = blob;
        uint8_t* d = nullptr;
        EZ_CUDA(cudaMalloc(&d, blob.size()));
        EZ_CUDA(cudaMemcpy(d, blob.data(), blob.size(), cudaMemcpyHostToDevice));
        cudaFree(w->d_blob[i]);
        w->d_blob[i] = d;
    }
    w->mf.blob = w->d_blob[0];
    w->md.blob = w->d_blob[1];
    w->n_blocks = static_cast<int32_t>(hm.blocks.size());
    w->n_hot = static_cast<int32_t>(hm.hot.size());
    return EZ_OK;
}

// CTA size with the most resident warps per SM.  The per-thread sphere-centre
// store makes shared memory the occupancy limiter and a 256-thread CTA can
// strand a large part of it (160 x 3 CTAs beats 256 x 1 for the 33-sphere
// arm), so every candidate size is an instantiation (constant smem strides)
// and the best is picked once per world from the occupancy calculator.
template <typename T, typename Q, int BT>
static int32_t eval_bt(const ez_world* w, const ModelDev<T>& M, int* best_warps, int* best_t, size_t* best_s,
                       int* best_occ) {
    auto kern = k_check<T, Q, BT>;
    cudaFuncAttributes fa{};
    EZ_CUDA(cudaFuncGetAttributes(&fa, kern));
    const size_t max_dyn = static_cast<size_t>(w->smem_optin) - fa.sharedSizeBytes;
    size_t b = M.blob_bytes + static_cast<size_t>(M.cen_words) * BT * sizeof(T);
    b = (b + 15) & ~static_cast<size_t>(15);
    b += static_cast<size_t>(BT) * M.dof * sizeof(Q);
    b = (b + 15) & ~static_cast<size_t>(15);
    if (b > max_dyn) return EZ_OK;
    EZ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(max_dyn)));
    int occ = 0;
    EZ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, BT, b));
    const int warps = occ * BT / 32;
    if (occ > 0 && warps >= *best_warps) {
        *best_warps = warps;
        *best_t = BT;
        *best_s = b;
        *best_occ = occ;
    }
    return EZ_OK;
}

template <typename T, typename Q, int BT>
static void launch_bt(const ModelDev<T>& M, unsigned grid, size_t smem, cudaStream_t stream, const Q* d_q, int64_t n,
                      int64_t ld, uint8_t* d_free, T margin, int64_t count_lim, int32_t* n_col) {
    k_check<T, Q, BT><<<grid, BT, smem, stream>>>(M, d_q, n, ld, d_free, margin, count_lim, n_col);
}

template <typename T, typename Q>
static int32_t launch_check_t(ez_world* w, const ModelDev<T>& M, const Q* d_q, int64_t n, int64_t ld,
                              uint8_t* d_free, cudaStream_t stream, int64_t count_lim, int32_t* n_col) {
    const int slot = (sizeof(T) == 8 ? 2 : 0) + (sizeof(Q) == 8 ? 1 : 0);
    if (sizeof(T) == 4) {
        // fp32 batches run the model-specialised kernel once ez_world_specialize
        // has published it (never compiled implicitly inside a check call);
        // the snapshot keeps it alive for this launch
        const std::shared_ptr<const JitCheck> jc = std::atomic_load(&w->jit);
        if (jc) return jit_launch(w, *jc, d_q, sizeof(Q) == 8, n, ld, d_free, stream, count_lim, n_col);
    }
    if (w->launch_threads[slot] == 0) {
        std::lock_guard<std::mutex> lk(w->cfg_mu);
        if (w->launch_threads[slot] == 0) {
            int bw = -1, bt = 0, bo = 0;
            size_t bs = 0;
            EZ_TRY((eval_bt<T, Q, 64>(w, M, &bw, &bt, &bs, &bo)));
            EZ_TRY((eval_bt<T, Q, 96>(w, M, &bw, &bt, &bs, &bo)));
            EZ_TRY((eval_bt<T, Q, 128>(w, M, &bw, &bt, &bs, &bo)));
            EZ_TRY((eval_bt<T, Q, 160>(w, M, &bw, &bt, &bs, &bo)));
            EZ_TRY((eval_bt<T, Q, 192>(w, M, &bw, &bt, &bs, &bo)));
            EZ_TRY((eval_bt<T, Q, 256>(w, M, &bw, &bt, &bs, &bo)));
            if (bt == 0) return fail(EZ_CAPACITY, "robot model too large for one checking CTA");
            w->launch_smem[slot] = bs;
            w->launch_occ[slot] = bo;
            std::atomic_thread_fence(std::memory_order_release);
            w->launch_threads[slot] = bt;  // published last: readers check it first
        }
    }
    const int threads = w->launch_threads[slot];
    const size_t smem = w->launch_smem[slot];
    const T margin = static_cast<T>(w->margin);
    const int64_t chunk = int64_t(1) << 30;  // queue entries are int32 row indices
    for (int64_t r0 = 0; r0 < n; r0 += chunk) {
        const int64_t rows = std::min(chunk, n - r0);
        const int64_t tiles = (rows + threads - 1) / threads;
        const unsigned grid =
            static_cast<unsigned>(std::min<int64_t>(tiles, static_cast<int64_t>(w->num_sms) * w->launch_occ[slot]));
        const Q* qp = d_q + r0 * ld;
        uint8_t* op = d_free + r0;
        const int64_t cl = count_lim - r0;
        switch (threads) {
            case 64: launch_bt<T, Q, 64>(M, grid, smem, stream, qp, rows, ld, op, margin, cl, n_col); break;
            case 96: launch_bt<T, Q, 96>(M, grid, smem, stream, qp, rows, ld, op, margin, cl, n_col); break;
            case 128: launch_bt<T, Q, 128>(M, grid, smem, stream, qp, rows, ld, op, margin, cl, n_col); break;
            case 160: launch_bt<T, Q, 160>(M, grid, smem, stream, qp, rows, ld, op, margin, cl, n_col); break;
            case 192: launch_bt<T, Q, 192>(M, grid, smem, stream, qp, rows, ld, op, margin, cl, n_col); break;
            default: launch_bt<T, Q, 256>(M, grid, smem, stream, qp, rows, ld, op, margin, cl, n_col); break;
        }
        EZ_CUDA(cudaGetLastError());
    }
    return EZ_OK;
}

int32_t launch_check(ez_world* w, const void* d_q, int32_t q_dtype, int64_t n, int64_t ld,
                     uint8_t* d_free, int32_t precision, cudaStream_t stream, int64_t count_lim,
                     int32_t* n_col) {
    if (n <= 0) return EZ_OK;
    if (precision == EZ_F64) {
        if (q_dtype == EZ_F64)
            return launch_check_t<double, double>(w, w->md, static_cast<const double*>(d_q), n, ld, d_free, stream, count_lim, n_col);
        return launch_check_t<double, float>(w, w->md, static_cast<const float*>(d_q), n, ld, d_free, stream, count_lim, n_col);
    }
    if (q_dtype == EZ_F64)
        return launch_check_t<float, double>(w, w->mf, static_cast<const double*>(d_q), n, ld, d_free, stream, count_lim, n_col);
    return launch_check_t<float, float>(w, w->mf, static_cast<const float*>(d_q), n, ld, d_free, stream, count_lim, n_col);
}

}  // namespace ez

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
using namespace ez;

static void world_free(ez_world* w) {
    if (!w) return;
    for (int i = 0; i < 2; ++i) cudaFree(w->d_blob[i]);
    for (int i = 0; i < ez_world::kHostLanes; ++i)
        if (w->hstream[i]) cudaStreamDestroy(w->hstream[i]);
    for (int i = 0; i < ez_world::kHostStages; ++i) {
        if (w->stage_done[i]) cudaEventDestroy(w->stage_done[i]);
        cudaFreeHost(w->h_stage_in[i]);
        cudaFreeHost(w->h_stage_out[i]);
        cudaFree(w->d_stage_in[i]);
        cudaFree(w->d_stage_out[i]);
    }
    cudaFree(w->d_cells);
    cudaFree(w->d_lists);
    cudaFree(w->d_occ_bits);
    cudaFree(w->d_linkQt);
    eizo_ws_free(w->eizo);
    delete w;
}

extern "C" int32_t ez_world_create(const ez_robot_desc* rb, const ez_scene_desc* sc, double margin,
                                   int32_t device, ez_world** out) {
    if (!rb || !out) return fail(EZ_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    const int dim = rb->dim;
    if (dim != 2 && dim != 3) return fail(EZ_INVALID_ARGUMENT, "task-space dimension must be 2 or 3");
    if (rb->n_joints < 1 || rb->n_joints > kMaxJoints) return fail(EZ_UNSUPPORTED, "joint count outside [1, 64]");
    if (rb->n_geoms > kMaxSpheres) return fail(EZ_UNSUPPORTED, "more than 1024 robot geometries");
    if (margin < 0.0) return fail(EZ_INVALID_ARGUMENT, "margin must be >= 0");
    EZ_ON_DEVICE(device);
    EZ_TRY(retain_async_pool());

    HModel hm;
    const int nj = rb->n_joints;
    std::vector<M3> Q(nj);
    std::vector<int> needs_store(nj, 0);
    for (int j = 0; j < nj; ++j) {
        const int p = rb->joint_parent[j];
        if (p >= j || p < -1) return fail(EZ_INVALID_ARGUMENT, "joint parent must precede the joint");
        if (p >= 0 && p != j - 1) needs_store[p] = 1;
    }
    int slots = 0;
    std::vector<int> slot_of(nj, -1);
    for (int j = 0; j < nj; ++j)
        if (needs_store[j]) slot_of[j] = slots++;
    if (slots > kMaxStore) return fail(EZ_UNSUPPORTED, "too many branching links");
    hm.n_store = slots;
    int qi = 0;
    for (int j = 0; j < nj; ++j) {
        HJoint h{};
        h.kind = rb->joint_kind[j];
        h.parent = rb->joint_parent[j];
        const M3 Ro = embed_rot(rb->joint_rot + j * dim * dim, dim);
        double to[3], ax[3];
        embed_vec(rb->joint_trans + j * dim, dim, to);
        embed_vec(rb->joint_axis + j * dim, dim, ax);
        const M3 Qpt = h.parent >= 0 ? mat_T(Q[h.parent]) : mat_eye();
        M3 P = mat_eye();
        if (h.kind == EZ_JOINT_REVOLUTE && dim == 3) {
            const double an = std::sqrt(ax[0] * ax[0] + ax[1] * ax[1] + ax[2] * ax[2]);
            if (!(an > 0.0)) return fail(EZ_INVALID_ARGUMENT, "revolute joint needs a nonzero axis");
            P = axis_frame(ax);
        }
        if (h.kind == EZ_JOINT_PRISMATIC) {
            for (int k = 0; k < 3; ++k) h.ax[k] = ax[k];
        } else if (h.kind != EZ_JOINT_REVOLUTE && h.kind != EZ_JOINT_FIXED) {
            return fail(EZ_INVALID_ARGUMENT, "unknown joint kind");
        }
        h.R = mat_mul(mat_mul(Qpt, Ro), P);
        mat_vec(Qpt, to, h.t);
        h.qidx = (h.kind == EZ_JOINT_FIXED) ? -1 : qi++;
        h.store_slot = slot_of[j];
        h.parent_slot = (h.parent >= 0) ? slot_of[h.parent] : -1;
        Q[j] = P;
        hm.joints.push_back(h);
        hm.linkQt.push_back(mat_T(P));
    }
    hm.dof = qi;
    if (hm.dof > 32) return fail(EZ_UNSUPPORTED, "more than 32 degrees of freedom");

    // robot geometry: spheres and boxes, each in link-major order
    const double r_vox = (sc && sc->n_voxels > 0) ? 0.5 * sc->voxel_side * std::sqrt(static_cast<double>(dim)) : 0.0;
    std::vector<int> sphere_of(rb->n_geoms, -1), box_of(rb->n_geoms, -1), geom_link(rb->n_geoms);
    for (int g = 0; g < rb->n_geoms; ++g) {
        const int link = rb->geom_link[g];
        if (link < 0 || link >= nj) return fail(EZ_INVALID_ARGUMENT, "geometry link out of range");
        if (g > 0 && link < rb->geom_link[g - 1]) return fail(EZ_INVALID_ARGUMENT, "geometries must be link-major");
        geom_link[g] = link;
        double tl[3];
        embed_vec(rb->geom_trans + g * dim, dim, tl);
        const M3 Qt = mat_T(Q[link]);
        if (rb->geom_kind[g] == EZ_GEOM_SPHERE) {
            HSphere s{};
            mat_vec(Qt, tl, s.p);
            s.r = rb->geom_radius[g];
            s.rvox = (s.r + r_vox) + margin;
            s.rmar = s.r + margin;
            sphere_of[g] = static_cast<int>(hm.spheres.size());
            hm.spheres.push_back(s);
        } else if (rb->geom_kind[g] == EZ_GEOM_BOX) {
            HBox bx{};
            bx.R = mat_mul(Qt, embed_rot(rb->geom_rot + g * dim * dim, dim));
            mat_vec(Qt, tl, bx.t);
            embed_vec(rb->geom_half + g * dim, dim, bx.he);
            bx.link = link;
            box_of[g] = static_cast<int>(hm.boxes.size());
            hm.boxes.push_back(bx);
        } else {
            return fail(EZ_INVALID_ARGUMENT, "unknown geometry kind");
        }
    }
    for (int j = 0; j < nj; ++j) {
        int sb = 0, bb = 0;
        for (int g = 0; g < rb->n_geoms; ++g) {
            if (geom_link[g] >= j) break;
            sb += sphere_of[g] >= 0;
            bb += box_of[g] >= 0;
        }
        int se = sb, be = bb;
        for (int g = 0; g < rb->n_geoms; ++g) {
            if (geom_link[g] != j) continue;
            se += sphere_of[g] >= 0;
            be += box_of[g] >= 0;
        }
        hm.joints[j].sb = sb;
        hm.joints[j].se = se;
        hm.joints[j].bb = bb;
        hm.joints[j].be = be;
    }
    // self pairs (input order); sphere-sphere pairs go through layout_pairs
    // (grouping, and after calibration the hot list), pairs with a box are
    // tested by the box stage (sphere first for sphere-box)
    for (int p = 0; p < rb->n_pairs; ++p) {
        const int a = rb->pairs[2 * p], b = rb->pairs[2 * p + 1];
        if (a < 0 || b < 0 || a >= rb->n_geoms || b >= rb->n_geoms)
            return fail(EZ_INVALID_ARGUMENT, "self pair index out of range");
        if (rb->geom_link[a] == rb->geom_link[b])
            return fail(EZ_INVALID_ARGUMENT, "self-collision pair on a single link");
        if (sphere_of[a] >= 0 && sphere_of[b] >= 0) {
            const double rr = (rb->geom_radius[a] + rb->geom_radius[b]) + margin;
            hm.all_pairs.push_back(HSelfPair{sphere_of[a], sphere_of[b], rr * rr});
        } else if (sphere_of[a] >= 0 || sphere_of[b] >= 0) {
            const int s = sphere_of[a] >= 0 ? a : b, x = sphere_of[a] >= 0 ? b : a;
            hm.mix.push_back(HMix{0, sphere_of[s], 1, box_of[x], rb->geom_radius[s]});
        } else {
            hm.mix.push_back(HMix{1, box_of[a], 1, box_of[b], 0.0});
        }
    }
    hm.margin = margin;
    layout_pairs(hm, nullptr, nullptr);
    // static obstacles
    for (int i = 0; sc && i < sc->n_static; ++i) {
        double c[3];
        embed_vec(sc->static_trans + i * dim, dim, c);
        if (sc->static_kind[i] == EZ_GEOM_SPHERE) {
            hm.ssph.insert(hm.ssph.end(), {c[0], c[1], c[2], sc->static_radius[i]});
        } else {
            const M3 Rt = mat_T(embed_rot(sc->static_rot + i * dim * dim, dim));
            double he[3];
            embed_vec(sc->static_half + i * dim, dim, he);
            for (int k = 0; k < 9; ++k) hm.sbox.push_back(Rt.a[k]);
            hm.sbox.insert(hm.sbox.end(), {c[0], c[1], c[2], he[0], he[1], he[2]});
        }
    }

    ez_world* w = new ez_world();
    w->device = device;
    cudaDeviceGetAttribute(&w->num_sms, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&w->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    w->dim = dim;
    w->dof = hm.dof;
    w->n_joints = nj;
    w->n_spheres = static_cast<int32_t>(hm.spheres.size());
    w->n_pairs = static_cast<int32_t>(hm.all_pairs.size());
    w->n_blocks = static_cast<int32_t>(hm.blocks.size());
    w->n_ssph = static_cast<int32_t>(hm.ssph.size() / 4);
    w->n_sbox = static_cast<int32_t>(hm.sbox.size() / 15);
    w->n_store = hm.n_store;
    w->margin = margin;
    w->n_voxels = sc ? sc->n_voxels : 0;

    auto upload = [&](const std::vector<uint8_t>& blob, uint8_t** dst) -> int32_t {
        EZ_CUDA(cudaMalloc(dst, blob.size()));
        EZ_CUDA(cudaMemcpy(*dst, blob.data(), blob.size(), cudaMemcpyHostToDevice));
        w->device_bytes += static_cast<int64_t>(blob.size());
        return EZ_OK;
    };
    int32_t st = EZ_OK;
    {
        std::vector<uint8_t> bf = pack_blob<float>(hm, w->mf);
        std::vector<uint8_t> bd = pack_blob<double>(hm, w->md);
        w->h_blob_f = bf;
        st = upload(bf, &w->d_blob[0]);
        if (st == EZ_OK) st = upload(bd, &w->d_blob[1]);
        w->mf.blob = w->d_blob[0];
        w->md.blob = w->d_blob[1];
    }
    if (st == EZ_OK) {
        std::vector<double> qt(9 * nj);
        for (int j = 0; j < nj; ++j)
            for (int k = 0; k < 9; ++k) qt[9 * j + k] = hm.linkQt[j].a[k];
        cudaError_t e = cudaMalloc(&w->d_linkQt, sizeof(double) * qt.size());
        if (e == cudaSuccess) e = cudaMemcpy(w->d_linkQt, qt.data(), sizeof(double) * qt.size(), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) st = cuda_fail(e, "upload link frames", __FILE__, __LINE__);
    }
    w->mf.vox.present = 0;
    w->md.vox.present = 0;
    if (st == EZ_OK && sc && sc->n_voxels > 0) st = build_voxel_grid(w, sc, hm, dim);
    if (st == EZ_OK && rb->joint_lower && rb->joint_upper && hm.dof > 0 && !hm.spheres.empty())
        st = calibrate_layout(w, hm, rb->joint_lower, rb->joint_upper);
    w->q_lo.assign(hm.dof, -3.14159265358979);
    w->q_hi.assign(hm.dof, 3.14159265358979);
    if (rb->joint_lower && rb->joint_upper)
        for (int k = 0; k < hm.dof; ++k) {
            w->q_lo[k] = rb->joint_lower[k];
            w->q_hi[k] = rb->joint_upper[k];
        }
    if (st != EZ_OK) {
        world_free(w);
        return st;
    }
    *out = w;
    return EZ_OK;
}

extern "C" int32_t ez_world_destroy(ez_world* w) {
    if (!w) return EZ_OK;
    ::ez::DeviceGuard dg(w->device);
    world_free(w);
    return EZ_OK;
}

extern "C" int32_t ez_world_get_info(const ez_world* w, ez_world_info* out) {
    if (!w || !out) return fail(EZ_INVALID_ARGUMENT, "null argument");
    out->dof = w->dof;
    out->n_links = w->n_joints;
    out->n_spheres = w->n_spheres;
    out->n_pairs = w->n_pairs;
    out->n_static = w->n_ssph + w->n_sbox;
    out->n_hot_pairs = w->n_hot;
    out->n_voxels = w->n_voxels;
    for (int k = 0; k < 3; ++k) out->grid_dims[k] = w->grid_n[k];
    out->cell_side = w->cell_h;
    out->list_entries = w->n_list;
    out->device_bytes = w->device_bytes;
    {
        std::lock_guard<std::mutex> lk(const_cast<ez_world*>(w)->cfg_mu);  // jit is published under cfg_mu
        const bool on = static_cast<bool>(std::atomic_load(&w->jit));
        out->check_cta = on ? w->jit_bt : 0;
        out->check_variant = on ? w->jit_variant : -1;
    }
    return EZ_OK;
}

extern "C" int32_t ez_check_batch(ez_world* w, const void* d_q, int32_t q_dtype, int64_t n, int64_t ld,
                                  uint8_t* d_free, int32_t precision, void* stream) {
    if (!w) return fail(EZ_INVALID_ARGUMENT, "null world");
    if (n < 0 || ld < w->dof) return fail(EZ_INVALID_ARGUMENT, "bad batch shape");
    if (n == 0) return EZ_OK;
    if (q_dtype != EZ_F32 && q_dtype != EZ_F64) return fail(EZ_INVALID_ARGUMENT, "bad dtype");
    EZ_ON_DEVICE(w->device);
    return launch_check(w, d_q, q_dtype, n, ld, d_free, precision, static_cast<cudaStream_t>(stream));
}

// Host-buffer check.  Rows stay in the caller's element type (fp32 rows cross
// PCIe at 4 B per value).  The batch is cut into chunks dealt round-robin to
// lanes; a lane is a stream with two pinned/device stages.  Per chunk a lane
// waits for the stage's previous use (event), moves the rows into the pinned
// stage (pageable caller buffer) or DMAs them directly (pinned), enqueues the
// H2D copy, the check kernel and the D2H copy of the flags.
//  * pinned rows: one host thread enqueues every lane in chunk order, so the
//    H2D copy of one chunk overlaps the kernel and D2H of the previous ones;
//  * pageable rows: one host thread per lane (ez_util host_parallel).  Lanes
//    never wait on one another, so the host moves of some chunks overlap the
//    DMA and kernels of others (one thread moving pageable rows runs far below
//    the PCIe rate).
// Stage buffers are allocated on first use at the path's chunk size (pinned
// callers never touch the host stages), so small batches hold little memory.
extern "C" int32_t ez_check_batch_host(ez_world* w, const void* h_q, int32_t q_dtype, int64_t n, int64_t ld,
                                       uint8_t* h_free, int32_t precision) {
    if (!w) return fail(EZ_INVALID_ARGUMENT, "null world");
    if (n < 0 || ld < w->dof) return fail(EZ_INVALID_ARGUMENT, "bad batch shape");
    if (q_dtype != EZ_F32 && q_dtype != EZ_F64) return fail(EZ_INVALID_ARGUMENT, "bad dtype");
    if (n == 0) return EZ_OK;
    std::lock_guard<std::mutex> lock(w->mu);
    EZ_ON_DEVICE(w->device);
    const int dof = w->dof;
    const size_t es = q_dtype == EZ_F64 ? sizeof(double) : sizeof(float);
    constexpr int NL = ez_world::kHostLanes;
    auto env_i = [](const char* name, int64_t dflt, int64_t lo, int64_t hi) {
        const char* e = getenv(name);
        const int64_t v = e ? atoll(e) : dflt;
        return std::min(hi, std::max(lo, v));
    };
    static const int64_t chunk_max = env_i("EZ_HOST_CHUNK_MAX", int64_t(1) << 22, 1024, int64_t(1) << 22);
    static const int64_t chunk_pg = std::min(chunk_max, env_i("EZ_HOST_CHUNK", int64_t(1) << 16, 1024, int64_t(1) << 22));
    static const int64_t chunk_pin =
        std::min(chunk_max, env_i("EZ_HOST_CHUNK_PINNED", int64_t(1) << 17, 1024, int64_t(1) << 22));
    static const int lanes_pin = static_cast<int>(env_i("EZ_HOST_LANES_PINNED", 2, 1, NL));
    static const int lanes_pg = static_cast<int>(env_i("EZ_HOST_LANES", 12, 1, NL));
    static const bool wc = !getenv("EZ_HOST_NO_WC");
    cudaPointerAttributes attr{};
    const bool pinned_in = cudaPointerGetAttributes(&attr, h_q) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    cudaGetLastError();
    const bool pinned_out = cudaPointerGetAttributes(&attr, h_free) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    cudaGetLastError();
    const int64_t chunk = std::min<int64_t>(pinned_in ? chunk_pin : chunk_pg, n);
    // stage capacity: a power of two >= 4096 rows, so a run of growing small
    // batches reallocates O(log) times
    int64_t cap = 4096;
    while (cap < chunk) cap <<= 1;
    // Chunk boundaries.  Pageable rows ramp up: chunk c holds min(chunk,
    // (c + 1) chunk / 8) rows, so the lanes' first host copies finish one after
    // another and the first H2D starts after a small copy instead of all lanes
    // finishing full-size copies at once while the DMA engine idles.
    std::vector<int64_t> cstart{0};
    while (cstart.back() < n) {
        const int64_t c = static_cast<int64_t>(cstart.size()) - 1;
        const int64_t sz = pinned_in ? chunk : std::min(chunk, std::max<int64_t>(1024, (c + 1) * (chunk / 8)));
        cstart.push_back(std::min(n, cstart.back() + sz));
    }
    const int64_t nchunks = static_cast<int64_t>(cstart.size()) - 1;
    const int lanes = static_cast<int>(std::min<int64_t>(pinned_in ? lanes_pin : lanes_pg, nchunks));
    for (int i = 0; i < lanes; ++i)
        if (!w->hstream[i]) EZ_CUDA(cudaStreamCreateWithFlags(&w->hstream[i], cudaStreamNonBlocking));
    // Only the buffers this call's path uses are allocated, at (at least) its
    // chunk size; every stage is idle here (each call drains all of its stages).
    for (int i = 0; i < 2 * lanes; ++i) {
        if (!w->stage_done[i]) EZ_CUDA(cudaEventCreateWithFlags(&w->stage_done[i], cudaEventDisableTiming));
        if (w->d_rows[i] < chunk) {
            cudaFree(w->d_stage_in[i]);
            cudaFree(w->d_stage_out[i]);
            w->d_stage_in[i] = w->d_stage_out[i] = nullptr;
            w->d_rows[i] = 0;
            EZ_CUDA(cudaMalloc(&w->d_stage_in[i], sizeof(double) * cap * dof));
            EZ_CUDA(cudaMalloc(reinterpret_cast<void**>(&w->d_stage_out[i]), cap));
            w->d_rows[i] = cap;
        }
        if (!pinned_in && w->h_in_rows[i] < chunk) {
            cudaFreeHost(w->h_stage_in[i]);
            w->h_stage_in[i] = nullptr;
            w->h_in_rows[i] = 0;
            // write-combined: the host only streams rows into it and the DMA
            // engine reads it (no cache snooping, streaming stores)
            EZ_CUDA(cudaHostAlloc(&w->h_stage_in[i], sizeof(double) * cap * dof,
                                  wc ? cudaHostAllocWriteCombined : cudaHostAllocDefault));
            w->h_in_rows[i] = cap;
        }
        if (!pinned_out && w->h_out_rows[i] < chunk) {
            cudaFreeHost(w->h_stage_out[i]);
            w->h_stage_out[i] = nullptr;
            w->h_out_rows[i] = 0;
            EZ_CUDA(cudaMallocHost(reinterpret_cast<void**>(&w->h_stage_out[i]), cap));
            w->h_out_rows[i] = cap;
        }
    }
    const char* q = static_cast<const char*>(h_q);
    static const bool prof = getenv("EZ_HOST_PROFILE") != nullptr;
    const auto tcall = std::chrono::steady_clock::now();
    // pending[stage]: chunk whose flags sit in the stage's pinned output
    std::vector<int64_t> pending(2 * lanes, -1);
    static const bool prof2 = prof && getenv("EZ_HOST_PROFILE")[0] == '2';
    std::atomic<int64_t> t_copy{0}, t_api{0}, t_wait{0};
    auto drain = [&](int st) -> int32_t {
        const auto tw0 = std::chrono::steady_clock::now();
        EZ_CUDA(cudaEventSynchronize(w->stage_done[st]));
        if (prof2) t_wait += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - tw0).count();
        if (pending[st] >= 0) {
            const int64_t pr0 = cstart[pending[st]];
            std::memcpy(h_free + pr0, w->h_stage_out[st], cstart[pending[st] + 1] - pr0);
            pending[st] = -1;
        }
        return EZ_OK;
    };
    auto one_chunk = [&](int64_t c) -> int32_t {
        const int lane = static_cast<int>(c % lanes);
        const int st = 2 * lane + static_cast<int>((c / lanes) & 1);
        cudaStream_t s = w->hstream[lane];
        const int64_t r0 = cstart[c];
        const int64_t rows = cstart[c + 1] - r0;
        const char* src = q + r0 * ld * es;
        const size_t row_bytes = es * dof;
        EZ_TRY(drain(st));  // the stage's previous chunk is done (and its flags delivered)
        if (pinned_in && ld == dof) {
            EZ_CUDA(cudaMemcpyAsync(w->d_stage_in[st], src, row_bytes * rows, cudaMemcpyHostToDevice, s));
        } else if (pinned_in) {
            EZ_CUDA(cudaMemcpy2DAsync(w->d_stage_in[st], row_bytes, src, es * ld, row_bytes, rows,
                                      cudaMemcpyHostToDevice, s));
        } else {
            char* dst = static_cast<char*>(w->h_stage_in[st]);
            const auto tc0 = std::chrono::steady_clock::now();
            if (ld == dof) {
                copy_to_staging(dst, src, row_bytes * rows);
            } else {
                for (int64_t r = 0; r < rows; ++r) std::memcpy(dst + r * row_bytes, src + r * ld * es, row_bytes);
            }
            if (prof2) t_copy += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - tc0).count();
            EZ_CUDA(cudaMemcpyAsync(w->d_stage_in[st], dst, row_bytes * rows, cudaMemcpyHostToDevice, s));
        }
        const auto ta0 = std::chrono::steady_clock::now();
        EZ_TRY(launch_check(w, w->d_stage_in[st], q_dtype, rows, dof, w->d_stage_out[st], precision, s));
        if (pinned_out) {
            EZ_CUDA(cudaMemcpyAsync(h_free + r0, w->d_stage_out[st], rows, cudaMemcpyDeviceToHost, s));
        } else {
            EZ_CUDA(cudaMemcpyAsync(w->h_stage_out[st], w->d_stage_out[st], rows, cudaMemcpyDeviceToHost, s));
            pending[st] = c;
        }
        EZ_CUDA(cudaEventRecord(w->stage_done[st], s));
        if (prof2) t_api += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - ta0).count();
        return EZ_OK;
    };
    int32_t status = EZ_OK;
    if (pinned_in || lanes == 1) {
        for (int64_t c = 0; c < nchunks && status == EZ_OK; ++c) status = one_chunk(c);
        for (int st = 0; st < 2 * lanes && status == EZ_OK; ++st) status = drain(st);
    } else {
        std::atomic<int32_t> first_err{EZ_OK};
        std::mutex err_mu;
        std::string err_msg;
        host_parallel(lanes, 1, [&](int64_t lo, int64_t hi) {
            for (int64_t lane = lo; lane < hi; ++lane) {
                int32_t st = EZ_OK;
                for (int64_t c = lane; c < nchunks && st == EZ_OK; c += lanes) {
                    if (first_err.load(std::memory_order_relaxed) != EZ_OK) return;
                    st = one_chunk(c);
                }
                for (int k = 0; k < 2 && st == EZ_OK; ++k) st = drain(2 * static_cast<int>(lane) + k);
                if (st != EZ_OK) {
                    int32_t expect = EZ_OK;
                    if (first_err.compare_exchange_strong(expect, st)) {
                        std::lock_guard<std::mutex> lk(err_mu);
                        err_msg = ez_last_error();  // thread-local in the worker
                    }
                }
            }
        });
        if (first_err.load() != EZ_OK) status = fail(first_err.load(), err_msg);
    }
    if (status != EZ_OK) {
        for (int i = 0; i < lanes; ++i) cudaStreamSynchronize(w->hstream[i]);
        return status;
    }
    if (prof)
        fprintf(stderr, "ez_check_batch_host n=%lld chunks=%lld lanes=%d pinned=%d: call %.3f ms (summed over lanes: "
                "copy %.3f, kernel+D2H+event calls %.3f, stage waits %.3f ms)\n",
                static_cast<long long>(n), static_cast<long long>(nchunks), lanes, int(pinned_in),
                1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - tcall).count(), t_copy * 1e-6,
                t_api * 1e-6, t_wait * 1e-6);
    return EZ_OK;
}

extern "C" int32_t ez_fk_batch(ez_world* w, const double* d_q, int64_t n, double* d_frames, void* stream) {
    if (!w) return fail(EZ_INVALID_ARGUMENT, "null world");
    if (n <= 0) return EZ_OK;
    EZ_ON_DEVICE(w->device);
    k_fk_frames<<<static_cast<unsigned>((n + 127) / 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(
        w->md, w->d_linkQt, d_q, n, d_frames);
    EZ_CUDA(cudaGetLastError());
    return EZ_OK;
}
