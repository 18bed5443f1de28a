// ez_jit.cu — per-model check kernels compiled at run time.
//
// The generic k_check reads the robot model from the blob it stages in shared
// memory: every joint rotation, sphere offset, pair index and threshold is a
// shared-memory load, every 3x3 product is a full 27-FMA product, and sphere
// centres go through a per-thread shared-memory store.  For one model, all of
// that is known when the world is built.  This file emits the model as
// straight-line CUDA (joint products with zero terms removed and unit terms
// folded, sphere offsets, pair indices and thresholds as literals, centres in
// registers), compiles it with NVRTC for sm_100a and loads it as a CUDA
// library.  The tile loop, the survivor queue and the voxel-grid tests are the
// generic ones (ez_check_core.cuh, ez_device.cuh), embedded into the library
// at build time.  Same arithmetic as the generic path (same expression order;
// joint-matrix entries below 1e-12, i.e. cos(pi/2) rounding residue, are
// dropped), so flags stay exact outside the 1e-5 contact band.
//
// Replaces corridor/world.py:483-565 (check_batch -> _check_chunk ->
// _sphere_vs_obstacles / _pair) for sphere-only robots on the fp32 path.
#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include <nvrtc.h>

#include "ez_device.cuh"
#include "ez_jit.h"
#include "ez_world.h"

#include "ez_jit_headers.inc"

namespace ez {
namespace {

// Batches up to this many rows on the small-CTA kernel run check_rows_full
// (EZ_JIT_FULL_ROWS, 0 = never).
long long full_rows() {
    static const long long v = [] {
        const char* e = getenv("EZ_JIT_FULL_ROWS");
        return e ? atoll(e) : 32768LL;
    }();
    return v;
}

// The next tile's rows are prefetched into shared memory with cp.async
// (check_tiles_reg's s_pf) for up to 8 joints (7-DOF: 78.9 -> 76.7 us per
// 2^20); EZ_JIT_PFSM=0 prefetches into registers.  More joints prefetch
// nothing (14-DOF: 188 us without, 201 us with the 57 KB of staged rows,
// which also shrink the L1 the grid lookups hit).
bool prefetch_sm(int dof) {
    static const bool on = [] {
        const char* e = getenv("EZ_JIT_PFSM");
        return !(e && e[0] == '0');
    }();
    return on && dof <= 8;
}

// ---------------------------------------------------------------------------
// NVRTC, opened at run time (no link-time dependency)
// ---------------------------------------------------------------------------
struct Nvrtc {
    decltype(&nvrtcCreateProgram) create = nullptr;
    decltype(&nvrtcCompileProgram) compile = nullptr;
    decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
    decltype(&nvrtcGetProgramLog) log = nullptr;
    decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
    decltype(&nvrtcGetCUBIN) cubin = nullptr;
    decltype(&nvrtcDestroyProgram) destroy = nullptr;
    decltype(&nvrtcGetErrorString) err = nullptr;
    bool ok = false;
};

const Nvrtc& nvrtc() {
    static Nvrtc n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12",
                               "/usr/local/cuda/lib64/libnvrtc.so"};
        void* h = nullptr;
        for (const char* nm : names)
            if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL)) != nullptr) break;
        if (!h) return;
        n.create = reinterpret_cast<decltype(n.create)>(dlsym(h, "nvrtcCreateProgram"));
        n.compile = reinterpret_cast<decltype(n.compile)>(dlsym(h, "nvrtcCompileProgram"));
        n.log_size = reinterpret_cast<decltype(n.log_size)>(dlsym(h, "nvrtcGetProgramLogSize"));
        n.log = reinterpret_cast<decltype(n.log)>(dlsym(h, "nvrtcGetProgramLog"));
        n.cubin_size = reinterpret_cast<decltype(n.cubin_size)>(dlsym(h, "nvrtcGetCUBINSize"));
        n.cubin = reinterpret_cast<decltype(n.cubin)>(dlsym(h, "nvrtcGetCUBIN"));
        n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(h, "nvrtcDestroyProgram"));
        n.err = reinterpret_cast<decltype(n.err)>(dlsym(h, "nvrtcGetErrorString"));
        n.ok = n.create && n.compile && n.log_size && n.log && n.cubin_size && n.cubin && n.destroy && n.err;
    });
    return n;
}

// Kernel shapes, per row type.  bt 0: one kernel for CTA sizes 64..256 (size
// from blockDim, registers up to 255; small batches such as the EI-ZO loop's
// are latency-bound per thread).  512 x 2 and 1024 x 1 resident CTAs per SM:
// 64 registers and 32 warps per SM; on large batches the extra warps hide the
// grid-cell and FMA-chain latency better than spill-free code at 128
// registers and 16 warps does (measured: 7-DOF +27%, 14-DOF +60%).
struct Shape {
    int bt;    // compile-time CTA size, 0 = run-time 64..256
    int minb;  // resident CTAs per SM requested from ptxas (0: none)
};
constexpr int kShapes = 3;
Shape shape(int i) {
    static const int minb256 = [] {  // EZ_JIT_MINB256: register cap for the 64..256 kernel
        const char* e = getenv("EZ_JIT_MINB256");
        return e ? std::max(0, std::min(8, atoi(e))) : 0;
    }();
    const Shape s[kShapes] = {{0, minb256}, {512, 2}, {1024, 1}};
    return s[i];
}
constexpr int kJitSizes[kJitSizeCount] = {64, 128, 256, 512, 1024};
int shape_of(int bt) { return bt <= 256 ? 0 : (bt == 512 ? 1 : 2); }
std::string kernel_name(char qt, int shp) {
    const int bt = shape(shp).bt;
    return std::string("ez_check_jit_") + qt + std::to_string(bt ? bt : 256);
}

// ---------------------------------------------------------------------------
// source generation
// ---------------------------------------------------------------------------
std::string lit(float v) {  // exact float literal
    if (v == 0.0f) return std::signbit(v) ? "(-0.0f)" : "0.0f";
    char buf[48];
    std::snprintf(buf, sizeof(buf), "(%af)", static_cast<double>(v));
    return buf;
}

// sum_k a_k * c_k in the generic order (a0*c0 + a1*c1 + a2*c2, left to right),
// zero coefficients removed and unit ones folded
std::string dot3(const std::string (&a)[3], const float (&c)[3]) {
    std::string out;
    for (int k = 0; k < 3; ++k) {
        if (c[k] == 0.0f) continue;
        std::string term = (c[k] == 1.0f) ? a[k] : (c[k] == -1.0f ? "(-" + a[k] + ")" : a[k] + " * " + lit(c[k]));
        out = out.empty() ? term : out + " + " + term;
    }
    return out.empty() ? std::string("0.0f") : out;
}

struct Gen {
    const ModelDev<float>& M;
    const uint8_t* blob;
    float margin;
    // voxel-map code: 0 = grid constants as literals and a 32-bit cell index
    // (vox_fetch / vox_decide), 1 = the generic voxel_cell / voxel_decide,
    // 2 = variant 0's lookups streamed with the FK (phase B below).
    // jit_specialize builds them all and keeps the fastest (their flags are
    // equal: every decision is conservative or exact)
    int variant = 0;
    std::ostringstream o;

    const JointRec<float>* J() const { return reinterpret_cast<const JointRec<float>*>(blob); }
    const SphereRec<float>* S() const { return reinterpret_cast<const SphereRec<float>*>(blob + M.off_spheres); }

    static float clean(float v) { return std::fabs(v) < 1e-12f ? 0.0f : v; }

    // obstacle tests moved into phase A (the most frequently hitting spheres;
    // EZ_JIT_A_OBST, for tuning); phase B tests the rest
    int a_obst() const {
        const char* e = getenv("EZ_JIT_A_OBST");
        const int k = e ? atoi(e) : 0;
        return std::max(0, std::min(k, M.n_spheres));
    }

    // joint chain: frame of link j in R{j}_k / t{j}_k, sphere s in c{s}_k
    // after_link(j), if set, is emitted right after link j's sphere centres
    void fk(const std::function<void(int)>& after_link = nullptr) {
        for (int j = 0; j < M.n_joints; ++j) {
            const JointRec<float>& jr = J()[j];
            float jR[9], jt[3];
            for (int k = 0; k < 9; ++k) jR[k] = clean(jr.R[k]);
            for (int k = 0; k < 3; ++k) jt[k] = clean(jr.t[k]);
            o << "    // joint " << j << "\n";
            const int p = jr.parent;
            for (int r = 0; r < 3; ++r) {
                for (int c = 0; c < 3; ++c) {
                    std::string e;
                    if (p < 0) {
                        e = lit(jR[3 * r + c]);
                    } else {
                        const std::string a[3] = {"R" + std::to_string(p) + "_" + std::to_string(3 * r),
                                                  "R" + std::to_string(p) + "_" + std::to_string(3 * r + 1),
                                                  "R" + std::to_string(p) + "_" + std::to_string(3 * r + 2)};
                        const float cc[3] = {jR[c], jR[3 + c], jR[6 + c]};
                        e = dot3(a, cc);
                    }
                    o << "    float R" << j << "_" << 3 * r + c << " = " << e << ";\n";
                }
                std::string e;
                if (p < 0) {
                    e = lit(jt[r]);
                } else {
                    const std::string a[3] = {"R" + std::to_string(p) + "_" + std::to_string(3 * r),
                                              "R" + std::to_string(p) + "_" + std::to_string(3 * r + 1),
                                              "R" + std::to_string(p) + "_" + std::to_string(3 * r + 2)};
                    const float cc[3] = {jt[0], jt[1], jt[2]};
                    const std::string d = dot3(a, cc);
                    e = "t" + std::to_string(p) + "_" + std::to_string(r) + " + (" + d + ")";
                }
                o << "    float t" << j << "_" << r << " = " << e << ";\n";
            }
            if (jr.kind == EZ_JOINT_REVOLUTE) {
                o << "    {\n        float s, c;\n        Angle<float, Q>::sc(row[" << jr.qidx << "], s, c);\n";
                for (int r = 0; r < 3; ++r) {
                    const std::string n0 = "R" + std::to_string(j) + "_" + std::to_string(3 * r);
                    const std::string n1 = "R" + std::to_string(j) + "_" + std::to_string(3 * r + 1);
                    o << "        { const float n0 = " << n0 << ", n1 = " << n1 << "; " << n0 << " = n0 * c + n1 * s; "
                      << n1 << " = n1 * c - n0 * s; }\n";
                }
                o << "    }\n";
            } else if (jr.kind == EZ_JOINT_PRISMATIC) {
                float ax[3];
                for (int k = 0; k < 3; ++k) ax[k] = clean(jr.ax[k]);
                o << "    {\n        const float qq = static_cast<float>(row[" << jr.qidx << "]);\n";
                for (int r = 0; r < 3; ++r) {
                    const std::string a[3] = {"R" + std::to_string(j) + "_" + std::to_string(3 * r),
                                              "R" + std::to_string(j) + "_" + std::to_string(3 * r + 1),
                                              "R" + std::to_string(j) + "_" + std::to_string(3 * r + 2)};
                    o << "        t" << j << "_" << r << " += (" << dot3(a, ax) << ") * qq;\n";
                }
                o << "    }\n";
            }
            for (int s = jr.sph_begin; s < jr.sph_end; ++s) {
                float pp[3];
                for (int k = 0; k < 3; ++k) pp[k] = clean(S()[s].p[k]);
                for (int r = 0; r < 3; ++r) {
                    const std::string a[3] = {"R" + std::to_string(j) + "_" + std::to_string(3 * r),
                                              "R" + std::to_string(j) + "_" + std::to_string(3 * r + 1),
                                              "R" + std::to_string(j) + "_" + std::to_string(3 * r + 2)};
                    o << "    const float c" << s << "_" << r << " = t" << j << "_" << r << " + (" << dot3(a, pp)
                      << ");\n";
                }
            }
            if (after_link) after_link(j);
        }
    }

    std::string d2(int a, int b) const {
        std::ostringstream e;
        e << "sq3(c" << a << "_0 - c" << b << "_0, c" << a << "_1 - c" << b << "_1, c" << a << "_2 - c" << b << "_2)";
        return e.str();
    }

    void hot() {
        const HotRec<float>* H = reinterpret_cast<const HotRec<float>*>(blob + M.off_hot);
        for (int p = 0; p < M.n_hot; ++p)
            o << "    if (" << d2(H[p].a, H[p].b) << " <= " << lit(H[p].thr2) << ") return true;\n";
    }

    void statics(int s) {
        const SphereRec<float>& sp = S()[s];
        const std::string X = "c" + std::to_string(s) + "_0", Y = "c" + std::to_string(s) + "_1",
                          Z = "c" + std::to_string(s) + "_2";
        const StaticSphereRec<float>* SS = reinterpret_cast<const StaticSphereRec<float>*>(blob + M.off_ssph);
        for (int i = 0; i < M.n_ssph; ++i) {
            o << "    { const float rr = (" << lit(SS[i].r) << " + " << lit(sp.r) << ") + " << lit(margin) << "; if (sq3("
              << X << " - " << lit(SS[i].c[0]) << ", " << Y << " - " << lit(SS[i].c[1]) << ", " << Z << " - "
              << lit(SS[i].c[2]) << ") <= rr * rr) return true; }\n";
        }
        const StaticBoxRec<float>* SB = reinterpret_cast<const StaticBoxRec<float>*>(blob + M.off_sbox);
        for (int i = 0; i < M.n_sbox; ++i) {
            const StaticBoxRec<float>& b = SB[i];
            o << "    { const float dx = " << X << " - " << lit(b.t[0]) << ", dy = " << Y << " - " << lit(b.t[1])
              << ", dz = " << Z << " - " << lit(b.t[2]) << "; float d2 = 0.0f;\n";
            for (int r = 0; r < 3; ++r)
                o << "      { const float l = " << lit(b.Rt[3 * r]) << " * dx + " << lit(b.Rt[3 * r + 1]) << " * dy + "
                  << lit(b.Rt[3 * r + 2]) << " * dz; const float cl = fmin(fmax(l, " << lit(-b.he[r]) << "), "
                  << lit(b.he[r]) << "); d2 += (l - cl) * (l - cl); }\n";
            o << "      if (d2 <= " << lit(sp.rmar) << " * " << lit(sp.rmar) << ") return true; }\n";
        }
    }

    // obstacles in calibrated order, cells of kVoxBatch spheres fetched together
    // distance-grid cells fetched together per batch of spheres (EZ_JIT_VOXB)
    // Deferred list walks (EZ_JIT_DEFER=0: walk in place).  An undecided
    // sphere's (cell word, bound, centre, radius) go to a per-thread queue and
    // the out-of-line walks run after every other test.  A call in the middle
    // of the straight-line tests made each fetched cell word live across it,
    // so it was stored to the stack right after its load: the store waited on
    // the load and the batched fetches lost their overlap.
    bool defer() const {
        static const bool on = [] {
            const char* e = getenv("EZ_JIT_DEFER");
            return !(e && e[0] == '0');
        }();
        return on && M.vox.present && variant != 1;
    }
    void walk_queue() {
        if (!defer()) return;
        const int nq = std::max(1, M.n_spheres);
        o << "    uint32_t wq_w[" << nq << "]; float wq_e[" << nq << "], wq_x[" << nq << "], wq_y[" << nq << "], wq_z["
          << nq << "], wq_r[" << nq << "]; int nwq = 0;\n";
    }
    void walk_flush() {
        if (!defer()) return;
        o << "    for (int i = 0; i < nwq; ++i)\n"
             "        if (voxel_walk<float>(M.vox, wq_w[i], wq_e[i], wq_x[i], wq_y[i], wq_z[i], wq_r[i])) return true;\n";
    }

    // full(): cells of this many spheres fetched together (its callers run at
    // >= 128 registers with one row per thread, where the chain of grid-cell
    // round trips is the latency; EZ_JIT_FULL_VOXB)
    static int full_vox_batch() {
        const char* e = getenv("EZ_JIT_FULL_VOXB");
        const int v = e ? atoi(e) : 12;  // 7-DOF region: 8, 12, 16, 33 within noise (12 kept)
        return (v >= 1 && v <= 64) ? v : 12;
    }
    static int vox_batch() {
        const char* e = getenv("EZ_JIT_VOXB");
        const int v = e ? atoi(e) : kVoxBatch;
        return (v >= 1 && v <= 64) ? v : kVoxBatch;
    }

    // float literal of a double bound, rounded toward -inf (down) or +inf (up)
    static std::string lit_dir(double v, bool up) {
        float f = static_cast<float>(v);
        if (up && static_cast<double>(f) < v) f = std::nextafter(f, INFINITY);
        if (!up && static_cast<double>(f) > v) f = std::nextafter(f, -INFINITY);
        return lit(f);
    }

    // Distance-grid lookup of sphere s with the grid's constants as literals:
    // in-grid test, cell index (32-bit: the grid has < 2^28 cells), an upper
    // bound e of the distance from the centre to its cell centre, the cell
    // word.  Any valid cell and bound give the same flag: the decisions below
    // are conservative by the grid's eps and the list walk is exact.
    void vox_fetch(int j, int s) {
        const VoxGrid<float>& V = M.vox;
        const std::string X = "c" + std::to_string(s) + "_0", Y = "c" + std::to_string(s) + "_1",
                          Z = "c" + std::to_string(s) + "_2";
        const std::string c[3] = {X, Y, Z};
        o << "        float e" << j << " = 0.0f; uint32_t w" << j << " = kFarCell;\n        {\n";
        for (int k = 0; k < 3; ++k)
            o << "            const float f" << k << " = (" << c[k] << " - " << lit(V.org[k]) << ") * " << lit(V.inv_h)
              << ";\n";
        o << "            if ((f0 >= 0.0f) & (f1 >= 0.0f) & (f2 >= 0.0f) & (f0 < " << lit(float(V.n[0])) << ") & (f1 < "
          << lit(float(V.n[1])) << ") & (f2 < " << lit(float(V.n[2])) << ")) {\n";
        for (int k = 0; k < 3; ++k) {
            const float ch = static_cast<float>(double(V.org[k]) + 0.5 * double(V.h));
            o << "                const int i" << k << " = static_cast<int>(f" << k << ");\n"
              << "                const float d" << k << " = " << c[k] << " - fmaf(static_cast<float>(i" << k << "), "
              << lit(V.h) << ", " << lit(ch) << ");\n";
        }
        o << "                e" << j << " = jit_dist_ub(d0 * d0 + d1 * d1 + d2 * d2);\n"
          << "                w" << j << " = __ldg(M.vox.cells + (i0 + " << V.n[0] << " * (i1 + " << V.n[1]
          << " * i2)));\n            }\n        }\n";
    }

    void vox_decide(int j, int s) {
        const VoxGrid<float>& V = M.vox;
        const double R = S()[s].rvox;
        // free: q dq - e > R + eps; hit: q < 255 and q dq + dq + e <= R - eps
        const std::string c_free = lit_dir(double(R) + double(V.eps), true);
        const std::string c_hit = lit_dir(double(R) - double(V.eps) - double(V.dq), false);
        o << "        if (w" << j << " != kFarCell) {\n"
          << "            const float qf = static_cast<float>(w" << j << " >> 24);\n"
          << "            if (!(fmaf(qf, " << lit(V.dq) << ", -e" << j << ") > " << c_free << ")) {\n"
          << "                if ((w" << j << " < 0xFF000000u) & (fmaf(qf, " << lit(V.dq) << ", e" << j << ") <= " << c_hit
          << ")) return true;\n"
          ;
        if (defer())
            o << "                wq_w[nwq] = w" << j << "; wq_e[nwq] = e" << j << "; wq_x[nwq] = c" << s << "_0; wq_y[nwq] = c"
              << s << "_1; wq_z[nwq] = c" << s << "_2; wq_r[nwq] = " << lit(S()[s].rvox) << "; ++nwq;\n";
        else
            o << "                if (voxel_walk<float>(M.vox, w" << j << ", e" << j << ", c" << s << "_0, c" << s << "_1, c"
              << s << "_2, " << lit(S()[s].rvox) << ")) return true;\n";
        o << "            }\n        }\n";
    }

    // spheres order[k_begin, k_end): static obstacles, then the voxel map
    // (cells of vox_batch() spheres fetched before any is decided)
    void obstacles(int k_begin, int k_end, int batch = 0) {
        const int vb = batch > 0 ? batch : vox_batch();
        const int32_t* order = reinterpret_cast<const int32_t*>(blob + M.off_order);
        const bool vox = M.vox.present;
        const bool legacy = variant == 1;
        for (int k0 = k_begin; k0 < k_end; k0 += vb) {
            const int nb = std::min(vb, k_end - k0);
            o << "    {\n";
            for (int j = 0; j < nb && vox; ++j) {
                const int s = order[k0 + j];
                if (!legacy) {
                    vox_fetch(j, s);
                    continue;
                }
                o << "        float e" << j << " = 0.0f; uint32_t w" << j << " = kFarCell;\n"
                  << "        { const int64_t cl = voxel_cell<float>(M.vox, c" << s << "_0, c" << s << "_1, c" << s
                  << "_2, e" << j << "); if (cl >= 0) w" << j << " = __ldg(M.vox.cells + cl); }\n";
            }
            for (int j = 0; j < nb; ++j) {
                const int s = order[k0 + j];
                statics(s);
                if (!vox) continue;
                if (!legacy) {
                    vox_decide(j, s);
                    continue;
                }
                o << "        if (w" << j << " != kFarCell && voxel_decide<float>(M.vox, w" << j << ", e" << j << ", c" << s
                  << "_0, c" << s << "_1, c" << s << "_2, " << lit(S()[s].rvox) << ")) return true;\n";
            }
            o << "    }\n";
        }
    }

    void blocks() {
        const BlockRec<float>* B = reinterpret_cast<const BlockRec<float>*>(blob + M.off_blocks);
        const HotRec<float>* P = reinterpret_cast<const HotRec<float>*>(blob + M.off_rest);
        for (int k = 0; k < M.n_blocks; ++k) {
            const BlockRec<float>& bk = B[k];
            const bool always = bk.thr2 >= 1e29f;
            if (!always) o << "    if (!(" << d2(bk.ba, bk.bb) << " > " << lit(bk.thr2) << ")) {\n";
            else o << "    {\n";
            int p = bk.begin;
            for (; p + 4 <= bk.end; p += 4) {
                o << "        if (";
                for (int u = 0; u < 4; ++u)
                    o << (u ? " | " : "") << "(" << d2(P[p + u].a, P[p + u].b) << " <= " << lit(P[p + u].thr2) << ")";
                o << ") return true;\n";
            }
            for (; p < bk.end; ++p)
                o << "        if (" << d2(P[p].a, P[p].b) << " <= " << lit(P[p].thr2) << ") return true;\n";
            o << "    }\n";
        }
    }

    // everything but the kernel entry points (kernel_source adds one)
    std::string source() {
        o << "// generated by ez_jit.cu for one robot model\n"
          << (getenv("EZ_JIT_NOPF") ? "#define EZ_CHECK_NO_PF 1\n" : "")
          << (getenv("EZ_JIT_BISECT_AB") ? "#define EZ_BISECT_AB 1\n" : "")
          << "#include \"ez_check_core.cuh\"\n\nnamespace ez {\n\n"
          << "__device__ __forceinline__ float sq3(float dx, float dy, float dz) { return dx * dx + dy * dy + dz * dz; }\n"
          // an upper bound of sqrt(x): one MUFU.RSQ (ftz; x below 1e-30 bounds by 1e-15), raised by 2^-20
          << "__device__ __forceinline__ float jit_dist_ub(float x) {\n"
             "    float r;\n    asm(\"rsqrt.approx.ftz.f32 %0, %1;\" : \"=f\"(r) : \"f\"(x));\n"
             "    return x > 1e-30f ? x * r * 1.00000095367431640625f : 1e-15f;\n}\n\n"
          << "struct JitPolicy {\n    static constexpr bool kRegRows = true;\n    const ModelDev<float>& M;\n"
          << "    template <typename Q>\n    __device__ __forceinline__ bool a(const Q* row, float*) const {\n";
        if (a_obst() > 0) walk_queue();
        fk();
        hot();
        obstacles(0, a_obst());
        if (a_obst() > 0) walk_flush();
        o << "    return false;\n    }\n"
          << "    template <typename Q>\n    __device__ __forceinline__ bool b(const Q* row, float*) const {\n";
        walk_queue();
        if (variant == 2 && M.vox.present && a_obst() == 0) {
            // variant 2: the obstacle tests stream with the kinematics (a link's
            // spheres are tested as soon as its frame exists, in link order, and
            // their centres die there); the pair blocks then recompute the FK
            // with every centre live.  Trades one FK for fewer live registers
            // during the grid lookups.
            const int32_t* order = reinterpret_cast<const int32_t*>(blob + M.off_order);
            std::vector<int> rank(M.n_spheres);
            for (int k = 0; k < M.n_spheres; ++k) rank[order[k]] = k;
            o << "    {\n";
            fk([&](int j) {
                const JointRec<float>& jr = J()[j];
                std::vector<int> sph;
                for (int t = jr.sph_begin; t < jr.sph_end; ++t) sph.push_back(t);
                // within a link, the calibrated (most-hit-first) order
                std::sort(sph.begin(), sph.end(), [&](int x, int y) { return rank[x] < rank[y]; });
                for (size_t k0 = 0; k0 < sph.size(); k0 += vox_batch()) {
                    const size_t nb = std::min<size_t>(vox_batch(), sph.size() - k0);
                    o << "    {\n";
                    for (size_t u = 0; u < nb; ++u) vox_fetch(static_cast<int>(u), sph[k0 + u]);
                    for (size_t u = 0; u < nb; ++u) {
                        statics(sph[k0 + u]);
                        vox_decide(static_cast<int>(u), sph[k0 + u]);
                    }
                    o << "    }\n";
                }
            });
            o << "    }\n";
            fk();
        } else {
            fk();
            obstacles(a_obst(), M.n_spheres);
        }
        blocks();
        walk_flush();
        o << "    return false;\n    }\n";
        // the whole check with one FK (the bisection's single-thread checks,
        // which run at up to 128 registers: a() then b() computed the FK three
        // times for a free configuration)
        o << "    template <typename Q>\n    __device__ __forceinline__ bool full(const Q* row, float*) const {\n";
        walk_queue();
        fk();
        hot();
        obstacles(0, M.n_spheres, full_vox_batch());
        blocks();
        walk_flush();
        o << "    return false;\n    }\n};\n\n";
        // dynamic shared memory = rows, then the survivor ring of 2 * bt entries
        o << "template <typename Q, int BT>\n__device__ __forceinline__ void jit_body(const ModelDev<float>& M, const Q* q, "
             "int64_t n, int64_t ld, uint8_t* out, int64_t count_lim, int32_t* n_col) {\n"
          << "    extern __shared__ __align__(16) uint8_t smem[];\n"
          << "    __shared__ int s_warp[32];\n"
          << "    const JitPolicy pol{M};\n"
          << "    if (BT == 0 && n <= " << full_rows() << ") {  // small batch: one row per thread, one FK\n"
          << "        check_rows_full<Q>(pol, " << M.dof << ", q, n, ld, out, count_lim, n_col);\n        return;\n    }\n"
          << "    check_tiles_reg<float, Q, BT>(pol, " << M.dof << ", reinterpret_cast<int32_t*>(smem), s_warp, "
          << (prefetch_sm(M.dof) ? "reinterpret_cast<Q*>(smem + 8 * (BT > 0 ? BT : blockDim.x))" : "static_cast<Q*>(nullptr)")
          << ", q, n, ld, out, count_lim, n_col);\n}\n\n"
          << "}  // namespace ez\n\n";
        return o.str();
    }
};

// one NVRTC program per kernel: the model source plus one entry point
std::string kernel_source(const std::string& body, char qt, int shp) {
    const Shape sh = shape(shp);
    const char* qn = qt == 'f' ? "float" : "double";
    std::ostringstream o;
    o << body << "extern \"C\" __global__ void __launch_bounds__(" << (sh.bt ? sh.bt : 256);
    if (sh.minb > 0) o << ", " << sh.minb;
    o << ") " << kernel_name(qt, shp) << "(const __grid_constant__ ez::ModelDev<float> M, const " << qn
      << "* __restrict__ q, int64_t n, int64_t ld, uint8_t* __restrict__ out, float, int64_t count_lim, "
         "int32_t* __restrict__ n_col) {\n    ez::jit_body<"
      << qn << ", " << sh.bt << ">(M, q, n, ld, out, count_lim, n_col);\n}\n";
    return o.str();
}

// the bisection entry point (one program; fp64 rows, fp32 checks).  128
// threads at <= 128 registers: 16 warps per SM (7-DOF: 143 registers
// uncapped, one 256-thread CTA per SM)
constexpr int kBisectThreads = 128;
constexpr int kBisectMinBlocks = 4;
std::string bisect_source(const std::string& body, int dof) {
    std::ostringstream o;
    o << body << "#include \"ez_bisect_core.cuh\"\n\nextern \"C\" __global__ void __launch_bounds__(" << kBisectThreads
      << ", " << kBisectMinBlocks
      << ") ez_bisect_jit(const __grid_constant__ ez::ModelDev<float> M, const double* __restrict__ X, "
         "const int32_t* __restrict__ col, int32_t* __restrict__ rec, const int32_t* __restrict__ n_cand, "
         "const double* __restrict__ seg, double ee, int n_b, double t_col, double* __restrict__ star, "
         "double* __restrict__ pstar, double* __restrict__ dstar, int64_t resident, int forced_l) {\n"
         "    const ez::JitPolicy pol{M};\n    ez::bisect_points<ez::JitPolicy, "
      << dof << ", " << kBisectThreads
      << ">(pol, X, col, rec, n_cand, seg, ee, n_b, t_col, star, pstar, dstar, resident, forced_l);\n}\n";
    return o.str();
}

// ---------------------------------------------------------------------------
// compile + load, cached by source text (same model and margin -> one module)
// ---------------------------------------------------------------------------
// never destroyed: modules stay loaded until the process exits
std::mutex g_mu;
std::map<std::string, std::shared_ptr<JitCheck>>& g_cache = *new std::map<std::string, std::shared_ptr<JitCheck>>();

// the rare list walk stays out of line: inlined at every unrolled sphere test
// it bloats the straight-line kernel
const char* const kNvrtcOpts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "-w",
                                  "-DEZ_VOXEL_WALK_ATTR=__noinline__"};
constexpr int kNvrtcOptCount = 5;

// On-disk cubin cache (an optimisation only: a miss recompiles).  Key: FNV-1a
// of the generated source, the embedded headers and the NVRTC options.
// EZ_JIT_CACHE=0 disables.
std::string cache_path(const std::string& src) {
    const char* off = getenv("EZ_JIT_CACHE");
    if (off && off[0] == '0') return "";
    std::string dir;
    if (const char* d = getenv("EZ_JIT_CACHE_DIR")) dir = d;
    else if (const char* x = getenv("XDG_CACHE_HOME")) dir = std::string(x) + "/corridor_b200";
    else if (const char* h = getenv("HOME")) dir = std::string(h) + "/.cache/corridor_b200";
    else return "";
    uint64_t hsh = 1469598103934665603ull;
    auto mix = [&](const char* p, size_t n) {
        for (size_t i = 0; i < n; ++i) hsh = (hsh ^ static_cast<uint8_t>(p[i])) * 1099511628211ull;
    };
    mix(src.data(), src.size());
    for (int i = 0; i < kJitHeaderCount; ++i) mix(kJitHeaderText[i], strlen(kJitHeaderText[i]));
    for (int i = 0; i < kNvrtcOptCount; ++i) mix(kNvrtcOpts[i], strlen(kNvrtcOpts[i]));
    char name[64];
    std::snprintf(name, sizeof(name), "/jit_%016llx.cubin", static_cast<unsigned long long>(hsh));
    return dir + name;
}

bool read_file(const std::string& path, std::vector<char>* out) {
    FILE* f = path.empty() ? nullptr : fopen(path.c_str(), "rb");
    if (!f) return false;
    fseek(f, 0, SEEK_END);
    const long n = ftell(f);
    fseek(f, 0, SEEK_SET);
    out->resize(n > 0 ? n : 0);
    const bool ok = n > 0 && fread(out->data(), 1, n, f) == static_cast<size_t>(n);
    fclose(f);
    return ok;
}

void write_file(const std::string& path, const std::vector<char>& data) {
    if (path.empty()) return;
    const std::string dir = path.substr(0, path.rfind('/'));
    for (size_t i = 1; i <= dir.size(); ++i)  // mkdir -p
        if (i == dir.size() || dir[i] == '/') mkdir(dir.substr(0, i).c_str(), 0755);
    const std::string tmp = path + ".tmp" + std::to_string(static_cast<long long>(getpid()));
    FILE* f = fopen(tmp.c_str(), "wb");
    if (!f) return;
    const bool ok = fwrite(data.data(), 1, data.size(), f) == data.size();
    fclose(f);
    if (ok) rename(tmp.c_str(), path.c_str());
    else remove(tmp.c_str());
}

int32_t nvrtc_cubin(const std::string& src, std::vector<char>* cubin) {
    const Nvrtc& nv = nvrtc();
    if (!nv.ok) return fail(EZ_UNSUPPORTED, "NVRTC (libnvrtc.so.12) not found; specialised check kernels unavailable");
    nvrtcProgram prog;
    nvrtcResult r = nv.create(&prog, src.c_str(), "ez_check_jit.cu", kJitHeaderCount, kJitHeaderText, kJitHeaderNames);
    if (r != NVRTC_SUCCESS) return fail(EZ_UNSUPPORTED, std::string("nvrtcCreateProgram: ") + nv.err(r));
    r = nv.compile(prog, kNvrtcOptCount, kNvrtcOpts);
    if (r != NVRTC_SUCCESS) {
        size_t n = 0;
        nv.log_size(prog, &n);
        std::string log(n, '\0');
        nv.log(prog, &log[0]);
        nv.destroy(&prog);
        return fail(EZ_UNSUPPORTED, "NVRTC compile of the specialised check kernel failed:\n" + log.substr(0, 4000));
    }
    size_t n = 0;
    nv.cubin_size(prog, &n);
    cubin->resize(n);
    nv.cubin(prog, cubin->data());
    nv.destroy(&prog);
    return EZ_OK;
}

// The six programs compile concurrently (one host thread each; NVRTC is
// thread-safe per program), each cached on disk under its own key.
int32_t compile(const std::string& body, int dof, std::shared_ptr<JitCheck>* out) {
    struct Job {
        std::string src, path, error;
        std::vector<char> cubin;
        int32_t st = EZ_OK;
        bool cached = false;
    };
    constexpr int kJobs = 2 * kShapes + 1;  // check kernels [rows][shape], then the bisection
    Job jobs[kJobs];
    std::vector<std::thread> threads;
    for (int n = 0; n < kJobs; ++n) {
        Job& j = jobs[n];
        j.src = n < 2 * kShapes ? kernel_source(body, n / kShapes ? 'd' : 'f', n % kShapes) : bisect_source(body, dof);
        j.path = cache_path(j.src);
        j.cached = read_file(j.path, &j.cubin);
        if (!j.cached)
            threads.emplace_back([&j] {
                j.st = nvrtc_cubin(j.src, &j.cubin);
                if (j.st != EZ_OK) j.error = ez_last_error();
            });
    }
    for (auto& t : threads) t.join();
    auto jc = std::make_shared<JitCheck>();
    for (int n = 0; n < kJobs; ++n) {
        Job& j = jobs[n];
        if (j.st != EZ_OK) return fail(j.st, j.error);
        const bool bis = n == 2 * kShapes;
        cudaLibrary_t* lib = bis ? &jc->blib : &jc->lib[n / kShapes][n % kShapes];
        bool loaded = cudaLibraryLoadData(lib, j.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) == cudaSuccess;
        if (!loaded && j.cached) {  // a cached cubin that does not load is rebuilt
            cudaGetLastError();
            EZ_TRY(nvrtc_cubin(j.src, &j.cubin));
            j.cached = false;
            loaded = cudaLibraryLoadData(lib, j.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) == cudaSuccess;
        }
        if (!loaded) EZ_CUDA(cudaGetLastError());
        if (!j.cached) write_file(j.path, j.cubin);
        if (bis) {
            EZ_CUDA(cudaLibraryGetKernel(&jc->bk, jc->blib, "ez_bisect_jit"));
            EZ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&jc->b_occ, reinterpret_cast<const void*>(jc->bk),
                                                                  kBisectThreads, 0));
        }
        else EZ_CUDA(cudaLibraryGetKernel(&jc->k[n / kShapes][n % kShapes], *lib, kernel_name(n / kShapes ? 'd' : 'f', n % kShapes).c_str()));
    }
    *out = jc;
    return EZ_OK;
}

}  // namespace

JitCheck::~JitCheck() {
    for (auto& row : lib)
        for (cudaLibrary_t l : row)
            if (l) cudaLibraryUnload(l);
    if (blib) cudaLibraryUnload(blib);
}

std::string jit_source(const ez_world* w, int variant) {
    Gen g{w->mf, w->h_blob_f.data(), static_cast<float>(w->margin), variant, {}};
    return g.source();
}

namespace {

// dynamic shared memory: the survivor ring of 2 * bt entries (rows live in
// registers, check_tiles_reg)
size_t jit_smem(const ez_world* w, int bt, bool q64) {
    // the survivor ring of 2 bt indices, then (prefetch_sm) one row per thread
    return 2 * static_cast<size_t>(bt) * sizeof(int32_t) +
           (prefetch_sm(w->dof) ? static_cast<size_t>(bt) * w->dof * (q64 ? sizeof(double) : sizeof(float)) : 0);
}

// random rows in the joint box for the CTA-size pick
__global__ void k_fill_box(float* q, int64_t n, int dof, const double* lo, const double* hi, uint64_t seed) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n * dof;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint64_t z = seed + static_cast<uint64_t>(i) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const int k = static_cast<int>(i % dof);
        q[i] = static_cast<float>(lo[k] + (hi[k] - lo[k]) * ((z >> 11) * 0x1p-53));
    }
}

int32_t launch_at(ez_world* w, const JitCheck& jc, int bt, const void* d_q, bool q64, int64_t n, int64_t ld,
                  uint8_t* d_free, cudaStream_t stream, int64_t count_lim, int32_t* n_col) {
    int si = 0;
    while (kJitSizes[si] != bt) ++si;
    const cudaKernel_t kern = jc.k[q64 ? 1 : 0][shape_of(bt)];
    const int64_t tiles = (n + bt - 1) / bt;
    const unsigned grid = static_cast<unsigned>(
        std::min<int64_t>(tiles, static_cast<int64_t>(w->num_sms) * w->jit_occ[q64 ? 1 : 0][si]));
    ModelDev<float> M = w->mf;
    float margin = static_cast<float>(w->margin);
    void* args[] = {&M, const_cast<void**>(&d_q), &n, &ld, &d_free, &margin, &count_lim, &n_col};
    EZ_CUDA(cudaLaunchKernel(reinterpret_cast<const void*>(kern), dim3(grid), dim3(bt), args, jit_smem(w, bt, q64),
                             stream));
    return EZ_OK;
}

// CTA size for large batches: time 1024, 512 and 256 threads (each at the
// residency its kernel was compiled for) on random configurations.
int32_t tune_bt(ez_world* w, const JitCheck& jc, float* best_ms) {
    *best_ms = 1e30f;
    const char* e = getenv("EZ_JIT_BT");
    const int forced = (e && (atoi(e) == 256 || atoi(e) == 512 || atoi(e) == 1024) &&
                        w->jit_occ[0][shape_of(atoi(e)) + 2] > 0) ? atoi(e) : 0;
    const int64_t n = int64_t(1) << 20;
    const int dof = w->dof;
    float* d_q = nullptr;
    double* d_box = nullptr;
    uint8_t* d_out = nullptr;
    cudaStream_t s = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int32_t st = EZ_OK;
    auto ck = [&](cudaError_t r) {
        if (r != cudaSuccess && st == EZ_OK) st = cuda_fail(r, "CTA-size pick", __FILE__, __LINE__);
        return st == EZ_OK;
    };
    // rotating batches larger than twice the L2 (as the workloads it is tuned
    // for): on one L2-resident batch the 14-DOF model timed 512 threads
    // faster, on the streamed batches 1024 is (193 vs 214 us per 2^20)
    const int nb = static_cast<int>(std::min<int64_t>(8, (int64_t(256) << 20) / (sizeof(float) * n * dof) + 1));
    auto qb = [&](int r) { return d_q + static_cast<int64_t>(r % nb) * n * dof; };
    if (ck(cudaMalloc(&d_q, sizeof(float) * n * dof * nb)) && ck(cudaMalloc(&d_out, n)) &&
        ck(cudaMalloc(&d_box, sizeof(double) * 2 * dof)) &&
        ck(cudaMemcpy(d_box, w->q_lo.data(), sizeof(double) * dof, cudaMemcpyHostToDevice)) &&
        ck(cudaMemcpy(d_box + dof, w->q_hi.data(), sizeof(double) * dof, cudaMemcpyHostToDevice)) &&
        ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)) && ck(cudaEventCreate(&e0)) &&
        ck(cudaEventCreate(&e1))) {
        k_fill_box<<<1024, 256, 0, s>>>(d_q, n * nb, dof, d_box, d_box + dof, 0x7E57ull);
        // a warm-up of ~30 launches (the GPU idled through the NVRTC compile
        // and its clocks ramp back up), then three interleaved passes, best
        // time per size (with two and no warm-up the 14-DOF model sometimes
        // kept 512 threads: 224 against 193 us per 2^20)
        const int sizes[3] = {1024, 512, 256};
        float best[3] = {1e30f, 1e30f, 1e30f};
        for (int r = 0; r < 30 && st == EZ_OK; ++r)
            if (w->jit_occ[0][shape_of(sizes[r % 3]) + 2] > 0)
                st = launch_at(w, jc, sizes[r % 3], qb(r), false, n, dof, d_out, s, 0, nullptr);
        for (int pass = 0; pass < 3 && st == EZ_OK; ++pass)
            for (int c = 0; c < 3 && st == EZ_OK; ++c) {
                const int bt = sizes[c];
                if (w->jit_occ[0][shape_of(bt) + 2] < 1 || (forced && bt != forced)) continue;
                for (int r = 0; r < 2 && st == EZ_OK; ++r) st = launch_at(w, jc, bt, qb(r), false, n, dof, d_out, s, 0, nullptr);
                if (!ck(cudaEventRecord(e0, s))) break;
                for (int r = 0; r < 2 * nb && st == EZ_OK; ++r)
                    st = launch_at(w, jc, bt, qb(r + 2), false, n, dof, d_out, s, 0, nullptr);
                float ms = 0.f;
                if (!ck(cudaEventRecord(e1, s)) || !ck(cudaEventSynchronize(e1)) || !ck(cudaEventElapsedTime(&ms, e0, e1)))
                    break;
                best[c] = std::min(best[c], ms);
            }
        int pick = -1;
        for (int c = 0; c < 3; ++c)
            if (best[c] < 1e30f && (pick < 0 || best[c] < best[pick])) pick = c;
        if (getenv("EZ_JIT_TUNE_LOG"))
            fprintf(stderr, "tune_bt dof %d: 1024 %.4f 512 %.4f 256 %.4f ms (%d launches)\n", dof, best[0], best[1], best[2],
                    2 * nb);
        if (pick >= 0) {
            w->jit_bt = sizes[pick];
            *best_ms = best[pick];
        }
    }
    cudaFree(d_q);
    cudaFree(d_out);
    cudaFree(d_box);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (s) cudaStreamDestroy(s);
    return st;
}

}  // namespace

int32_t jit_specialize(ez_world* w) {
    std::lock_guard<std::mutex> cfg(w->cfg_mu);  // concurrent callers compile once
    if (std::atomic_load(&w->jit)) return EZ_OK;
    if (w->jit_failed) return fail(EZ_UNSUPPORTED, w->jit_error);
    auto refuse = [&](int32_t st, const std::string& why) {
        w->jit_failed = true;
        w->jit_error = why;
        return fail(st, why);
    };
    if (w->mf.n_boxes > 0 || w->mf.n_mix > 0) return refuse(EZ_UNSUPPORTED, "robot boxes use the generic check kernel");
    if (w->h_blob_f.empty()) return refuse(EZ_UNSUPPORTED, "no host copy of the model");
    // EZ_JIT_VOX=0/1 forces one voxel-code variant (Gen::variant); otherwise
    // both are built and timed, and the faster one is kept (measured: the
    // literal-constant code wins for the 7-DOF model, the generic calls for
    // the 14-DOF one, where the longer code spills more at 64 registers)
    const char* ev = getenv("EZ_JIT_VOX");
    const int forced = (ev && ev[0] >= '0' && ev[0] <= '2') ? ev[0] - '0' : -1;
    const int v_lo = forced >= 0 ? forced : 0, v_hi = forced >= 0 ? forced : (w->mf.vox.present ? 2 : 0);
    int max_smem = 0;
    EZ_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, w->device));
    std::shared_ptr<JitCheck> best;
    float best_ms = 1e30f;
    int best_bt = 0, best_var = -1;
    int32_t best_occ[2][kJitSizeCount] = {};
    for (int variant = v_lo; variant <= v_hi; ++variant) {
        const std::string src = jit_source(w, variant);
        if (const char* dump = getenv("EZ_JIT_DUMP")) {  // inspection: write the generated source
            if (FILE* f = fopen((std::string(dump) + (variant ? ".v" + std::to_string(variant) : std::string())).c_str(), "w")) {
                fwrite(src.data(), 1, src.size(), f);
                fclose(f);
            }
        }
        std::shared_ptr<JitCheck> jc;
        {
            std::lock_guard<std::mutex> lk(g_mu);
            auto it = g_cache.find(src);
            if (it != g_cache.end()) jc = it->second;
        }
        if (!jc) {
            const int32_t st = compile(src, w->dof, &jc);
            if (st != EZ_OK) {
                w->jit_failed = true;
                w->jit_error = ez_last_error();
                return st;
            }
            std::lock_guard<std::mutex> lk(g_mu);
            g_cache.emplace(src, jc);
        }
        // a size whose rows do not fit in shared memory (many joints, fp64 rows,
        // 1024 threads) keeps occupancy 0 and is never launched
        for (int i = 0; i < 2; ++i)
            for (int si = 0; si < kJitSizeCount; ++si) {
                const int bt = kJitSizes[si];
                const size_t smem = jit_smem(w, bt, i == 1);
                w->jit_occ[i][si] = 0;
                if (smem > static_cast<size_t>(max_smem)) continue;
                const void* k = reinterpret_cast<const void*>(jc->k[i][shape_of(bt)]);
                if (bt == 256 || bt == 512 || bt == 1024)
                    EZ_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
                int occ = 0;
                EZ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, bt, smem));
                w->jit_occ[i][si] = occ;
            }
        if (w->jit_occ[0][0] < 1 || w->jit_occ[1][0] < 1) continue;
        float ms = 1e30f;
        EZ_TRY(tune_bt(w, *jc, &ms));
        if (!best || ms < best_ms) {
            best = jc;
            best_ms = ms;
            best_bt = w->jit_bt;
            best_var = variant;
            std::memcpy(best_occ, w->jit_occ, sizeof(best_occ));
        }
    }
    if (!best) return refuse(EZ_CAPACITY, "specialised check kernel does not fit on an SM");
    // tuned before it is published: a launch that sees the kernel (atomic
    // snapshot in launch_check_t) also sees its CTA size and occupancies
    std::memcpy(w->jit_occ, best_occ, sizeof(best_occ));
    w->jit_bt = best_bt;
    w->jit_variant = best_var;
    std::atomic_store(&w->jit, std::shared_ptr<const JitCheck>(best));
    return EZ_OK;
}

// Large batches run at the tuned CTA size; a batch too small to give every
// SM a CTA at that size (host-path chunks, the EI-ZO loop's 1e4-row batches)
// drops to the largest size that does, down to 64 threads.
int32_t jit_launch(ez_world* w, const JitCheck& jc, const void* d_q, bool q64, int64_t n, int64_t ld, uint8_t* d_free,
                   cudaStream_t stream, int64_t count_lim, int32_t* n_col) {
    // the survivor queue holds int32 row indices: launches of at most 2^30 rows
    const int64_t kMaxRows = int64_t(1) << 30;
    if (n > kMaxRows) {
        const size_t es = q64 ? sizeof(double) : sizeof(float);
        for (int64_t r0 = 0; r0 < n; r0 += kMaxRows)
            EZ_TRY(jit_launch(w, jc, static_cast<const char*>(d_q) + r0 * ld * es, q64, std::min(kMaxRows, n - r0), ld,
                              d_free + r0, stream, count_lim - r0, n_col));
        return EZ_OK;
    }
    int bt = 64;
    for (int si = kJitSizeCount - 1; si >= 0; --si) {
        const int cand = kJitSizes[si];
        if (cand > w->jit_bt || w->jit_occ[q64 ? 1 : 0][si] < 1) continue;
        if ((n + cand - 1) / cand >= static_cast<int64_t>(w->num_sms)) {
            bt = cand;
            break;
        }
    }
    return launch_at(w, jc, bt, d_q, q64, n, ld, d_free, stream, count_lim, n_col);
}

// EZ_BISECT_LEVELS=1..4 (read per call) forces the binary steps per round;
// otherwise the kernel picks from the device-side candidate count.
int32_t jit_bisect_launch(ez_world* w, const JitCheck& jc, const double* X, const int32_t* col, int32_t* rec,
                          const int32_t* n_cand, int n_p, const double* seg, double ee, int n_b, double t_col,
                          double* star, double* pstar, double* dstar, cudaStream_t stream) {
    if (n_p <= 0) return EZ_OK;
    int forced_l = 0;
    if (const char* e = getenv("EZ_BISECT_LEVELS"))
        if (e[0] >= '1' && e[0] <= '4') forced_l = e[0] - '0';
    int64_t resident = static_cast<int64_t>(w->num_sms) * std::max(jc.b_occ, 1) * kBisectThreads;
    ModelDev<float> M = w->mf;
    void* args[] = {&M, const_cast<double**>(&X), const_cast<int32_t**>(&col), &rec, const_cast<int32_t**>(&n_cand),
                    const_cast<double**>(&seg), &ee, &n_b, &t_col, &star, &pstar, &dstar, &resident, &forced_l};
    const int64_t threads = static_cast<int64_t>(n_p) << 4;  // up to 16 threads per candidate
    EZ_CUDA(cudaLaunchKernel(reinterpret_cast<const void*>(jc.bk),
                             dim3(static_cast<unsigned>((threads + kBisectThreads - 1) / kBisectThreads)),
                             dim3(kBisectThreads), args, 0, stream));
    return EZ_OK;
}

}  // namespace ez

extern "C" int32_t ez_world_specialize(ez_world* w, int32_t mode) {
    if (!w) return ez::fail(EZ_INVALID_ARGUMENT, "null world");
    std::lock_guard<std::mutex> lock(w->mu);
    EZ_ON_DEVICE(w->device);
    if (mode < 0) {
        std::lock_guard<std::mutex> cfg(w->cfg_mu);
        std::atomic_store(&w->jit, std::shared_ptr<const ez::JitCheck>());
        w->jit_failed = true;
        w->jit_error = "specialised check kernel disabled for this world";
        return EZ_OK;
    }
    if (mode > 0) return ez::jit_specialize(w);
    if (std::atomic_load(&w->jit)) return EZ_OK;
    return ez::fail(EZ_UNSUPPORTED, w->jit_failed ? w->jit_error : std::string("not specialised"));
}
