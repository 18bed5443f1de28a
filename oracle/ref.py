"""numpy restatement of the reference hot path — TEST INFRASTRUCTURE ONLY.

Every function cites the reference file:line it restates
(``/root/reference/pkg/src/corridor``).  Inputs are the drop-in package's
plain host data classes (RobotModel, World, HPolytope, ...), which carry the
same fields as the reference's.  Third-party arithmetic: the reference's
voxel test uses ``scipy.spatial.cKDTree`` (scipy 1.18.1 here, unpinned
``>=1.10`` in pkg/pyproject.toml:12); normals use ``scipy.special.ndtri``.
Both are used identically here.
"""

from __future__ import annotations

import math

import numpy as np
from scipy.spatial import cKDTree
from scipy.special import ndtri

# ---------------------------------------------------------------------------
# seeding.py:19-60 — splitmix64 counter streams
# ---------------------------------------------------------------------------
_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
SEED_STEP = 1 << 32


def _mix(z):
    with np.errstate(over="ignore"):
        z = z + _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def hash_words(*words):
    """seeding.py:38-44 hash_u64."""
    h = np.uint64(0)
    for w in words:
        h = _mix(h ^ np.asarray(w).astype(np.uint64, casting="unsafe"))
    return h


def child_seed(master: int, *words) -> int:
    """seeding.py:47-49."""
    return int(hash_words(np.uint64(master & 0xFFFFFFFFFFFFFFFF), *words))


def counter_uniforms(seed, walks, step, slot):
    """seeding.py:52-55."""
    h = hash_words(seed, np.asarray(walks).astype(np.uint64), np.uint64(step) * np.uint64(64) + np.uint64(slot))
    return ((h >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53


def counter_normals(seed, walks, step, slot):
    """seeding.py:58-60."""
    return ndtri(counter_uniforms(seed, walks, step, slot))


# ---------------------------------------------------------------------------
# world.py:64-69, 174-223 — kinematics
# ---------------------------------------------------------------------------
def _skew(a):
    return np.array([[0.0, -a[2], a[1]], [a[2], 0.0, -a[0]], [-a[1], a[0], 0.0]])


def fk_batch(model, Q):
    """Link frames (rots (L, n, d, d), trans (L, n, d)); world.py:195-223 with a batched Rodrigues."""
    Q = np.atleast_2d(np.asarray(Q, dtype=float))
    n, d = Q.shape[0], model.dim
    rots, trans = [], []
    qi = 0
    for joint in model.joints:
        if joint.parent < 0:
            pr = np.broadcast_to(np.eye(d), (n, d, d))
            pt = np.zeros((n, d))
        else:
            pr, pt = rots[joint.parent], trans[joint.parent]
        base_r = pr @ joint.origin.rot
        base_t = pt + np.einsum("bij,j->bi", pr, joint.origin.trans)
        if joint.kind == "fixed":
            rots.append(base_r)
            trans.append(base_t)
            continue
        q = Q[:, qi]
        qi += 1
        if joint.kind == "prismatic":
            rots.append(base_r)
            trans.append(base_t + np.einsum("bij,bj->bi", base_r, q[:, None] * joint.axis[None, :]))
            continue
        if d == 2:
            c, s = np.cos(q), np.sin(q)
            mr = np.empty((n, 2, 2))
            mr[:, 0, 0], mr[:, 0, 1], mr[:, 1, 0], mr[:, 1, 1] = c, -s, s, c
        else:
            a = np.asarray(joint.axis, dtype=float)
            K = _skew(a / np.linalg.norm(a))
            mr = (np.eye(3)[None] + np.sin(q)[:, None, None] * K[None]
                  + (1.0 - np.cos(q))[:, None, None] * (K @ K)[None])
        rots.append(base_r @ mr)
        trans.append(base_t)
    return rots, trans


def geometry_poses(model, Q):
    """world.py:467-475: per-geometry world rotations / translations."""
    rots, trans = fk_batch(model, Q)
    g_rot, g_tr = [], []
    for li, link in enumerate(model.links):
        for g in link.geometries:
            g_rot.append(rots[li] @ g.local_pose.rot)
            g_tr.append(trans[li] + np.einsum("bij,j->bi", rots[li], g.local_pose.trans))
    return g_rot, g_tr


# ---------------------------------------------------------------------------
# world.py:394-565 — collision tests and fp64 clearance
# ---------------------------------------------------------------------------
def _point_box_d2(pts, rot, tr, he):
    """world.py:394-398."""
    local = np.einsum("ji,...j->...i", rot, pts - tr)
    return np.sum((local - np.clip(local, -he, he)) ** 2, axis=-1)


class OracleChecker:
    """Restatement of CollisionChecker (world.py:430-565) for sphere robots.

    ``check_batch`` returns the reference's free mask; ``clearance`` the
    signed fp64 contact distance (min over all tests of distance minus the
    threshold), whose sign reproduces the mask.
    """

    def __init__(self, world, margin: float = 0.0, workers: int = 1):
        self.model = world.model
        self.margin = float(margin)
        self.workers = workers
        self.calls = 0
        self.geoms = self.model.geometries()
        if any(g.kind != "sphere" for g in self.geoms):
            raise NotImplementedError("oracle covers sphere robots")
        d = self.model.dim
        sph = [g for g in world.static if g.kind == "sphere"]
        self.ss_c = np.array([g.local_pose.trans for g in sph], dtype=float).reshape(-1, d)
        self.ss_r = np.array([g.radius for g in sph], dtype=float)
        self.boxes = [g for g in world.static if g.kind == "box"]
        vm = world.vmap
        if vm is not None and vm.n_occupied:
            self.vox_c = vm.centers()
            self.vox_r = vm.sphere_radius
            self.tree = cKDTree(self.vox_c)
        else:
            self.vox_c = np.zeros((0, d))
            self.vox_r = 0.0
            self.tree = None
        self.pairs = np.array(self.model.self_pairs, dtype=np.int64).reshape(-1, 2)

    def _terms(self, Q):
        """Yield (clearance_array) per test family for a chunk."""
        _, tr = geometry_poses(self.model, Q)
        m = self.margin
        out = []
        for gi, g in enumerate(self.geoms):
            c = tr[gi]
            if self.ss_c.shape[0]:
                dist = np.linalg.norm(c[:, None, :] - self.ss_c[None], axis=2)
                out.append(np.min(dist - (self.ss_r[None] + g.radius + m), axis=1))
            if self.tree is not None:
                dnn, _ = self.tree.query(c, k=1, workers=self.workers)
                out.append(dnn - (g.radius + self.vox_r + m))
            for b in self.boxes:
                d2 = _point_box_d2(c, b.local_pose.rot, b.local_pose.trans, b.half_extents)
                out.append(np.sqrt(d2) - (g.radius + m))
        for a, b in self.pairs:
            ga, gb = self.geoms[a], self.geoms[b]
            out.append(np.linalg.norm(tr[a] - tr[b], axis=1) - (ga.radius + gb.radius + m))
        return out

    def clearance(self, Q):
        Q = np.atleast_2d(np.asarray(Q, dtype=float))
        if Q.shape[0] == 0:
            return np.zeros(0)
        terms = self._terms(Q)
        if not terms:
            return np.full(Q.shape[0], np.inf)
        return np.min(np.stack(terms), axis=0)

    def check_batch(self, Q):
        """Free mask with the reference's exact comparisons (world.py:505-565)."""
        Q = np.atleast_2d(np.asarray(Q, dtype=float))
        self.calls += Q.shape[0]
        if Q.shape[0] == 0:
            return np.zeros(0, dtype=bool)
        _, tr = geometry_poses(self.model, Q)
        m = self.margin
        col = np.zeros(Q.shape[0], dtype=bool)
        for gi, g in enumerate(self.geoms):
            c = tr[gi]
            if self.ss_c.shape[0]:
                d2 = (np.sum(c ** 2, axis=1)[:, None] + np.sum(self.ss_c ** 2, axis=1)[None, :]
                      - 2.0 * c @ self.ss_c.T)
                col |= np.any(d2 <= ((self.ss_r + g.radius + m) ** 2)[None, :], axis=1)
            if self.tree is not None:
                dnn, _ = self.tree.query(c, k=1, workers=self.workers)
                col |= dnn <= g.radius + self.vox_r + m
            for b in self.boxes:
                col |= _point_box_d2(c, b.local_pose.rot, b.local_pose.trans, b.half_extents) <= (g.radius + m) ** 2
        for a, b in self.pairs:
            ga, gb = self.geoms[a], self.geoms[b]
            col |= np.sum((tr[a] - tr[b]) ** 2, axis=1) <= (ga.radius + gb.radius + m) ** 2
        return ~col

    def check(self, q):
        return bool(self.check_batch(np.asarray(q, dtype=float)[None, :])[0])


# ---------------------------------------------------------------------------
# cpoly.py:127-173 — hit-and-run
# ---------------------------------------------------------------------------
def chords(A, b, X, D):
    """cpoly.py:127-138."""
    G = X @ A.T
    H = D @ A.T
    slack = b[None, :] - G
    with np.errstate(divide="ignore", invalid="ignore"):
        t = slack / H
    t_hi = np.where(H > 1e-14, t, np.inf).min(axis=1)
    t_lo = np.where(H < -1e-14, t, -np.inf).max(axis=1)
    return t_lo, t_hi


def hit_and_run(A, b, seeds, count, n_ms, seed, walk_offset=0):
    """cpoly.py:141-173 (raises ValueError for the reference's SeedOutside/EmptyChord cases)."""
    d = A.shape[1]
    if count == 0:
        return np.zeros((0, d))
    seeds = np.atleast_2d(np.asarray(seeds, dtype=float))
    if not np.all(np.max(seeds @ A.T - b, axis=1) <= 1e-9):
        raise ValueError("SeedOutside")
    walks = np.uint64(walk_offset) + np.arange(count, dtype=np.uint64)
    X = seeds[np.arange(count) % seeds.shape[0]].copy()
    for step in range(n_ms):
        D = np.stack([counter_normals(seed, walks, step, s) for s in range(d)], axis=1)
        D /= np.linalg.norm(D, axis=1, keepdims=True)
        t_lo, t_hi = chords(A, b, X, D)
        if np.any(t_hi < t_lo - 1e-12):
            raise ValueError("EmptyChord")
        t_lo = np.minimum(t_lo, 0.0)
        t_hi = np.maximum(t_hi, 0.0)
        u = counter_uniforms(seed, walks, step, d)
        X = X + D * (t_lo + u * (t_hi - t_lo))[:, None]
    return X


# ---------------------------------------------------------------------------
# inflation.py:124-325 — EI-ZO
# ---------------------------------------------------------------------------
def project(C, v1, v2):
    """inflation.py:124-137: (proj, alpha, dist)."""
    C = np.atleast_2d(np.asarray(C, dtype=float))
    e = v2 - v1
    ee = float(e @ e)
    if ee == 0.0:
        return np.broadcast_to(v1, C.shape).copy(), np.zeros(C.shape[0]), np.linalg.norm(C - v1, axis=1)
    alpha = np.clip((C - v1) @ e / ee, 0.0, 1.0)
    proj = v1 + alpha[:, None] * e
    return proj, alpha, np.linalg.norm(C - proj, axis=1)


def batch_size(k, delta, eps, tau):
    """inflation.py:156-161."""
    delta_k = 6.0 * delta / (math.pi ** 2 * k ** 2)
    return int(math.ceil(2.0 * math.log(1.0 / delta_k) / (eps * tau ** 2)))


def step_back(a, b_raw, v1, v2, delta_max):
    """inflation.py:203-212."""
    r = max(float(a @ v1), float(a @ v2)) - b_raw + delta_max
    return delta_max - r if r > 0.0 else delta_max


def bisection_steps(A, b, delta_max):
    """inflation.py:219-229."""
    spans = []
    for i in range(A.shape[1]):
        col = A[:, i]
        hi = np.min(np.where(col > 1e-12, b / np.maximum(col, 1e-12), np.inf))
        lo = np.max(np.where(col < -1e-12, b / np.minimum(col, -1e-12), -np.inf))
        spans.append(hi - lo if np.isfinite(hi) and np.isfinite(lo) else 1.0)
    diag = float(np.linalg.norm(spans))
    return max(1, int(math.ceil(math.log2(max(diag, delta_max * 2.0) / delta_max))))


def _normalise_rows(A, b):
    n = np.linalg.norm(A, axis=1)
    off = np.abs(n - 1.0) > 1e-12
    if np.any(off):
        A = A / n[:, None]
        b = b / n
    return A, b


def inflate_edge(v1, v2, A, b, checker, delta=0.05, eps=0.01, tau=0.5, delta_max=0.01, n_p=1000, n_f=10,
                 n_b=None, n_ms=30, t_col=1e-4, n_it=None, seed=0):
    """inflation.py:262-325; returns dict(A, b, iterations, hyperplanes_added, collision_checks, terminated_by)."""
    v1 = np.asarray(v1, dtype=float)
    v2 = np.asarray(v2, dtype=float)
    A = np.array(A, dtype=float)
    b = np.array(b, dtype=float)
    if np.max(A @ v1 - b) >= 0 or np.max(A @ v2 - b) >= 0:
        raise ValueError("SeedOutsideDomain")
    if n_b is None:
        n_b = bisection_steps(A, b, delta_max)
    walk_offset = 0
    k = 1
    hyper = 0
    calls0 = checker.calls
    while True:
        m = batch_size(k, delta, eps, tau)
        n_s = max(n_p, m)
        walks = np.uint64(walk_offset) + np.arange(n_s, dtype=np.uint64)
        alphas = counter_uniforms(seed, walks, SEED_STEP, 0)
        seeds = v1 + np.multiply.outer(alphas, v2 - v1)
        X = hit_and_run(A, b, seeds, n_s, n_ms, seed, walk_offset)
        walk_offset += n_s
        free = checker.check_batch(X)
        n_col_m = int(np.count_nonzero(~free[:m]))
        if n_col_m <= m * (1.0 - tau) * eps:
            term = "test_accepted"
            break
        col = X[np.flatnonzero(~free)[:n_p]]
        proj, _, _ = project(col, v1, v2)
        if not np.all(checker.check_batch(proj)):
            raise ValueError("SegmentInCollision")
        lo, hi = proj.copy(), col.copy()
        for _ in range(n_b):
            mid = 0.5 * (lo + hi)
            fr = checker.check_batch(mid)
            hi = np.where(fr[:, None], hi, mid)
            lo = np.where(fr[:, None], mid, lo)
        star = hi
        _, _, dstar = project(star, v1, v2)
        if np.any(dstar <= t_col):
            raise ValueError("SegmentInCollision")
        order = np.argsort(dstar, kind="stable")
        anchors = star[order]
        pa, _, da = project(anchors, v1, v2)
        alive = np.ones(anchors.shape[0], dtype=bool)
        placed = 0
        while np.any(alive) and placed < n_f:
            i = int(np.argmax(alive))
            if da[i] <= 1e-12:
                raise ValueError("GradientUndefined")
            a = (anchors[i] - pa[i]) / da[i]
            b_raw = float(a @ anchors[i])
            rhs = b_raw - step_back(a, b_raw, v1, v2, delta_max)
            A, b = _normalise_rows(np.vstack([A, a]), np.concatenate([b, [rhs]]))
            placed += 1
            alive &= anchors @ a <= rhs
        hyper += placed
        if n_it is not None and k >= n_it:
            term = "max_iterations"
            break
        k += 1
    return dict(A=A, b=b, iterations=k, hyperplanes_added=hyper, collision_checks=checker.calls - calls0,
                terminated_by=term)


# ---------------------------------------------------------------------------
# world.py:315-328, drm.py:53-71, 170-204, 262-296 — DRM online phase
# ---------------------------------------------------------------------------
def voxelize(points, side, origin):
    """world.py:315-328 -> sorted unique (n, dim) int64 indices."""
    origin = np.asarray(origin, dtype=float)
    pts = np.asarray(points, dtype=float).reshape(-1, origin.shape[0])
    if pts.shape[0] == 0:
        return np.zeros((0, origin.shape[0]), dtype=np.int64)
    idx = np.floor((pts - origin) / side).astype(np.int64)
    return np.unique(idx, axis=0)


def ids_of(extents, idx):
    """drm.py:59-64 (x fastest)."""
    idx = np.atleast_2d(np.asarray(idx, dtype=np.int64))
    vid = np.zeros(idx.shape[0], dtype=np.int64)
    for ax in reversed(range(len(extents))):
        vid = vid * extents[ax] + idx[:, ax]
    return vid


def collision_set(cmap_off, cmap_ids, grid_origin, grid_side, extents, vox_idx, vmap_origin, vmap_side):
    """drm.py:262-296 -> sorted blocked node ids."""
    grid_origin = np.asarray(grid_origin, dtype=float)
    vmap_origin = np.asarray(vmap_origin, dtype=float)
    vox_idx = np.asarray(vox_idx, dtype=np.int64).reshape(-1, grid_origin.shape[0])
    if vox_idx.shape[0] == 0:
        return np.zeros(0, dtype=np.int64)
    same = np.allclose(vmap_origin, grid_origin) and np.isclose(vmap_side, grid_side)
    if same:
        idx = vox_idx
    else:
        lo_c = vox_idx.astype(np.float64) * vmap_side + vmap_origin
        hi_c = lo_c + vmap_side
        lo = np.floor((lo_c - grid_origin) / grid_side + 1e-12).astype(np.int64)
        hi = np.floor((hi_c - grid_origin) / grid_side - 1e-12).astype(np.int64)
        cells = []
        for l, h in zip(lo, hi):
            rng = [np.arange(l[a], h[a] + 1) for a in range(len(extents))]
            mesh = np.meshgrid(*rng, indexing="ij")
            cells.append(np.stack([mm.ravel() for mm in mesh], axis=1))
        idx = np.unique(np.concatenate(cells), axis=0)
    ok = np.all((idx >= 0) & (idx < np.asarray(extents)), axis=1)
    idx = idx[ok]
    if idx.shape[0] == 0:
        return np.zeros(0, dtype=np.int64)
    parts = [cmap_ids[cmap_off[v]:cmap_off[v + 1]] for v in ids_of(extents, idx)]
    return np.unique(np.concatenate(parts).astype(np.int64)) if parts else np.zeros(0, dtype=np.int64)


def node_voxel_pairs(model, nodes, grid_origin, grid_side, extents):
    """drm.py:170-204 for sphere robots: (node, voxel) pairs with d2 <= (r + r_vox)^2."""
    axes = [grid_origin[a] + (np.arange(extents[a]) + 0.5) * grid_side for a in range(len(extents))]
    mesh = np.meshgrid(*axes, indexing="ij")
    centers = np.stack([mm.ravel(order="F") for mm in mesh], axis=1)
    r_vox = 0.5 * grid_side * np.sqrt(len(extents))
    _, tr = geometry_poses(model, nodes)
    rows, cols = [], []
    for gi, g in enumerate(model.geometries()):
        d2 = np.sum((tr[gi][:, None, :] - centers[None, :, :]) ** 2, axis=2)
        bi, vi = np.nonzero(d2 <= (g.radius + r_vox) ** 2)
        rows.append(bi)
        cols.append(vi)
    pairs = np.unique(np.stack([np.concatenate(rows), np.concatenate(cols)], axis=1), axis=0)
    return pairs[:, 0], pairs[:, 1]


def roadmap_adjacency(nodes, ee_pos, k, d_cs, d_ts):
    """drm.py:219-248: k nearest-first edges under the d_cs / d_ts rules, symmetrised CSR."""
    n = nodes.shape[0]
    k_query = min(n, 4 * k + 1)
    dists, idx = cKDTree(nodes).query(nodes, k=k_query)
    rows, cols = [], []
    for i in range(n):
        picked = 0
        for j_pos in range(1, k_query):
            j = int(idx[i, j_pos])
            if dists[i, j_pos] > d_cs:
                break
            if np.linalg.norm(ee_pos[i] - ee_pos[j]) > d_ts:
                continue
            rows.append(i)
            cols.append(j)
            picked += 1
            if picked >= k:
                break
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    und = np.unique(np.stack([np.concatenate([rows, cols]), np.concatenate([cols, rows])], axis=1), axis=0)
    order = np.lexsort((und[:, 1], und[:, 0]))
    r, c = und[order, 0], und[order, 1]
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=off[1:])
    return off, c.astype(np.int32)
