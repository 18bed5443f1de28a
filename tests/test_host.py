"""Host-side API semantics (no GPU): polytopes, parameters, primitives, file formats, grids."""

import numpy as np
import pytest

from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.eizo import (InflationParams, Segment, bisection_update, compute_step_back, default_bisection_steps,
                                        dist_gradient, dist_to_segment, project_to_segment, required_batch_size,
                                        unadaptive_test)
from paper_2504_10783_b200.errors import DimensionMismatch, GradientUndefined
from paper_2504_10783_b200.model import REVOLUTE, SPHERE, Geometry, Joint, Link, RigidTransform, RobotModel
from paper_2504_10783_b200.polytope import HPolytope, dumps_polytopes, loads_polytopes
from paper_2504_10783_b200.roadmap import Drm, Grid, load_drm, save_drm
from paper_2504_10783_b200.scene import (VoxelMap, World, load_point_cloud, load_scene, save_point_cloud,
                                         save_scene)

SEG_X = Segment(np.array([0.0, 0.0]), np.array([2.0, 0.0]))


def unit_box(d=2):
    return HPolytope.from_bounds(np.zeros(d), np.ones(d))


def test_polytope_membership_and_normalisation():
    box = HPolytope.from_bounds([-1, -1], [1, 1])
    assert box.contains([0.0, 0.0]) and not box.contains([2.0, 0.0]) and box.contains([1.0, 0.0])
    with pytest.raises(DimensionMismatch):
        box.contains([0.0, 0.0, 0.0])
    p = HPolytope(np.array([[2.0, 0.0]]), np.array([4.0]))
    assert np.allclose(np.linalg.norm(p.A, axis=1), 1.0) and np.isclose(p.b[0], 2.0)
    assert unit_box().contains_segment([0.1, 0.1], [0.9, 0.9])
    assert not unit_box().contains_segment([0.1, 0.1], [1.5, 0.5])
    with pytest.raises(AttributeError):
        box.A = None


def test_intersection_and_json_and_prune():
    box = unit_box()
    cut = box.intersect_halfspace(np.array([1.0, 0.0]), 0.5)
    assert cut.n_faces == 5
    X = np.random.default_rng(0).uniform(-0.5, 1.5, size=(2000, 2))
    assert np.all(~cut.contains_many(X) | box.contains_many(X))
    p3 = unit_box(3).intersect_halfspace(np.array([1.0, 1.0, 0.0]) / np.sqrt(2), 1.2)
    q = HPolytope.from_json(p3.to_json())
    assert np.allclose(q.A, p3.A) and np.allclose(q.b, p3.b)
    assert len(loads_polytopes(dumps_polytopes([p3, box]))) == 2
    assert box.intersect_halfspace(np.array([1.0, 0.0]), 3.0).pruned().n_faces == 4


def test_projection_gradient_primitives():
    proj, a, d = project_to_segment(np.array([1.0, 1.0]), SEG_X)
    assert np.allclose(proj, [1, 0]) and a == 0.5 and d == 1.0
    proj, a, d = project_to_segment(np.array([-3.0, 4.0]), SEG_X)
    assert np.allclose(proj, [0, 0]) and a == 0.0 and d == 5.0
    proj, a, d = project_to_segment(np.array([5.0, 0.0]), Segment(np.zeros(2), np.zeros(2)))
    assert np.allclose(proj, 0) and d == 5.0
    assert np.allclose(dist_gradient(np.array([1.0, 1.0]), SEG_X), [0, 1])
    with pytest.raises(GradientUndefined):
        dist_gradient(np.array([1.0, 0.0]), SEG_X)
    rng = np.random.default_rng(0)
    for _ in range(200):
        seg = Segment(rng.normal(size=3), rng.normal(size=3))
        x1, x2 = rng.normal(size=(2, 3)) * 3
        lam = rng.uniform()
        assert dist_to_segment(lam * x1 + (1 - lam) * x2, seg) <= (
            lam * dist_to_segment(x1, seg) + (1 - lam) * dist_to_segment(x2, seg) + 1e-9)


def test_batch_size_and_test():
    import mpmath

    mpmath.mp.dps = 50
    params = InflationParams(delta=0.05, eps=0.01, tau=0.5)
    for k in (1, 2, 3, 10):
        dk = 6 * mpmath.mpf("0.05") / (mpmath.pi ** 2 * k ** 2)
        assert required_batch_size(k, params) == int(mpmath.ceil(2 * mpmath.log(1 / dk) / mpmath.mpf("0.0025")))
    assert required_batch_size(1, params) == 2795
    assert unadaptive_test(0, 1, InflationParams())[0]
    assert not unadaptive_test(required_batch_size(3, params), 3, params)[0]


class _CountingChecker:
    """Duck-typed checker over a numpy predicate, counting the configurations it is asked about."""

    def __init__(self, free_fn):
        self.free_fn, self.calls = free_fn, 0

    def check_batch(self, Q):
        Q = np.atleast_2d(Q)
        self.calls += len(Q)
        return self.free_fn(Q)


def test_bisection_known_answers():
    """Reference test_inflation.py:116-135: convergence bound, retention, one check per step."""
    seg = Segment(np.array([0.0, 0.0]), np.array([0.0, 1.0]))
    half = _CountingChecker(lambda Q: Q[:, 0] < 2.0)
    star = bisection_update(np.array([4.0, 0.0]), seg, 20, half)
    assert np.linalg.norm(star - [2.0, 0.0]) <= 2 * 4 / 2 ** 20
    assert half.calls == 20
    c = np.array([3.0, 0.0])
    only_c = _CountingChecker(lambda Q: ~np.all(np.isclose(Q, c), axis=1))
    assert np.array_equal(bisection_update(c.copy(), seg, 8, only_c), c)
    one = _CountingChecker(lambda Q: Q[:, 0] < 2.0)
    bisection_update(np.array([4.0, 0.0]), seg, 1, one)
    assert one.calls == 1


def test_step_back_identity_and_default_nb():
    seg = Segment(np.array([0.0, 0.0]), np.array([1.0, 0.0]))
    assert compute_step_back(np.array([0.0, 1.0]), 5.0, seg, 0.01) == 0.01
    assert np.isclose(compute_step_back(np.array([0.0, 1.0]), 0.005, seg, 0.01), 0.005, atol=1e-15)
    rng = np.random.default_rng(70)
    worst = -np.inf
    for _ in range(2000):
        d = int(rng.integers(2, 6))
        a = rng.normal(size=d)
        a /= np.linalg.norm(a)
        s = Segment(rng.normal(size=d) * 5, rng.normal(size=d) * 5)
        c = rng.normal(size=d) * 5
        dm = rng.uniform(1e-4, 1.0)
        rhs = float(a @ c) - compute_step_back(a, float(a @ c), s, dm)
        worst = max(worst, float(a @ s.v1 - rhs), float(a @ s.v2 - rhs))
    assert worst <= 1e-12
    dom = HPolytope.from_bounds([-5, -5], [5, 5])
    assert default_bisection_steps(dom, 0.01) == int(np.ceil(np.log2(np.sqrt(200) / 0.01)))


def test_params_validation():
    with pytest.raises(ValueError):
        InflationParams(delta=0.0)
    with pytest.raises(ValueError):
        InflationParams(t_col=0.02, delta_max=0.01)
    with pytest.raises(ValueError):
        InflationParams(n_f=0)
    p = InflationParams.from_dict({"delta": 0.1, "eps": 0.02, "n_p": 500, "junk": 1})
    assert p.delta == 0.1 and p.n_p == 500 and InflationParams.from_dict(p.to_dict()) == p


def test_self_pair_same_link_rejected():
    """Reference test_world.py:114-119."""
    joints = (Joint(REVOLUTE, -1, RigidTransform.identity(2)),)
    links = (Link((Geometry(SPHERE, RigidTransform.identity(2), radius=0.1),
                   Geometry(SPHERE, RigidTransform.planar(0.5, 0.0), radius=0.1))),)
    with pytest.raises(ValueError):
        RobotModel(2, joints, links, [-1.0], [1.0], self_pairs=((0, 1),))


def test_scene_json_roundtrip(tmp_path):
    for w in (fx.arm3_world(), fx.franka7_world(False), fx.disc_world(fx.forest_centers(5))):
        p = tmp_path / "s.json"
        save_scene(p, w)
        l2 = load_scene(p)
        assert l2.model.dof == w.model.dof and len(l2.static) == len(w.static)
        assert l2.model.self_pairs == w.model.self_pairs
        for ja, jb in zip(w.model.joints, l2.model.joints):
            assert np.allclose(ja.origin.rot, jb.origin.rot) and np.allclose(ja.origin.trans, jb.origin.trans)


def test_point_cloud_io(tmp_path):
    pts = np.random.default_rng(3).normal(size=(257, 3))
    p = tmp_path / "c.pcb"
    save_point_cloud(p, pts, binary=True)
    assert np.array_equal(load_point_cloud(p), pts.astype(np.float32).astype(np.float64))
    raw = p.read_bytes()
    assert raw[:4] == b"PCB1" and int.from_bytes(raw[4:12], "little") == 257 and len(raw) == 16 + 257 * 12
    t = tmp_path / "c.xyz"
    save_point_cloud(t, pts[:2])
    assert np.allclose(load_point_cloud(t), pts[:2])


def test_voxel_map_views():
    vm = VoxelMap(np.zeros(2), 0.5, {(2, 0), (0, 0), (0, 1)})
    assert vm.index_array().tolist() == [[0, 0], [0, 1], [2, 0]]
    assert np.allclose(vm.centers()[0], [0.25, 0.25]) and np.isclose(vm.sphere_radius, 0.5 * 0.5 * np.sqrt(2))
    vm2 = VoxelMap(np.zeros(2), 0.5, np.array([[2, 0], [0, 0], [2, 0]]))
    assert vm2.occupied == frozenset({(2, 0), (0, 0)})


def test_grid_and_drm_io(tmp_path):
    g = Grid(np.array([-1.0, -2.0, 0.0]), 0.5, (3, 4, 5))
    assert g.voxel_id((1, 2, 3)) == 1 + 3 * (2 + 4 * 3)
    assert np.array_equal(g.ids_of([[1, 2, 3], [0, 0, 0]]), [g.voxel_id((1, 2, 3)), 0])
    assert np.array_equal(g.in_bounds([[0, 0, 0], [3, 0, 0], [-1, 0, 0]]), [True, False, False])
    c = g.all_centers()
    assert np.allclose(c[g.voxel_id((1, 2, 3))], g.origin + (np.array([1, 2, 3]) + 0.5) * 0.5)
    rng = np.random.default_rng(0)
    n = 10
    off = np.zeros(g.n_voxels + 1, np.int64)
    off[1:] = np.cumsum(rng.integers(0, 3, size=g.n_voxels))
    ids = rng.integers(0, n, size=off[-1]).astype(np.int32)
    drm = Drm(rng.normal(size=(n, 7)), np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), off, ids,
              rng.normal(size=(n, 7)), g)
    p = tmp_path / "r.drm"
    save_drm(drm, p)
    d2 = load_drm(p)
    assert np.array_equal(d2.nodes, drm.nodes) and np.array_equal(d2.cmap_ids, ids)
    assert np.array_equal(d2.cmap_offsets, off) and d2.grid.extents == g.extents
