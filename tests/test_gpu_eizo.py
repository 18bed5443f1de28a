"""GPU EI-ZO (ez_inflate_edge) against the reference's own inflations and test_inflation.py contracts."""

import numpy as np
import pytest

from conftest import golden, inflate_index
from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge
from paper_2504_10783_b200.errors import SeedOutsideDomain, SegmentInCollision
from paper_2504_10783_b200.polytope import HPolytope
from paper_2504_10783_b200.scene import World

pytestmark = pytest.mark.gpu


def _world(scene):
    if scene == "arm3":
        return fx.arm3_world()
    return {"disc_0_3": fx.disc_world([[0.0, 3.0]], 1.0), "disc_0_2": fx.disc_world([[0.0, 2.0]], 0.6),
            "disc_two": fx.disc_world([[0.0, 2.0], [0.0, -2.0]], 0.7),
            "disc_nit": fx.disc_world([[0.0, 1.2], [0.0, -1.2], [2.0, 1.2]], 0.5)}[scene]


def _run(rec, z, precision):
    world = _world(rec["scene"])
    v = z[f"{rec['key']}_v"]
    dom = HPolytope.from_bounds(world.lower, world.upper)
    ck = world.checker(precision=precision)
    rep = inflate_edge(Segment(v[0], v[1]), dom, InflationParams(**rec["params"]), ck, seed=rec["seed"])
    return rep, ck, dom, v


def test_fp64_reproduces_reference_polytopes():
    # same RNG stream + fp64 checks: the reference's polytope, iteration and check counts
    z, index = inflate_index()
    for rec in index:
        rep, ck, dom, v = _run(rec, z, "fp64")
        assert rep.iterations == rec["iterations"], rec["key"]
        assert rep.hyperplanes_added == rec["hyperplanes_added"], rec["key"]
        assert rep.collision_checks == rec["collision_checks"], rec["key"]
        assert rep.terminated_by == rec["terminated_by"], rec["key"]
        assert ck.calls == rec["collision_checks"]
        assert np.allclose(rep.polytope.A, z[f"{rec['key']}_A"], atol=1e-9), rec["key"]
        assert np.allclose(rep.polytope.b, z[f"{rec['key']}_b"], atol=1e-9), rec["key"]


def test_fp32_matches_reference_outside_contact_band():
    z, index = inflate_index()
    same = 0
    for rec in index:
        rep, ck, dom, v = _run(rec, z, "fp32")
        P = rep.polytope
        assert P.contains(v[0], 1e-9) and P.contains(v[1], 1e-9)
        if (rep.hyperplanes_added == rec["hyperplanes_added"] and P.n_faces == z[f"{rec['key']}_A"].shape[0]
                and np.allclose(P.A, z[f"{rec['key']}_A"], atol=1e-6)):
            same += 1
    assert same >= len(index) - 1


def test_empty_world_returns_domain():
    dom = HPolytope.from_bounds([-5, -5], [5, 5])
    ck = World(fx.point_robot_model()).checker()
    rep = inflate_edge(Segment(np.array([-1.0, 0.0]), np.array([1.0, 0.0])), dom, InflationParams(), ck, seed=3)
    assert rep.terminated_by == "test_accepted" and rep.iterations == 1 and rep.hyperplanes_added == 0
    assert np.array_equal(rep.polytope.A, dom.A) and np.array_equal(rep.polytope.b, dom.b)


def test_seed_outside_domain_and_segment_in_collision():
    dom = HPolytope.from_bounds([-1, -1], [1, 1])
    ck = World(fx.point_robot_model()).checker()
    with pytest.raises(SeedOutsideDomain):
        inflate_edge(Segment(np.array([0.0, 0.0]), np.array([2.0, 0.0])), dom, InflationParams(), ck)
    w = fx.disc_world([[1.0, 0.0]], radius=1.0)
    with pytest.raises(SegmentInCollision):
        inflate_edge(Segment(np.array([1.0, 0.0]), np.array([3.0, 0.0])), HPolytope.from_bounds([-5, -5], [5, 5]),
                     InflationParams(), w.checker(), seed=1)


@pytest.mark.parametrize("rng", ["counter", "philox"])
def test_structure_determinism_and_eps_audit(rng):
    dom = HPolytope.from_bounds([-5, -5], [5, 5])
    seg = Segment(np.array([-1.0, 0.0]), np.array([1.0, 0.0]))
    world = fx.disc_world([[0.0, 3.0]], radius=1.0)
    passes = 0
    for run in range(10):
        rep = inflate_edge(seg, dom, InflationParams(), world.checker(), seed=run, rng=rng)
        P = rep.polytope
        assert P.contains(seg.v1, 1e-9) and P.contains(seg.v2, 1e-9)
        assert rep.terminated_by == "test_accepted"
        assert np.array_equal(P.A[:dom.n_faces], dom.A) and P.n_faces == dom.n_faces + rep.hyperplanes_added
        mc = np.random.default_rng(10_000 + run)
        pts = mc.uniform(-5, 5, size=(200_000, 2))
        inside = pts[P.contains_many(pts)][:20_000]
        passes += np.mean(~world.checker().check_batch(inside)) <= 0.01
    assert passes >= 8
    r1 = inflate_edge(seg, dom, InflationParams(), world.checker(), seed=11, rng=rng)
    r2 = inflate_edge(seg, dom, InflationParams(), world.checker(), seed=11, rng=rng)
    assert np.array_equal(r1.polytope.A, r2.polytope.A) and r1.collision_checks == r2.collision_checks


def test_franka7_region_contains_segment():
    world = fx.franka7_world()
    v1, v2 = fx.random_free_segment(world, seed=3)
    dom = HPolytope.from_bounds(world.lower, world.upper)
    rep = inflate_edge(Segment(v1, v2), dom, InflationParams(**fx.FRANKA_PARAMS), world.checker(), seed=7)
    P = rep.polytope
    assert rep.terminated_by == "test_accepted"
    assert P.contains(v1, 1e-9) and P.contains(v2, 1e-9)
    assert rep.iterations >= 2 and rep.hyperplanes_added >= 10
    assert np.allclose(np.linalg.norm(P.A, axis=1), 1.0, atol=1e-12)


def test_degenerate_segment_matches_oracle():
    # v1 == v2: projection alpha = 0, c_proj = v1 (inflation.py:129-132); fp64 checks give the
    # oracle's (the reference algorithm's) iterations, faces and counters exactly
    from oracle import ref
    world = fx.disc_world([[0.0, 2.0]], 0.6)
    v = np.array([0.3, 0.4])
    dom = HPolytope.from_bounds(world.lower, world.upper)
    rep = inflate_edge(Segment(v, v.copy()), dom, InflationParams(), world.checker(precision="fp64"), seed=5)
    r = ref.inflate_edge(v, v.copy(), dom.A, dom.b, ref.OracleChecker(world), seed=5)
    assert rep.iterations == r["iterations"] and rep.hyperplanes_added == r["hyperplanes_added"]
    assert rep.collision_checks == r["collision_checks"]
    assert np.allclose(rep.polytope.A, r["A"], atol=1e-9) and np.allclose(rep.polytope.b, r["b"], atol=1e-9)
    assert rep.polytope.contains(v, 1e-9)


def test_n_it_one_places_once_then_stops():
    # n_it is checked after placement: exactly one round, "max_iterations" (inflation.py:314-316)
    world = fx.disc_world([[0.0, 1.2], [0.0, -1.2], [2.0, 1.2]], 0.5)
    seg = Segment(np.array([-1.0, 0.0]), np.array([1.0, 0.0]))
    dom = HPolytope.from_bounds(world.lower, world.upper)
    rep = inflate_edge(seg, dom, InflationParams(n_it=1), world.checker(), seed=2)
    assert rep.iterations == 1 and rep.terminated_by == "max_iterations"
    assert 0 < rep.hyperplanes_added <= InflationParams().n_f
    assert rep.polytope.contains(seg.v1, 1e-9) and rep.polytope.contains(seg.v2, 1e-9)


_BISECT_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge
from paper_2504_10783_b200.polytope import HPolytope
out = []
for world, prec in ((fx.franka7_world(), "fp32"), (fx.arm3_world(), "fp64")):
    v1, v2 = fx.random_free_segment(world, seed=3) if world.model.dof == 7 else fx.ARM3_SEGMENT
    dom = HPolytope.from_bounds(world.lower, world.upper)
    params = InflationParams(**fx.FRANKA_PARAMS) if world.model.dof == 7 else InflationParams()
    rep = inflate_edge(Segment(v1, v2), dom, params, world.checker(precision=prec), seed=7)
    out += [rep.polytope.A, rep.polytope.b, np.array([rep.collision_checks, rep.iterations])]
np.savez({path!r}, *out)
"""


def test_two_level_bisection_equals_one_step(tmp_path):
    """The bisection kernels against the one-step loop (`k_bisect`, EZ_BISECT1=1): `k_bisect2`
    (two binary levels per round of 8-lane checks, EZ_BISECT_JIT=0) and, for the specialised
    fp32 world, `ez_bisect_jit` (3-4 levels per round of single-thread checks, the default):
    same regions."""
    import os, subprocess, sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parents[1])
    res = []
    for flag, extra in (("1", {}), ("0", {"EZ_BISECT_JIT": "0"}), ("0", {})):
        path = str(tmp_path / f"b{flag}{len(extra)}.npz")
        env = dict(os.environ, EZ_BISECT1=flag, **extra)
        subprocess.run([sys.executable, "-c", _BISECT_CHILD.format(root=root, path=path)], env=env, check=True,
                       timeout=600)
        z = np.load(path)
        res.append([z[k] for k in sorted(z.files, key=lambda s: int(s.split("_")[1]))])
    for other in res[1:]:
        for a, b in zip(res[0], other):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("which", ["franka7", "bimanual14"])
def test_cluster_placement_equals_one_cta(which, monkeypatch):
    """k_place_cl (8-CTA cluster, anchors in shared memory) against k_place (one CTA,
    EZ_PLACE_1CTA=1, read per call): identical regions and counters."""
    world = fx.franka7_world() if which == "franka7" else fx.bimanual14_world()
    v1, v2 = fx.random_free_segment(world, seed=3)
    dom = HPolytope.from_bounds(world.lower, world.upper)
    params = InflationParams(**{**fx.FRANKA_PARAMS, **({"n_it": 4} if which == "bimanual14" else {})})
    ck = world.checker()
    reps = []
    for flag in (None, "1"):
        if flag:
            monkeypatch.setenv("EZ_PLACE_1CTA", flag)
        reps.append(inflate_edge(Segment(v1, v2), dom, params, ck, seed=7))
    a, b = reps
    assert (a.iterations, a.hyperplanes_added, a.collision_checks) == (b.iterations, b.hyperplanes_added, b.collision_checks)
    assert np.array_equal(a.polytope.A, b.polytope.A) and np.array_equal(a.polytope.b, b.polytope.b)


def test_franka7_region_eps_audit_independent_sampler():
    """SURVEY 8(c)(ii) audit in 7-D: the region's collision fraction, measured on an
    independent hit-and-run stream (other seed, 200 mixing steps) with flags from the CPU
    oracle, is at most eps (0.005; the survey measured 0.0025 on this region)."""
    from oracle import ref
    from paper_2504_10783_b200.polytope import hit_and_run_sample
    world = fx.franka7_world()
    v1, v2 = fx.random_free_segment(world, seed=3)
    dom = HPolytope.from_bounds(world.lower, world.upper)
    rep = inflate_edge(Segment(v1, v2), dom, InflationParams(**fx.FRANKA_PARAMS), world.checker(), seed=7)
    P = rep.polytope
    assert P.contains(v1, 1e-9) and P.contains(v2, 1e-9)
    X = hit_and_run_sample(P, (0.5 * (v1 + v2))[None, :], 20_000, 200, seed=424_242).points
    assert P.contains_many(X, 1e-9).all()
    colliding = ~ref.OracleChecker(world).check_batch(X)
    assert colliding.mean() <= FRANKA_EPS
    # the GPU checker agrees with the oracle on these samples outside the contact band
    clr = ref.OracleChecker(world).clearance(X)
    free = world.checker().check_batch(X)
    assert not ((free != (clr > 0)) & (np.abs(clr) >= 1e-5)).any()


FRANKA_EPS = fx.FRANKA_PARAMS["eps"]


def test_face_cap_overflow_counts_then_copies():
    """ez_inflate_edge with a face_cap below the result: EZ_CAPACITY with a complete report, the
    rows kept for ez_inflate_edge_result (count, then copy), equal to a normal call's."""
    import ctypes as C

    from paper_2504_10783_b200 import _native as N
    from paper_2504_10783_b200.eizo import default_bisection_steps

    world = fx.disc_world([[0.0, 1.2], [0.0, -1.2], [2.0, 1.2]], 0.5)
    seg = Segment(np.array([-1.0, 0.0]), np.array([1.0, 0.0]))
    dom = HPolytope.from_bounds(world.lower, world.upper)
    params = InflationParams()
    ck = world.checker()
    full = inflate_edge(seg, dom, params, ck, seed=4)
    assert full.polytope.n_faces > 5
    p = N.EizoParams(params.delta, params.eps, params.tau, params.delta_max, params.t_col, params.n_p, params.n_f,
                     default_bisection_steps(dom, params.delta_max), params.n_ms, 0)
    rep = N.EizoReport()
    small = 2
    A_out, b_out = np.empty((small, 2)), np.empty(small)
    v1, v2 = np.ascontiguousarray(seg.v1), np.ascontiguousarray(seg.v2)
    A0, b0 = np.ascontiguousarray(dom.A), np.ascontiguousarray(dom.b)
    st = N.lib().ez_inflate_edge(ck.native.handle, N.ptr(v1), N.ptr(v2), 2, N.ptr(A0), N.ptr(b0), dom.n_faces,
                                 C.byref(p), 4, 0, 0, C.byref(rep), N.ptr(A_out), N.ptr(b_out), small)
    assert st == 11 and rep.n_faces == full.polytope.n_faces and rep.iterations == full.iterations
    A2, b2 = np.empty((rep.n_faces, 2)), np.empty(rep.n_faces)
    nf = C.c_int32(0)
    assert N.lib().ez_inflate_edge_result(N.ptr(A2), N.ptr(b2), rep.n_faces, C.byref(nf)) == 0
    assert nf.value == rep.n_faces
    assert np.array_equal(A2, full.polytope.A) and np.array_equal(b2, full.polytope.b)
