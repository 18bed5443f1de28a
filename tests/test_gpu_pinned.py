"""Parity at the benchmark configurations themselves, against the reference's own outputs.

* config 2 at full size: the 2^20 fp32 rows of ``fixtures.config2_rows()`` through the exact
  launch ``bench.py`` times (``ez_check_batch`` on fp32 device rows, model-specialised kernel)
  against the reference's flags (``tests/golden/config2_1m.npz``, made by the reference's
  ``check_batch``, world.py:483-565);
* the benchmark's 7-DOF EI-ZO region (segment seed 3, EI-ZO seed 7) against the reference's
  ``inflate_edge`` (inflation.py:262-325) on the same segment (``tests/golden/region7.npz``);
* config 4: the 14-DOF region's held-out eps-audit;
* acceptance criterion 3 (test_acceptance.py:96-131) on the GPU path, and the 100 reference
  polytopes it produces reproduced with fp64 checks (``tests/golden/criterion3.npz``);
* oblique revolute axes and a 3-D prismatic joint (world.py:64-69, 174-192) against the
  reference's FK and flags (``tests/golden/check_oblique.npz``).
"""

import ctypes as C

import numpy as np
import pytest
import torch

from conftest import golden
from paper_2504_10783_b200 import _native as N
from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge
from paper_2504_10783_b200.polytope import HPolytope, hit_and_run_sample
from paper_2504_10783_b200.rng import child_seed

pytestmark = pytest.mark.gpu

BAND = 1e-5


def _config2_golden():
    z = golden("config2_1m.npz")
    n = int(z["n"])
    free = np.unpackbits(z["free_bits"])[:n].astype(bool)
    band = np.zeros(n, dtype=bool)
    band[z["band"]] = True
    return free, band


def test_config2_full_size_through_the_bench_launch():
    """2^20 config-2 rows through bench.py's timed call, against the reference's flags."""
    free_ref, band = _config2_golden()
    world = fx.franka7_world()
    nat = world.checker().native
    assert nat.specialize(1), "NVRTC specialisation unavailable on this box"
    Q = torch.as_tensor(fx.config2_rows(), device="cuda")
    out = torch.empty(Q.shape[0], dtype=torch.uint8, device="cuda")
    sh = torch.cuda.current_stream().cuda_stream
    # exactly bench.py's step(): fp32 device rows, ld 7, fp32 arithmetic, current stream
    N.check(N.lib().ez_check_batch(nat.handle, Q.data_ptr(), 0, Q.shape[0], 7, out.data_ptr(), 0, sh))
    torch.cuda.synchronize()
    assert nat.info()["check_cta"] in (256, 512, 1024)
    free = out.cpu().numpy().astype(bool)
    mism = (free != free_ref) & ~band
    assert not mism.any(), f"{int(mism.sum())} flag mismatches outside the {BAND} band of {free.size}"
    # and the fp64 arithmetic path: bit-exact except at |clearance| < 1e-12 (a subset of the band)
    N.check(N.lib().ez_check_batch(nat.handle, Q.data_ptr(), 0, Q.shape[0], 7, out.data_ptr(), 1, sh))
    torch.cuda.synchronize()
    free64 = out.cpu().numpy().astype(bool)
    assert not ((free64 != free_ref) & ~band).any()
    assert int((free64 != free_ref).sum()) <= int(band.sum())


def test_config2_host_fp32_rows_match_reference():
    """The drop-in numpy call with fp32 rows (the e2e path) gives the same flags."""
    free_ref, band = _config2_golden()
    Q = fx.config2_rows()[:200_000]
    ck = fx.franka7_world().checker()
    free = ck.check_batch(Q)
    assert ck.calls == Q.shape[0]
    assert not ((free != free_ref[:200_000]) & ~band[:200_000]).any()


def _region7():
    z = golden("region7.npz")
    world = fx.franka7_world()
    v1, v2 = fx.random_free_segment(world, seed=3)
    # the benchmark segment found with the GPU checker is the one the reference's checker finds
    assert np.array_equal(v1, z["v1"]) and np.array_equal(v2, z["v2"])
    dom = HPolytope.from_bounds(world.lower, world.upper)
    return z, world, v1, v2, dom


def test_region7_fp64_reproduces_reference():
    """The benchmark region with fp64 checks: the reference's polytope and counters."""
    z, world, v1, v2, dom = _region7()
    ck = world.checker(precision="fp64")
    rep = inflate_edge(Segment(v1, v2), dom, InflationParams(**fx.FRANKA_PARAMS), ck, seed=7)
    assert rep.iterations == int(z["iterations"])
    assert rep.hyperplanes_added == int(z["hyperplanes_added"])
    assert rep.collision_checks == int(z["collision_checks"]) == ck.calls
    assert rep.terminated_by == str(z["terminated_by"])
    assert rep.polytope.A.shape == z["A"].shape
    assert np.allclose(rep.polytope.A, z["A"], atol=1e-9) and np.allclose(rep.polytope.b, z["b"], atol=1e-9)


def test_region7_fp32_matches_reference_counters():
    """The benchmark's own (fp32) region: same iterations, faces and checks as the reference,
    segment contained, faces within 1e-6 of the reference's."""
    z, world, v1, v2, dom = _region7()
    rep = inflate_edge(Segment(v1, v2), dom, InflationParams(**fx.FRANKA_PARAMS), world.checker(), seed=7)
    P = rep.polytope
    assert P.contains(v1, 1e-9) and P.contains(v2, 1e-9)
    assert (rep.iterations, rep.hyperplanes_added, rep.collision_checks) == (
        int(z["iterations"]), int(z["hyperplanes_added"]), int(z["collision_checks"]))
    assert np.allclose(P.A, z["A"], atol=1e-6) and np.allclose(P.b, z["b"], atol=1e-6)


def test_region14_eps_audit_independent_sampler():
    """Config 4 (14-DOF bimanual, paper Franka (eps, delta)): containment and the SURVEY 8(c)(ii)
    audit -- 2e4 points from an independent hit-and-run stream (other seed, 200 mixing steps),
    flagged by the CPU oracle, collide at a fraction <= eps."""
    from oracle import ref

    z = golden("region7.npz")
    world = fx.bimanual14_world()
    v1, v2 = fx.random_free_segment(world, seed=3)
    assert np.array_equal(v1, z["seg14_v1"]) and np.array_equal(v2, z["seg14_v2"])
    dom = HPolytope.from_bounds(world.lower, world.upper)
    rep = inflate_edge(Segment(v1, v2), dom, InflationParams(**fx.FRANKA_PARAMS), world.checker(), seed=7)
    P = rep.polytope
    assert rep.terminated_by == "test_accepted"
    assert P.contains(v1, 1e-9) and P.contains(v2, 1e-9)
    assert np.allclose(np.linalg.norm(P.A, axis=1), 1.0, atol=1e-12)
    X = hit_and_run_sample(P, (0.5 * (v1 + v2))[None, :], 20_000, 200, seed=424_242).points
    assert P.contains_many(X, 1e-9).all()
    oc = ref.OracleChecker(world, workers=8)
    colliding = ~oc.check_batch(X)
    assert colliding.mean() <= fx.FRANKA_PARAMS["eps"], f"collision fraction {colliding.mean():.4f}"
    clr = oc.clearance(X)
    free = world.checker().check_batch(X)
    assert not ((free != (clr > 0)) & (np.abs(clr) >= BAND)).any()


def _criterion3_world(z, run):
    return fx.disc_world(z[f"r{run}_centers"], float(z["radius"]))


def test_criterion3_reference_polytopes_fp64():
    """The 100 acceptance-audit inflations (test_acceptance.py:96-131): with fp64 checks the GPU
    path returns the reference's polytope and counters for every run."""
    z = golden("criterion3.npz")
    dom = HPolytope.from_bounds([-5, -5], [5, 5])
    params = InflationParams(delta=0.05, eps=0.01)
    bad = []
    for run in range(100):
        v = z[f"r{run}_v"]
        it, faces, checks, accepted, seed = (int(x) for x in z["recs"][run])
        assert seed == child_seed(77, run)
        rep = inflate_edge(Segment(v[0], v[1]), dom, params, _criterion3_world(z, run).checker(precision="fp64"),
                           seed=seed)
        same = ((rep.iterations, rep.hyperplanes_added, rep.collision_checks) == (it, faces, checks)
                and rep.polytope.A.shape == z[f"r{run}_A"].shape
                and np.allclose(rep.polytope.A, z[f"r{run}_A"], atol=1e-9)
                and np.allclose(rep.polytope.b, z[f"r{run}_b"], atol=1e-9))
        if not same:
            bad.append(run)
    assert not bad, f"runs differing from the reference: {bad}"


def test_criterion3_guarantee_on_gpu_path():
    """Criterion 3 as the reference states it, on the default (fp32) GPU path: segments found by
    the reference's rejection rule with the GPU checker, each region audited with 5e4
    independent uniform samples (rejection from the box); <= 15/100 exceed eps = 0.01."""
    import time

    z = golden("criterion3.npz")
    dom = HPolytope.from_bounds([-5, -5], [5, 5])
    params = InflationParams(delta=0.05, eps=0.01)
    exceed = 0
    t0 = time.perf_counter()
    for run in range(100):
        world = _criterion3_world(z, run)
        rng = np.random.default_rng(child_seed(31, run))
        ck = world.checker(margin=0.01)
        while True:  # test_acceptance.py:80-92
            v1 = rng.uniform(-4.5, 4.5, 2)
            if not ck.check(v1):
                continue
            direction = rng.normal(size=2)
            direction /= np.linalg.norm(direction)
            v2 = v1 + direction * rng.uniform(0.5, 2.5)
            if np.any(np.abs(v2) > 4.7):
                continue
            if ck.check_segment(v1, v2, 0.01):
                break
        assert np.array_equal(np.stack([v1, v2]), z[f"r{run}_v"]), run
        rep = inflate_edge(Segment(v1, v2), dom, params, world.checker(), seed=child_seed(77, run))
        P = rep.polytope
        assert P.contains(v1, 1e-9) and P.contains(v2, 1e-9)
        mc = np.random.default_rng(child_seed(99, run))
        kept, need = [], 50_000
        while need > 0:
            draw = mc.uniform(-5, 5, size=(200_000, 2))
            take = draw[P.contains_many(draw)][:need]
            kept.append(take)
            need -= take.shape[0]
        frac = float(np.mean(~world.checker().check_batch(np.concatenate(kept))))
        exceed += frac > params.eps
    elapsed = time.perf_counter() - t0
    assert exceed <= 15 and elapsed < 300.0, (exceed, elapsed)


@pytest.mark.parametrize("mode", ["generic", "specialised", "fp64"])
def test_oblique_axes_and_prismatic_match_reference(mode):
    from oracle.gen_goldens import oblique_world

    z = golden("check_oblique.npz")
    w = oblique_world()
    ck = w.checker(precision="fp64" if mode == "fp64" else "fp32")
    if mode == "generic":
        ck.native.specialize(-1)
    elif mode == "specialised":
        assert ck.native.specialize(1)
    Q = torch.as_tensor(z["Q"], device="cuda")
    free = ck.check_batch(Q).cpu().numpy()
    band = np.abs(z["clearance"]) < (1e-12 if mode == "fp64" else BAND)
    assert not ((free != z["free"]) & ~band).any()


def test_oblique_fk_matches_reference():
    from oracle.gen_goldens import oblique_world
    from paper_2504_10783_b200.model import fk_batch

    z = golden("check_oblique.npz")
    rots, trans = fk_batch(oblique_world().model, z["fk_Q"])
    assert np.allclose(np.stack(rots, axis=1), z["fk_rot"], atol=1e-12)
    assert np.allclose(np.stack(trans, axis=1), z["fk_trans"], atol=1e-12)
