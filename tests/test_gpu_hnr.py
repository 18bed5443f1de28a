"""GPU hit-and-run (k_hnr) against the reference's samples and its property tests (test_cpoly.py:69-131)."""

import numpy as np
import pytest

from conftest import golden
from paper_2504_10783_b200.errors import EmptyChord, SeedOutside
from paper_2504_10783_b200.polytope import HPolytope, hit_and_run_sample

pytestmark = pytest.mark.gpu


def unit_box(d=2):
    return HPolytope.from_bounds(np.zeros(d), np.ones(d))


@pytest.mark.parametrize("name", ["box2", "box3", "poly7"])
def test_counter_stream_reproduces_reference_samples(name):
    # same (seed, walk, step, slot) stream as the reference: samples agree to rounding
    z = golden("hnr.npz")
    count, n_ms, seed, off = (int(v) for v in z[f"{name}_meta"])
    poly = HPolytope(z[f"{name}_A"], z[f"{name}_b"])
    sb = hit_and_run_sample(poly, z[f"{name}_seeds"], count, n_ms, seed, off)
    assert sb.rng_state == (seed, off + count)
    assert np.max(np.abs(sb.points - z[f"{name}_X"])) <= 1e-9


@pytest.mark.parametrize("rng", ["counter", "philox"])
def test_membership_of_all_samples(rng):
    box = unit_box()
    sb = hit_and_run_sample(box, np.array([[0.5, 0.5]]), 100_000, 30, seed=9, rng=rng)
    assert np.max(sb.points @ box.A.T - box.b) <= 1e-9


@pytest.mark.parametrize("rng", ["counter", "philox"])
def test_uniformity_grid_audit(rng):
    sb = hit_and_run_sample(unit_box(), np.array([[0.5, 0.5]]), 100_000, 30, seed=4, rng=rng)
    counts, _, _ = np.histogram2d(sb.points[:, 0], sb.points[:, 1], bins=4, range=[[0, 1], [0, 1]])
    assert np.all(np.abs(counts / 100_000 - 1 / 16) <= 0.15 / 16)


@pytest.mark.parametrize("rng", ["counter", "philox"])
def test_determinism_and_partition_invariance(rng):
    box = HPolytope.from_bounds([-2, 0, 1], [3, 4, 2])
    seeds = np.array([[0.0, 2.0, 1.5]])
    a = hit_and_run_sample(box, seeds, 600, 15, seed=77, rng=rng)
    b = hit_and_run_sample(box, seeds, 600, 15, seed=77, rng=rng)
    assert np.array_equal(a.points, b.points)
    first = hit_and_run_sample(box, seeds, 250, 15, seed=77, walk_offset=0, rng=rng)
    second = hit_and_run_sample(box, seeds, 350, 15, seed=77, walk_offset=250, rng=rng)
    assert np.array_equal(np.vstack([first.points, second.points]), a.points)
    assert second.rng_state == (77, 600)


def test_empty_batch_and_errors():
    sb = hit_and_run_sample(unit_box(), np.array([[0.5, 0.5]]), 0, 30, seed=1)
    assert sb.points.shape == (0, 2) and sb.rng_state == (1, 0)
    with pytest.raises(ValueError):
        hit_and_run_sample(unit_box(), np.array([[0.5, 0.5]]), 10, 0, seed=1)
    with pytest.raises(SeedOutside):
        hit_and_run_sample(unit_box(), np.array([[2.0, 0.5]]), 10, 5, seed=0)
    poly = HPolytope(np.array([[1.0, 0.0], [-1.0, 0.0], [0.0, 1.0], [0.0, -1.0]]),
                     np.array([-1e-10, -1e-10, 1.0, 0.0]))
    with pytest.raises(EmptyChord):
        hit_and_run_sample(poly, np.array([[0.0, 0.5]]), 10, 5, seed=0)


def test_many_faces_high_dim():
    rng = np.random.default_rng(0)
    d = 14
    A = rng.normal(size=(200, d))
    A /= np.linalg.norm(A, axis=1, keepdims=True)
    poly = HPolytope(A, np.full(200, 0.5))
    sb = hit_and_run_sample(poly, np.zeros((1, d)), 5000, 40, seed=3)
    assert np.max(sb.points @ poly.A.T - poly.b) <= 1e-9


# --- the FP64 tensor-core walk (k_hnr_mma; the lane-per-face walk under EZ_HNR_NO_MMA) -----

def _random_poly(d, n_faces, seed, r=0.5):
    rng = np.random.default_rng(seed)
    A = rng.normal(size=(n_faces, d))
    A /= np.linalg.norm(A, axis=1, keepdims=True)
    return HPolytope(A, np.full(n_faces, r))


@pytest.mark.parametrize("d,n_faces", [(7, 120), (14, 300), (20, 150)])
def test_mma_walk_matches_oracle(d, n_faces):
    from oracle import ref
    poly = _random_poly(d, n_faces, seed=d)
    seeds = np.zeros((1, d))
    sb = hit_and_run_sample(poly, seeds, 257, 12, seed=5, walk_offset=3)
    X = ref.hit_and_run(poly.A, poly.b, seeds, 257, 12, 5, walk_offset=3)
    # rounding-level differences in the face sums only (tolerance as the goldens above)
    assert np.max(np.abs(sb.points - X)) <= 1e-9
    assert np.max(sb.points @ poly.A.T - poly.b) <= 1e-9


def test_mma_walk_agrees_with_lane_walk(monkeypatch):
    poly = _random_poly(14, 400, seed=2)
    seeds = np.zeros((1, 14))
    a = hit_and_run_sample(poly, seeds, 3000, 30, seed=8)
    monkeypatch.setenv("EZ_HNR_NO_MMA", "1")
    b = hit_and_run_sample(poly, seeds, 3000, 30, seed=8)
    assert np.max(np.abs(a.points - b.points)) <= 1e-9


def test_mma_walk_partition_invariance():
    poly = _random_poly(14, 200, seed=3)
    seeds = np.zeros((1, 14))
    a = hit_and_run_sample(poly, seeds, 1000, 10, seed=77)
    first = hit_and_run_sample(poly, seeds, 333, 10, seed=77, walk_offset=0)
    second = hit_and_run_sample(poly, seeds, 667, 10, seed=77, walk_offset=333)
    assert np.array_equal(np.vstack([first.points, second.points]), a.points)


def test_mma_walk_errors():
    poly = _random_poly(14, 128, seed=4)
    with pytest.raises(SeedOutside):
        hit_and_run_sample(poly, np.full((1, 14), 5.0), 10, 5, seed=0)
    # two opposite faces leave an empty slab (x_0 <= -1e-10 and -x_0 <= -1e-10)
    A = np.vstack([poly.A, np.eye(14)[:1], -np.eye(14)[:1]])
    b = np.concatenate([poly.b, [-1e-10, -1e-10]])
    with pytest.raises(EmptyChord):
        hit_and_run_sample(HPolytope(A, b), np.zeros((1, 14)), 10, 5, seed=0)
