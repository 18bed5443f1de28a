"""inflate_path / refine_sets (planner.py:103-224) on the GPU vs the reference's own run."""

import numpy as np
import pytest

from conftest import golden
from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.corridor import find_path_collisions, inflate_path, refine_sets
from paper_2504_10783_b200.eizo import InflationParams
from paper_2504_10783_b200.polytope import HPolytope
from paper_2504_10783_b200.roadmap import PwlPath

pytestmark = pytest.mark.gpu


def _setup(precision="fp64"):
    z = golden("corridor.npz")
    world = fx.disc_world(z["centers"])
    path = PwlPath(z["knots"])
    dom = HPolytope.from_bounds([-5, -5], [5, 5])
    params = InflationParams(n_it=1, n_f=2)
    return z, world, path, dom, params


def test_inflate_path_matches_reference():
    z, world, path, dom, params = _setup()
    scs = inflate_path(path, dom, params, world.checker(precision="fp64"), seed=21)
    assert len(scs.sets) == int(z["n_sets"])
    assert list(scs.coverage) == list(z["coverage"])
    for i, P in enumerate(scs.sets):
        assert np.allclose(P.A, z[f"set{i}_A"], atol=1e-9) and np.allclose(P.b, z[f"set{i}_b"], atol=1e-9)


def test_refine_sets_matches_reference():
    z, world, path, dom, params = _setup()
    ck = world.checker(precision="fp64")
    scs = inflate_path(path, dom, params, ck, seed=21)
    cols = [(int(j), c) for j, c in zip(z["col_sets"], z["cols"])]
    ref = refine_sets(scs, cols, path, params, ck, seed=9)
    assert len(ref.sets) == int(z["r_n_sets"])
    assert list(ref.coverage) == list(z["r_coverage"])
    for i, P in enumerate(ref.sets):
        assert np.allclose(P.A, z[f"rset{i}_A"], atol=1e-9) and np.allclose(P.b, z[f"rset{i}_b"], atol=1e-9)
    # every reported collision is now outside its set
    for j, c in cols:
        assert not ref.sets[j].contains(c, 0.0)


def test_find_path_collisions_attribution():
    z, world, path, dom, params = _setup()
    scs = inflate_path(path, dom, params, world.checker(), seed=21)
    straight = np.array([[-4.5, -4.5], [4.5, 4.5]])  # crosses discs
    found = find_path_collisions(scs, straight, world.checker(), 0.01)
    assert found and all(0 <= j < len(scs.sets) for j, _ in found)
    assert not np.any(world.checker().check_batch(np.array([c for _, c in found])))
