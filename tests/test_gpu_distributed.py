"""Sharded EI-ZO on the GPU: G shards (driven in one process) reproduce the single-GPU inflation exactly.

Mirrors the reference's partition-invariance tests (test_cpoly.py:98-118):
the samples of any walk range depend only on the global walk index, so 1 and
G shards must produce identical flags, candidates and polytopes.
"""

import numpy as np
import pytest

from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.distributed import inflate_edge_sharded, inflate_segments_sharded
from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge
from paper_2504_10783_b200.polytope import HPolytope
from paper_2504_10783_b200.roadmap import PwlPath

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shards", [1, 2, 3, 4])
def test_sharded_equals_single_planar(shards):
    world = fx.arm3_world()
    v1, v2 = fx.ARM3_SEGMENT
    dom = HPolytope.from_bounds(world.lower, world.upper)
    params = InflationParams()
    single = inflate_edge(Segment(v1, v2), dom, params, world.checker(), seed=1)
    sh = inflate_edge_sharded(Segment(v1, v2), dom, params, world.checker(), seed=1, shards=shards)
    assert sh.iterations == single.iterations and sh.collision_checks == single.collision_checks
    assert np.array_equal(sh.polytope.A, single.polytope.A) and np.array_equal(sh.polytope.b, single.polytope.b)


def test_sharded_equals_single_franka7():
    world = fx.franka7_world()
    v1, v2 = fx.random_free_segment(world, seed=3)
    dom = HPolytope.from_bounds(world.lower, world.upper)
    params = InflationParams(**fx.FRANKA_PARAMS)
    ck = world.checker()
    single = inflate_edge(Segment(v1, v2), dom, params, ck, seed=7)
    sh = inflate_edge_sharded(Segment(v1, v2), dom, params, ck, seed=7, shards=3)
    assert sh.iterations == single.iterations and sh.hyperplanes_added == single.hyperplanes_added
    assert sh.collision_checks == single.collision_checks
    assert np.array_equal(sh.polytope.A, single.polytope.A) and np.array_equal(sh.polytope.b, single.polytope.b)


def test_segment_sharding_single_rank_covers_path():
    world = fx.franka7_world()
    ck = world.checker()
    knots = [fx.random_free_segment(world, seed=3)[0]]
    rng = np.random.default_rng(0)
    while len(knots) < 4:
        d = rng.normal(size=7)
        nxt = knots[-1] + d / np.linalg.norm(d) * 0.4
        if np.all(nxt > world.lower) and np.all(nxt < world.upper) and world.checker(margin=0.02).check_segment(
                knots[-1], nxt, 0.01):
            knots.append(nxt)
    path = PwlPath(np.array(knots))
    dom = HPolytope.from_bounds(world.lower, world.upper)
    scs, mine = inflate_segments_sharded(path, dom, InflationParams(**fx.FRANKA_PARAMS), ck, seed=5)
    assert sorted(mine) == [0, 1, 2]
    for k, c in enumerate(scs.coverage):
        assert scs.sets[c].contains_segment(knots[k], knots[k + 1])


def test_concurrent_segments_equal_sequential():
    # several inflations in flight on one GPU (one workspace and stream each): same corridor
    from paper_2504_10783_b200.distributed import inflate_segments_sharded
    from paper_2504_10783_b200.eizo import InflationParams
    from paper_2504_10783_b200.polytope import HPolytope
    from paper_2504_10783_b200.roadmap import PwlPath

    world = fx.franka7_world()
    path = PwlPath(fx.random_free_path(world, 6, seed=5))
    dom = HPolytope.from_bounds(world.lower, world.upper)
    params = InflationParams(**fx.FRANKA_PARAMS)
    ck = world.checker()
    seq, mine1 = inflate_segments_sharded(path, dom, params, ck, seed=3, concurrency=1)
    calls1 = ck.calls
    par, mine4 = inflate_segments_sharded(path, dom, params, ck, seed=3, concurrency=4)
    assert seq.coverage == par.coverage and len(seq.sets) == len(par.sets)
    for a, b in zip(seq.sets, par.sets):
        assert np.array_equal(a.A, b.A) and np.array_equal(a.b, b.b)
    assert {k: v[4] for k, v in mine1.items()} == {k: v[4] for k, v in mine4.items()}
    assert ck.calls == 2 * calls1
