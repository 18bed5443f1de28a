"""GPU voxelisation (ez_voxelize) and DRM prune (ez_collision_set) vs the reference: exact set equality."""

import numpy as np
import pytest

from conftest import golden
from paper_2504_10783_b200.errors import GridMismatch
from paper_2504_10783_b200.roadmap import CollisionSet, Drm, Grid, collision_set
from paper_2504_10783_b200.scene import VoxelMap, voxelize_point_cloud

pytestmark = pytest.mark.gpu


def test_voxelize_matches_reference():
    z = golden("voxelize.npz")
    vm3 = voxelize_point_cloud(z["p3"], 0.02, z["o3"])
    assert np.array_equal(vm3.index_array(), z["idx3"])
    vm2 = voxelize_point_cloud(z["p2"], 0.5, z["o2"])
    assert np.array_equal(vm2.index_array(), z["idx2"])
    assert vm2.occupied == frozenset(map(tuple, z["idx2"].tolist()))


def test_voxelize_conventions():
    assert voxelize_point_cloud(np.zeros((0, 2)), 0.5, np.zeros(2)).n_occupied == 0
    vm = voxelize_point_cloud(np.array([[0.25, 0.25], [0.26, 0.24]]), 0.5, np.zeros(2))
    assert vm.occupied == frozenset({(0, 0)})
    assert voxelize_point_cloud(np.array([[1.0, 0.2]]), 0.5, np.zeros(2)).occupied == frozenset({(2, 0)})
    neg = voxelize_point_cloud(np.array([[-0.1, -3.0, 0.0]]), 0.5, np.zeros(3))
    assert neg.occupied == frozenset({(-1, -6, 0)})
    with pytest.raises(ValueError):
        voxelize_point_cloud(np.zeros((1, 2)), 0.0, np.zeros(2))


def _drm(off, ids, grid):
    n_nodes = int(ids.max()) + 1 if ids.size else 1
    z = np.zeros((n_nodes, 2))
    return Drm(z, np.zeros(n_nodes + 1, np.int64), np.zeros(0, np.int32), off, ids, z, grid)


def test_collision_set_forest_matches_reference():
    z = golden("drm.npz")
    grid = Grid(np.array([-5.0, -5.0]), 0.25, (40, 40))
    drm = Drm(np.zeros((200, 2)), np.zeros(201, np.int64), np.zeros(0, np.int32), z["f_off"], z["f_ids"],
              np.zeros((200, 3)), grid)
    for i in range(int(z["f_nmaps"])):
        vm = VoxelMap(z[f"f{i}_org"], float(z[f"f{i}_side"]), z[f"f{i}_idx"])
        got = collision_set(drm, vm)
        assert np.array_equal(got.ids, z[f"f{i}_blocked"])
        assert got.blocked == frozenset(z[f"f{i}_blocked"].tolist())


def test_collision_set_franka_matches_reference():
    z = golden("drm.npz")
    grid = Grid(np.array([-0.75, -1.02, -0.36]), 0.06, (25, 34, 26))
    n = z["g_nodes"].shape[0]
    drm = Drm(z["g_nodes"], np.zeros(n + 1, np.int64), np.zeros(0, np.int32), z["g_off"], z["g_ids"],
              np.zeros((n, 7)), grid)
    for tag in ("same", "fine"):
        vm = VoxelMap(z[f"g_{tag}_org"], float(z[f"g_{tag}_side"]), z[f"g_{tag}_idx"])
        assert np.array_equal(collision_set(drm, vm).ids, z[f"g_{tag}_blocked"])


def test_collision_set_empty_all_and_mismatch():
    z = golden("drm.npz")
    grid = Grid(np.array([-5.0, -5.0]), 0.25, (40, 40))
    drm = Drm(np.zeros((200, 2)), np.zeros(201, np.int64), np.zeros(0, np.int32), z["f_off"], z["f_ids"],
              np.zeros((200, 3)), grid)
    assert collision_set(drm, VoxelMap(grid.origin, grid.side, ())).blocked == frozenset()
    allv = VoxelMap(grid.origin, grid.side, [(i, j) for i in range(40) for j in range(40)])
    union = np.unique(z["f_ids"]).astype(np.int64)
    assert np.array_equal(collision_set(drm, allv).ids, union)
    with pytest.raises(GridMismatch):
        collision_set(drm, VoxelMap(np.zeros(3), 0.25, [(0, 0, 0)]))


def test_collision_map_build_matches_reference():
    # the reference's own build_drm collision map for its 300 nodes (drm.py:170-204, 250-251)
    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.roadmap import build_collision_map

    z = golden("drm.npz")
    grid = Grid(np.array([-0.75, -1.02, -0.36]), 0.06, (25, 34, 26))
    off, ids = build_collision_map(fx.franka7_world(False), z["g_nodes"], grid)
    assert np.array_equal(off, z["g_off"])
    assert np.array_equal(ids, z["g_ids"])


def test_collision_map_build_planar():
    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.roadmap import build_collision_map

    z = golden("drm.npz")
    grid = Grid(np.array([-5.0, -5.0]), 0.25, (40, 40))
    # nodes of the 2-D golden are not stored; rebuild a map from random nodes and check it against the oracle
    from oracle import ref

    rng = np.random.default_rng(4)
    nodes = rng.uniform(-5, 5, size=(300, 2))
    model = fx.point_robot_model()
    off, ids = build_collision_map(model, nodes, grid)
    rows, cols = ref.node_voxel_pairs(model, nodes, grid.origin, grid.side, grid.extents)
    order = np.lexsort((rows, cols))
    counts = np.bincount(cols, minlength=grid.n_voxels)
    assert np.array_equal(np.diff(off), counts)
    assert np.array_equal(ids, rows[order].astype(np.int32))


def test_free_node_sampling():
    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.roadmap import sample_free_nodes

    w = fx.franka7_world(False)
    nodes = sample_free_nodes(w, 5000, seed=1, batch=1 << 14)
    assert nodes.shape == (5000, 7)
    assert np.all(w.checker().check_batch(nodes))
    assert np.all(nodes >= w.lower) and np.all(nodes <= w.upper)


@pytest.mark.parametrize("which", ["forest", "franka", "franka_filtered"])
def test_build_drm_matches_reference(which):
    """The drop-in build_drm (drm.py:207-255) against the reference's own builds: the same
    nodes (same draws, GPU fp64 checks), poses to 1e-12, adjacency and collision map exact."""
    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.roadmap import build_drm
    from paper_2504_10783_b200.scene import World

    z = golden("drm.npz")
    if which == "forest":
        model = fx.point_robot_model()
        world = World(model)
        grid = Grid(np.array([-5.0, -5.0]), 0.25, (40, 40))
        args, seed, key = (200, 10, 10.0, 10.0), 8, "f"
    else:
        world = fx.franka7_world(False)
        model = world.model
        grid = Grid(np.array([-0.75, -1.02, -0.36]), 0.06, (25, 34, 26))
        args, seed, key = ((300, 10, 10.0, 10.0), 0, "g") if which == "franka" else ((400, 4, 2.5, 0.35), 5, "h")
    d = build_drm(model, world.checker(precision="fp64"), model.lower, model.upper, *args, grid, seed=seed)
    assert np.array_equal(d.nodes, z[f"{key}_nodes"])
    assert d.poses.shape == z[f"{key}_poses"].shape
    assert np.allclose(d.poses, z[f"{key}_poses"], atol=1e-12)
    assert np.array_equal(d.adj_offsets, z[f"{key}_adj_off"])
    assert np.array_equal(d.adj_ids, z[f"{key}_adj_ids"])
    off_key, ids_key = (f"{key}_off", f"{key}_ids")
    assert np.array_equal(d.cmap_offsets, z[off_key]) and np.array_equal(d.cmap_ids, z[ids_key])
    # reference properties (test_drm.py:30-66): symmetric adjacency, free nodes
    for i in range(d.n_nodes):
        for j in d.neighbors(i):
            assert i in set(int(v) for v in d.neighbors(int(j)))
    assert world.checker(precision="fp64").check_batch(d.nodes).all()


def test_build_drm_two_nodes_and_validation():
    """test_drm.py:45-51: two nodes with k = 1 give one undirected edge; bad sizes raise."""
    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.roadmap import build_drm
    from paper_2504_10783_b200.scene import World

    base = World(fx.point_robot_model())
    grid = Grid(np.array([-5.0, -5.0]), 0.25, (40, 40))
    d = build_drm(base.model, base.checker(), base.lower, base.upper, 2, 1, 100.0, 100.0, grid, seed=1)
    assert d.adj_ids.shape[0] == 2
    assert set(d.neighbors(0)) == {1} and set(d.neighbors(1)) == {0}
    with pytest.raises(ValueError):
        build_drm(base.model, base.checker(), base.lower, base.upper, 1, 1, 1.0, 1.0, grid)
    with pytest.raises(ValueError):
        build_drm(base.model, base.checker(), base.lower, base.upper, 10, 0, 1.0, 1.0, grid)
