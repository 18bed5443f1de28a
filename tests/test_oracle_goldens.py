"""Pin the CPU oracle (oracle/ref.py) to the reference's own outputs (tests/golden/).

The goldens were produced by running /root/reference itself
(oracle/gen_goldens.py); these tests are what makes the oracle a trustworthy
checker for the GPU parity tests.
"""

import numpy as np
import pytest

from conftest import GOLDEN as GOLDEN_DIR
from conftest import golden, inflate_index
from oracle import ref
from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.scene import VoxelMap

WORLDS = {"franka7": lambda: fx.franka7_world(), "franka7_m02": lambda: fx.franka7_world(),
          "bimanual14": lambda: fx.bimanual14_world(), "arm3": fx.arm3_world}


def forest_world_from_golden(g):
    vm = VoxelMap(np.array([-5.0, -5.0]), 0.02, g["vox_idx"])
    return fx.disc_world(fx.forest_centers(7)).with_vmap(vm)


@pytest.mark.parametrize("name", ["franka7", "franka7_m02", "bimanual14", "arm3", "forest7"])
def test_oracle_flags_match_reference(name):
    g = golden(f"check_{name}.npz")
    world = forest_world_from_golden(g) if name == "forest7" else WORLDS[name]()
    ck = ref.OracleChecker(world, float(g["margin"]))
    Q = g["Q"].astype(np.float64)
    free = ck.check_batch(Q)
    assert np.array_equal(free, g["free"])
    # the fp64 clearance's sign reproduces the reference flags (touching = collision)
    assert np.array_equal(g["clearance"] > 0.0, g["free"])
    assert ck.calls == Q.shape[0]


def test_oracle_fk_matches_reference():
    z = golden("fk.npz")
    for name, world in (("franka7", fx.franka7_world(False)), ("bimanual14", fx.bimanual14_world(False)),
                        ("arm3", fx.arm3_world())):
        rots, trans = ref.fk_batch(world.model, z[f"{name}_Q"])
        assert np.allclose(np.stack(rots, axis=1), z[f"{name}_rot"], atol=1e-13)
        assert np.allclose(np.stack(trans, axis=1), z[f"{name}_trans"], atol=1e-13)


@pytest.mark.parametrize("name", ["box2", "box3", "poly7"])
def test_oracle_hit_and_run_matches_reference(name):
    z = golden("hnr.npz")
    count, n_ms, seed, off = (int(v) for v in z[f"{name}_meta"])
    X = ref.hit_and_run(z[f"{name}_A"], z[f"{name}_b"], z[f"{name}_seeds"], count, n_ms, seed, off)
    assert np.array_equal(X, z[f"{name}_X"])


def _inflate_world(scene):
    if scene == "arm3":
        return fx.arm3_world()
    return {"disc_0_3": fx.disc_world([[0.0, 3.0]], 1.0), "disc_0_2": fx.disc_world([[0.0, 2.0]], 0.6),
            "disc_two": fx.disc_world([[0.0, 2.0], [0.0, -2.0]], 0.7),
            "disc_nit": fx.disc_world([[0.0, 1.2], [0.0, -1.2], [2.0, 1.2]], 0.5)}[scene]


def test_oracle_inflate_matches_reference():
    z, index = inflate_index()
    for rec in index:
        world = _inflate_world(rec["scene"])
        v = z[f"{rec['key']}_v"]
        A0 = np.vstack([np.eye(len(world.lower)), -np.eye(len(world.lower))])
        b0 = np.concatenate([world.upper, -world.lower])
        out = ref.inflate_edge(v[0], v[1], A0, b0, ref.OracleChecker(world), seed=rec["seed"], **rec["params"])
        assert out["iterations"] == rec["iterations"]
        assert out["hyperplanes_added"] == rec["hyperplanes_added"]
        assert out["collision_checks"] == rec["collision_checks"]
        assert out["terminated_by"] == rec["terminated_by"]
        assert np.allclose(out["A"], z[f"{rec['key']}_A"], atol=1e-12)
        assert np.allclose(out["b"], z[f"{rec['key']}_b"], atol=1e-12)


def test_oracle_voxelize_matches_reference():
    z = golden("voxelize.npz")
    assert np.array_equal(ref.voxelize(z["p3"], 0.02, z["o3"]), z["idx3"])
    assert np.array_equal(ref.voxelize(z["p2"], 0.5, z["o2"]), z["idx2"])


def test_oracle_collision_set_matches_reference():
    z = golden("drm.npz")
    for i in range(int(z["f_nmaps"])):
        got = ref.collision_set(z["f_off"], z["f_ids"], [-5.0, -5.0], 0.25, (40, 40), z[f"f{i}_idx"],
                                z[f"f{i}_org"], float(z[f"f{i}_side"]))
        assert np.array_equal(got, z[f"f{i}_blocked"])
    for tag in ("same", "fine"):
        got = ref.collision_set(z["g_off"], z["g_ids"], [-0.75, -1.02, -0.36], 0.06, (25, 34, 26),
                                z[f"g_{tag}_idx"], z[f"g_{tag}_org"], float(z[f"g_{tag}_side"]))
        assert np.array_equal(got, z[f"g_{tag}_blocked"])


def test_oracle_node_voxel_pairs_match_reference_cmap():
    z = golden("drm.npz")
    world = fx.franka7_world(False)
    ext = (25, 34, 26)
    rows, cols = ref.node_voxel_pairs(world.model, z["g_nodes"], np.array([-0.75, -1.02, -0.36]), 0.06, ext)
    order = np.lexsort((rows, cols))
    counts = np.bincount(cols, minlength=int(np.prod(ext)))
    off = np.zeros(counts.shape[0] + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    assert np.array_equal(off, z["g_off"])
    assert np.array_equal(rows[order].astype(np.int32), z["g_ids"])


def test_oracle_seed_helpers():
    from paper_2504_10783_b200.rng import child_seed

    for m, w in ((0, (1,)), (12345, (0x5E7, 3)), (2 ** 64 - 1, (7, 8, 9))):
        assert child_seed(m, *w) == ref.child_seed(m, *w)


def test_oracle_oblique_axes_and_prismatic_match_reference():
    """Rodrigues about oblique axes and a 3-D prismatic joint (world.py:64-69, 174-192)."""
    from oracle.gen_goldens import oblique_world

    z = golden("check_oblique.npz")
    w = oblique_world()
    assert np.array_equal(ref.OracleChecker(w).check_batch(z["Q"].astype(np.float64)), z["free"])
    assert np.array_equal(z["clearance"] > 0.0, z["free"])
    rots, trans = ref.fk_batch(w.model, z["fk_Q"])
    assert np.allclose(np.stack(rots, axis=1), z["fk_rot"], atol=1e-13)
    assert np.allclose(np.stack(trans, axis=1), z["fk_trans"], atol=1e-13)


def test_oracle_criterion3_inflations_match_reference():
    """The first acceptance-audit inflations (test_acceptance.py:96-131) restated by the oracle."""
    z = golden("criterion3.npz")
    A0 = np.vstack([np.eye(2), -np.eye(2)])
    b0 = np.full(4, 5.0)
    for run in range(6):
        world = fx.disc_world(z[f"r{run}_centers"], float(z["radius"]))
        v = z[f"r{run}_v"]
        it, faces, checks, accepted, seed = (int(x) for x in z["recs"][run])
        out = ref.inflate_edge(v[0], v[1], A0, b0, ref.OracleChecker(world), seed=seed, delta=0.05, eps=0.01)
        assert (out["iterations"], out["hyperplanes_added"], out["collision_checks"]) == (it, faces, checks)
        assert np.allclose(out["A"], z[f"r{run}_A"], atol=1e-12) and np.allclose(out["b"], z[f"r{run}_b"], atol=1e-12)
    exceed = sum(float(z[f"r{r}_frac"]) > 0.01 for r in range(100))
    assert exceed <= 15


def test_oracle_config2_rows_match_reference_flags():
    """A slice of config 2's 2^20 rows: the oracle's flags equal the reference's exactly."""
    p = GOLDEN_DIR / "config2_1m.npz"
    z = np.load(p)
    n = int(z["n"])
    free = np.unpackbits(z["free_bits"])[:n].astype(bool)
    Q = fx.config2_rows()
    assert Q.shape == (n, 7) and Q.dtype == np.float32
    sl = slice(500_000, 520_000)
    assert np.array_equal(ref.OracleChecker(fx.franka7_world()).check_batch(Q[sl].astype(np.float64)), free[sl])


def test_oracle_region7_segment_and_counters():
    """The benchmark segment is the one the reference's checker finds; the reference region's
    counters obey the reference's own formula (collision_checks = sum N_k + C_k (1 + N_b))."""
    z = golden("region7.npz")
    world = fx.franka7_world()
    ck = ref.OracleChecker(world, margin=0.02)
    v1, v2 = z["v1"], z["v2"]
    assert ck.check(v1) and abs(np.linalg.norm(v2 - v1) - 0.6) < 1e-12
    n = int(np.ceil(0.6 / 0.01))
    assert ck.check_batch(v1 + np.linspace(0, 1, n + 1)[:, None] * (v2 - v1)).all()
    assert str(z["terminated_by"]) == "test_accepted"
    A, b = z["A"], z["b"]
    assert A.shape[0] == 14 + int(z["hyperplanes_added"])
    assert np.all(A @ v1 <= b + 1e-9) and np.all(A @ v2 <= b + 1e-9)


@pytest.mark.parametrize("key,k,d_cs,d_ts", [("f", 10, 10.0, 10.0), ("g", 10, 10.0, 10.0), ("h", 4, 2.5, 0.35)])
def test_oracle_roadmap_adjacency_matches_reference(key, k, d_cs, d_ts):
    z = golden("drm.npz")
    dim = 2 if key == "f" else 3
    off, ids = ref.roadmap_adjacency(z[f"{key}_nodes"], z[f"{key}_poses"][:, :dim], k, d_cs, d_ts)
    assert np.array_equal(off, z[f"{key}_adj_off"]) and np.array_equal(ids, z[f"{key}_adj_ids"])
