"""Generate golden vectors by running the REFERENCE itself — TEST INFRASTRUCTURE.

Imports the read-only reference package from /root/reference/pkg/src (only
possible in the build container; the GPU box has no /root/reference) and
writes small fixtures to tests/golden/.  The oracle (oracle/ref.py) and the
GPU path are both checked against these files.

    PYTHONDONTWRITEBYTECODE=1 python -m oracle.gen_goldens
"""

from __future__ import annotations

import json
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
REF_SRC = Path("/root/reference/pkg/src")


def _import_reference():
    sys.dont_write_bytecode = True
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import corridor  # noqa: F401

    return corridor


def _to_ref_world(world, C):
    """Convert one of our World objects into a reference World through scene JSON."""
    from paper_2504_10783_b200.scene import save_scene

    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "scene.json"
        save_scene(p, world)
        rw = C.world.load_scene(p)
    if world.vmap is not None:
        occ = frozenset(map(tuple, world.vmap.index_array().tolist()))
        rw = rw.with_vmap(C.world.VoxelMap(world.vmap.origin, world.vmap.side, occ))
    return rw


def _oracle_clearance(world, Q, margin=0.0):
    from oracle.ref import OracleChecker

    return OracleChecker(world, margin).clearance(Q)


def gen_checks(C):
    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.scene import VoxelMap, World

    cases = {
        "franka7": (fx.franka7_world(), 20_000, 0.0),
        "franka7_m02": (fx.franka7_world(), 5_000, 0.02),
        "bimanual14": (fx.bimanual14_world(), 4_000, 0.0),
        "arm3": (fx.arm3_world(), 20_000, 0.0),
    }
    # forest scene: discs + reference-voxelised cloud (point robot)
    centers = fx.forest_centers(7)
    ref_vm = C.world.voxelize_point_cloud(fx.disc_point_cloud(centers), 0.02, np.array([-5.0, -5.0]))
    vm = VoxelMap(ref_vm.origin, ref_vm.side, np.array(sorted(ref_vm.occupied), dtype=np.int64))
    forest = fx.disc_world(centers).with_vmap(vm)
    cases["forest7"] = (forest, 20_000, 0.0)
    for name, (world, n, margin) in cases.items():
        rng = np.random.default_rng(0)
        lo, hi = world.lower, world.upper
        Q = rng.uniform(lo, hi, size=(n, len(lo))).astype(np.float32)
        rw = _to_ref_world(world, C)
        free = rw.checker(margin=margin).check_batch(Q.astype(np.float64))
        clr = _oracle_clearance(world, Q.astype(np.float64), margin)
        extra = {}
        if name == "forest7":
            extra["vox_idx"] = vm.index_array()
        np.savez_compressed(GOLDEN / f"check_{name}.npz", Q=Q, free=free, clearance=clr, margin=margin, **extra)
        print(f"check_{name}: n={n} free={free.mean():.3f} band(1e-5)={np.mean(np.abs(clr) < 1e-5):.2e}")


def gen_fk(C):
    from paper_2504_10783_b200 import fixtures as fx

    out = {}
    for name, world in (("franka7", fx.franka7_world(False)), ("bimanual14", fx.bimanual14_world(False)),
                        ("arm3", fx.arm3_world())):
        rw = _to_ref_world(world, C)
        rng = np.random.default_rng(1)
        Q = rng.uniform(world.lower, world.upper, size=(64, len(world.lower)))
        rots, trans = C.world.fk_batch(rw.model, Q)
        out[f"{name}_Q"] = Q
        out[f"{name}_rot"] = np.stack(rots, axis=1)
        out[f"{name}_trans"] = np.stack(trans, axis=1)
    np.savez_compressed(GOLDEN / "fk.npz", **out)
    print("fk: ok")


def _poly7():
    rng = np.random.default_rng(11)
    from paper_2504_10783_b200.fixtures import HOME7

    lo = np.array([-2.8973, -1.7628, -2.8973, -3.0718, -2.8973, -0.0175, -2.8973])
    hi = np.array([2.8973, 1.7628, 2.8973, -0.0698, 2.8973, 3.7525, 2.8973])
    A = [np.eye(7), -np.eye(7)]
    b = [hi, -lo]
    extra_a = rng.normal(size=(8, 7))
    extra_a /= np.linalg.norm(extra_a, axis=1, keepdims=True)
    extra_b = extra_a @ HOME7 + rng.uniform(0.2, 0.6, size=8)
    return np.vstack(A + [extra_a]), np.concatenate(b + [extra_b]), HOME7


def gen_hnr(C):
    cases = {}
    box2 = C.cpoly.HPolytope.from_bounds(np.zeros(2), np.ones(2))
    cases["box2"] = (box2, np.array([[0.5, 0.5]]), 2000, 30, 9, 0)
    box3 = C.cpoly.HPolytope.from_bounds([-2, 0, 1], [3, 4, 2])
    cases["box3"] = (box3, np.array([[0.0, 2.0, 1.5]]), 600, 15, 77, 0)
    A7, b7, s7 = _poly7()
    p7 = C.cpoly.HPolytope(A7, b7)
    cases["poly7"] = (p7, s7[None, :], 1000, 60, 5, 123)
    out = {}
    for name, (poly, seeds, count, n_ms, seed, off) in cases.items():
        sb = C.cpoly.hit_and_run_sample(poly, seeds, count, n_ms, seed, off)
        out[f"{name}_A"] = poly.A
        out[f"{name}_b"] = poly.b
        out[f"{name}_seeds"] = seeds
        out[f"{name}_meta"] = np.array([count, n_ms, seed, off], dtype=np.int64)
        out[f"{name}_X"] = sb.points
    np.savez_compressed(GOLDEN / "hnr.npz", **out)
    print("hnr: ok")


def gen_inflate(C):
    from paper_2504_10783_b200 import fixtures as fx

    records = []
    arm = fx.arm3_world()
    rarm = _to_ref_world(arm, C)
    v1, v2 = fx.ARM3_SEGMENT
    dom = C.cpoly.HPolytope.from_bounds(arm.lower, arm.upper)
    for seed in (0, 1, 2):
        rep = C.inflation.inflate_edge(C.inflation.Segment(v1, v2), dom, C.inflation.InflationParams(),
                                       rarm.checker(), seed=seed)
        records.append(("arm3", seed, {}, v1, v2, rep))
    disc_cases = [("disc_0_3", [[0.0, 3.0]], 1.0, 0, {}), ("disc_0_2", [[0.0, 2.0]], 0.6, 11, {}),
                  ("disc_two", [[0.0, 2.0], [0.0, -2.0]], 0.7, 2, {}),
                  ("disc_nit", [[0.0, 1.2], [0.0, -1.2], [2.0, 1.2]], 0.5, 5, {"n_it": 1})]
    for name, centers, radius, seed, kw in disc_cases:
        w = fx.disc_world(centers, radius)
        rw = _to_ref_world(w, C)
        dom2 = C.cpoly.HPolytope.from_bounds([-5, -5], [5, 5])
        a, bb = np.array([-1.0, 0.0]), np.array([1.0, 0.0])
        rep = C.inflation.inflate_edge(C.inflation.Segment(a, bb), dom2, C.inflation.InflationParams(**kw),
                                       rw.checker(), seed=seed)
        records.append((name, seed, kw, a, bb, rep))
    out = {}
    index = []
    for name, seed, kw, a, bb, rep in records:
        key = f"{name}_s{seed}"
        index.append({"key": key, "scene": name, "seed": seed, "params": kw, "iterations": rep.iterations,
                      "hyperplanes_added": rep.hyperplanes_added, "collision_checks": rep.collision_checks,
                      "terminated_by": rep.terminated_by})
        out[f"{key}_A"] = rep.polytope.A
        out[f"{key}_b"] = rep.polytope.b
        out[f"{key}_v"] = np.stack([a, bb])
        print(f"inflate {key}: it={rep.iterations} faces={rep.hyperplanes_added} checks={rep.collision_checks}")
    out["index"] = np.array(json.dumps(index))
    np.savez_compressed(GOLDEN / "inflate.npz", **out)


def gen_voxelize(C):
    rng = np.random.default_rng(5)
    out = {}
    pts3 = rng.normal(size=(20_000, 3)) * 0.3
    pts3[:50] = np.round(pts3[:50] / 0.02) * 0.02  # exactly on bin boundaries
    org3 = np.array([-1.0, -1.0, -1.0])
    vm3 = C.world.voxelize_point_cloud(pts3, 0.02, org3)
    out["p3"], out["o3"], out["idx3"] = pts3, org3, np.array(sorted(vm3.occupied), dtype=np.int64)
    pts2 = rng.uniform(-2, 2, size=(5_000, 2))
    pts2[:10] = np.array([[1.0, 0.2]] * 10)
    org2 = np.zeros(2)
    vm2 = C.world.voxelize_point_cloud(pts2, 0.5, org2)
    out["p2"], out["o2"], out["idx2"] = pts2, org2, np.array(sorted(vm2.occupied), dtype=np.int64)
    np.savez_compressed(GOLDEN / "voxelize.npz", **out)
    print(f"voxelize: {out['idx3'].shape[0]} / {out['idx2'].shape[0]} voxels")


def gen_drm(C):
    from paper_2504_10783_b200 import fixtures as fx

    out = {}
    # 2-D forest roadmap of the reference tests (test_drm.py:15-23)
    grid = C.drm.Grid(np.array([-5.0, -5.0]), 0.25, (40, 40))
    base = C.world.World(C.bench.point_robot_model())
    d2 = C.drm.build_drm(base.model, base.checker(), base.lower, base.upper, 200, 10, 10.0, 10.0, grid, seed=8)
    out["f_off"], out["f_ids"] = d2.cmap_offsets, d2.cmap_ids
    out["f_nodes"], out["f_adj_off"], out["f_adj_ids"], out["f_poses"] = d2.nodes, d2.adj_offsets, d2.adj_ids, d2.poses
    rng = np.random.default_rng(5)
    maps = []
    for case in range(20):
        occ = frozenset((int(rng.integers(0, 40)), int(rng.integers(0, 40))) for _ in range(rng.integers(1, 30)))
        vm = C.world.VoxelMap(grid.origin, grid.side, occ)
        blocked = np.array(sorted(C.drm.collision_set(d2, vm).blocked), dtype=np.int64)
        maps.append((np.array(sorted(occ), dtype=np.int64), grid.origin, grid.side, blocked))
    fine = C.world.VoxelMap(grid.origin, 0.1, frozenset({(3, 3), (24, 17)}))
    maps.append((np.array(sorted(fine.occupied), dtype=np.int64), fine.origin, 0.1,
                 np.array(sorted(C.drm.collision_set(d2, fine).blocked), dtype=np.int64)))
    for i, (idx, org, side, blocked) in enumerate(maps):
        out[f"f{i}_idx"], out[f"f{i}_org"], out[f"f{i}_side"], out[f"f{i}_blocked"] = idx, org, side, blocked
    out["f_nmaps"] = len(maps)
    # 3-D Franka roadmap on the config-5 grid (small node count)
    w7 = fx.franka7_world(False)
    rw7 = _to_ref_world(w7, C)
    g3 = C.drm.Grid(np.array([-0.75, -1.02, -0.36]), 0.06, (25, 34, 26))
    d3 = C.drm.build_drm(rw7.model, rw7.checker(), rw7.model.lower, rw7.model.upper, 300, 10, 10.0, 10.0, g3, seed=0)
    out["g_nodes"], out["g_off"], out["g_ids"] = d3.nodes, d3.cmap_offsets, d3.cmap_ids
    out["g_adj_off"], out["g_adj_ids"], out["g_poses"] = d3.adj_offsets, d3.adj_ids, d3.poses
    # a build with binding d_cs / d_ts filters (drm.py:226-229) and a small k
    d4 = C.drm.build_drm(rw7.model, rw7.checker(), rw7.model.lower, rw7.model.upper, 400, 4, 2.5, 0.35, g3, seed=5)
    out["h_nodes"], out["h_adj_off"], out["h_adj_ids"], out["h_poses"] = d4.nodes, d4.adj_offsets, d4.adj_ids, d4.poses
    out["h_off"], out["h_ids"] = d4.cmap_offsets, d4.cmap_ids
    cloud = fx.cloud10k()
    pts = cloud.centers()
    vm_same = C.world.voxelize_point_cloud(pts, 0.06, g3.origin)
    vm_fine = C.world.voxelize_point_cloud(pts[::7], 0.02, np.array([-1.0, -1.0, 0.0]))
    for tag, vm in (("same", vm_same), ("fine", vm_fine)):
        out[f"g_{tag}_idx"] = np.array(sorted(vm.occupied), dtype=np.int64)
        out[f"g_{tag}_org"], out[f"g_{tag}_side"] = vm.origin, vm.side
        out[f"g_{tag}_blocked"] = np.array(sorted(C.drm.collision_set(d3, vm).blocked), dtype=np.int64)
        print(f"drm franka {tag}: {len(vm.occupied)} voxels -> {out[f'g_{tag}_blocked'].shape[0]} blocked")
    np.savez_compressed(GOLDEN / "drm.npz", **out)


def gen_corridor(C):
    """inflate_path + refine_sets (planner.py:103-224) on a Forest disc world."""
    import corridor.planner as PL
    from paper_2504_10783_b200 import fixtures as fx

    centers = fx.forest_centers(7003)
    world = fx.disc_world(centers)
    rw = _to_ref_world(world, C)
    ck = rw.checker(margin=0.05)
    rng = np.random.default_rng(12)
    knots = [np.array([1.2, 0.6])]
    while len(knots) < 5:  # chained free segments (margin 0.05, step 0.01), length 1.0..1.5
        d = rng.normal(size=2)
        d /= np.linalg.norm(d)
        nxt = knots[-1] + d * rng.uniform(1.0, 1.5)
        if np.all(np.abs(nxt) < 4.6) and ck.check_segment(knots[-1], nxt, 0.01):
            knots.append(nxt)
    path = C.drm.PwlPath(np.array(knots))
    dom = C.cpoly.HPolytope.from_bounds([-5, -5], [5, 5])
    # a capped inflation (n_it=1, n_f=3) leaves collisions inside the sets for the repair
    params = C.inflation.InflationParams(n_it=1, n_f=2)
    scs = PL.inflate_path(path, dom, params, rw.checker(), seed=21)
    pts = np.random.default_rng(5).uniform(-5, 5, size=(400_000, 2))
    cols = []
    for j, P in enumerate(scs.sets):
        inside = pts[P.contains_many(pts)]
        for c in inside[~rw.checker().check_batch(inside)][:4]:
            cols.append((j, c))
    col = [c for _, c in cols]
    assert cols, "no collisions inside the capped sets"
    ref = PL.refine_sets(scs, cols, path, params, rw.checker(), seed=9)
    out = {"knots": path.knots, "centers": centers, "n_cols": len(cols), "cols": np.array(col),
           "col_sets": np.array([j for j, _ in cols]),
           "n_sets": len(scs.sets), "coverage": np.array(scs.coverage),
           "r_n_sets": len(ref.sets), "r_coverage": np.array(ref.coverage)}
    for i, Pi in enumerate(scs.sets):
        out[f"set{i}_A"], out[f"set{i}_b"] = Pi.A, Pi.b
    for i, Pi in enumerate(ref.sets):
        out[f"rset{i}_A"], out[f"rset{i}_b"] = Pi.A, Pi.b
    np.savez_compressed(GOLDEN / "corridor.npz", **out)
    print(f"corridor: {len(scs.sets)} sets (coverage {scs.coverage}), {len(cols)} collisions -> "
          f"{len(ref.sets)} sets after repair")


def gen_boxes(C):
    """Robot box geometries (world.py:538-565): flags from the reference; the contact band is where the
    reference's own flags change between margin -1e-5 and +1e-5."""
    from oracle.make_scenes import box_arm2d, box_arm3d
    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.model import BOX, SPHERE, Geometry, RigidTransform
    from paper_2504_10783_b200.scene import VoxelMap, World

    table = Geometry(BOX, RigidTransform.planar(0.0, -0.2), half_extents=np.array([2.5, 0.1]))
    disc = Geometry(SPHERE, RigidTransform.planar(0.9, 1.2), radius=0.15)
    tilted = Geometry(BOX, RigidTransform.planar(-0.9, 1.1, 0.5), half_extents=np.array([0.2, 0.1]))
    vm2 = VoxelMap(np.array([-2.3, -0.4]), 0.08, [(12, 20), (13, 20), (12, 21), (40, 22), (41, 23)])
    w2 = World(box_arm2d(), static=(table, disc, tilted), vmap=vm2)
    stat3 = Geometry(BOX, RigidTransform(np.eye(3), np.array([0.5, 0.0, -0.05])), half_extents=np.array([0.6, 0.6, 0.05]))
    w3 = World(box_arm3d(), static=(stat3,), vmap=fx.cloud10k())
    m3 = box_arm3d()
    from paper_2504_10783_b200.model import RobotModel
    m3n = RobotModel(3, m3.joints, m3.links, m3.lower, m3.upper, ())
    w3n = World(m3n, static=(stat3,), vmap=fx.cloud10k())
    import os

    only = os.environ.get("EZ_GOLDEN_ONLY")
    for name, world, n in (("box2d", w2, 20_000), ("box3d", w3, 10_000), ("box3d_noself", w3n, 2_000)):
        if only and name not in only.split(","):
            continue
        rng = np.random.default_rng(0)
        Q = rng.uniform(world.lower, world.upper, size=(n, len(world.lower))).astype(np.float32)
        rw = _to_ref_world(world, C)
        Qd = Q.astype(np.float64)
        free = rw.checker().check_batch(Qd)
        lo = rw.checker(margin=-1e-5).check_batch(Qd)
        hi = rw.checker(margin=1e-5).check_batch(Qd)
        band = lo != hi
        from paper_2504_10783_b200.scene import save_scene
        save_scene(GOLDEN / f"scene_{name}.json", world)
        extra = {"vox_idx": world.vmap.index_array(), "vox_origin": world.vmap.origin, "vox_side": world.vmap.side}
        np.savez_compressed(GOLDEN / f"check_{name}.npz", Q=Q, free=free, band=band, margin=0.0, **extra)
        print(f"check_{name}: n={n} free={free.mean():.3f} band={band.mean():.2e}")


def _ref_free_segment(world, rw, seed, length=0.6, margin=0.02, step=0.01, inner=0.3):
    """fixtures.random_free_segment's rejection sampling, every check by the REFERENCE checker
    (world.py:479-501).  The GPU tests assert that fixtures.random_free_segment (GPU checker)
    finds the same segment, which pins the benchmark segments themselves."""
    ck = rw.checker(margin=margin)
    rng = np.random.default_rng(seed)
    lo, hi = world.lower, world.upper
    while True:
        v1 = rng.uniform(lo + inner * (hi - lo), hi - inner * (hi - lo))
        if not ck.check(v1):
            continue
        d = rng.normal(size=v1.shape[0])
        d /= np.linalg.norm(d)
        v2 = v1 + d * length
        if np.all(v2 > lo) and np.all(v2 < hi) and ck.check_segment(v1, v2, step):
            return v1, v2


def _ref_check_chunk(args):
    """Worker: the reference's own check_batch on one chunk (batch == sequential is a
    reference-tested property, test_world.py:129-139)."""
    scene_path, vox_idx, vox_origin, vox_side, Q = args
    C = _import_reference()
    rw = C.world.load_scene(scene_path)
    occ = frozenset(map(tuple, vox_idx.tolist()))
    rw = rw.with_vmap(C.world.VoxelMap(vox_origin, vox_side, occ))
    return rw.checker().check_batch(Q)


def gen_config2(C):
    """Config 2 at full size: the reference's flags on the benchmark's 2^20 fp32 rows, computed by
    the reference's check_batch in 8 worker processes; the oracle's fp64 clearance marks the
    1e-5 contact band, and the oracle's flags must equal the reference's on every row."""
    import multiprocessing as mp
    import os
    import time

    from oracle.ref import OracleChecker
    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.scene import save_scene

    world = fx.franka7_world()
    Q = fx.config2_rows().astype(np.float64)
    with tempfile.TemporaryDirectory() as td:
        p = str(Path(td) / "scene.json")
        save_scene(p, world)
        vm = world.vmap
        chunks = np.array_split(Q, 64)
        t0 = time.perf_counter()
        ctx = mp.get_context("fork")
        with ctx.Pool(os.cpu_count()) as pool:
            parts = pool.map(_ref_check_chunk, [(p, vm.index_array(), vm.origin, vm.side, c) for c in chunks])
        free = np.concatenate(parts)
        t_ref = time.perf_counter() - t0
    oc = OracleChecker(world, workers=os.cpu_count())
    clr = np.concatenate([oc.clearance(c) for c in np.array_split(Q, 64)])
    assert np.array_equal(free, clr > 0) or np.all(np.abs(clr[free != (clr > 0)]) < 1e-12)
    band = np.flatnonzero(np.abs(clr) < 1e-5).astype(np.int64)
    np.savez_compressed(GOLDEN / "config2_1m.npz", free_bits=np.packbits(free), n=Q.shape[0], seed=0, band=band,
                        ref_seconds=t_ref)
    print(f"config2_1m: n={Q.shape[0]} free={free.mean():.4f} band={band.size} reference {t_ref:.0f}s "
          f"on {os.cpu_count()} processes")


def gen_region7(C):
    """The benchmark's 7-DOF EI-ZO region (BASELINE config 2/3 segment, seed 7) computed by the
    reference's inflate_edge (inflation.py:262-325), plus the config-4 (14-DOF) segment."""
    import time

    from paper_2504_10783_b200 import fixtures as fx

    w7 = fx.franka7_world()
    rw7 = _to_ref_world(w7, C)
    v1, v2 = _ref_free_segment(w7, rw7, seed=3)
    dom = C.cpoly.HPolytope.from_bounds(w7.lower, w7.upper)
    params = C.inflation.InflationParams(**fx.FRANKA_PARAMS)
    t0 = time.perf_counter()
    rep = C.inflation.inflate_edge(C.inflation.Segment(v1, v2), dom, params, rw7.checker(), seed=7)
    dt = time.perf_counter() - t0
    w14 = fx.bimanual14_world()
    rw14 = _to_ref_world(w14, C)
    u1, u2 = _ref_free_segment(w14, rw14, seed=3)
    np.savez_compressed(GOLDEN / "region7.npz", v1=v1, v2=v2, A=rep.polytope.A, b=rep.polytope.b,
                        iterations=rep.iterations, hyperplanes_added=rep.hyperplanes_added,
                        collision_checks=rep.collision_checks, terminated_by=rep.terminated_by,
                        ref_seconds=dt, seg14_v1=u1, seg14_v2=u2)
    print(f"region7: it={rep.iterations} faces={rep.hyperplanes_added} checks={rep.collision_checks} "
          f"in {dt:.1f}s (reference, 1 process)")


def gen_criterion3(C):
    """Acceptance criterion 3 (test_acceptance.py:96-131) as the reference runs it: 100 Forest
    inflations (delta=0.05, eps=0.01), each audited with 5e4 rejection samples.  Stores every
    segment, polytope, counter and audited fraction."""
    import time

    from corridor.seeding import child_seed

    domain = C.cpoly.HPolytope.from_bounds([-5, -5], [5, 5])
    params = C.inflation.InflationParams(delta=0.05, eps=0.01)
    out = {}
    recs = []
    t0 = time.perf_counter()
    for run in range(100):
        scene = C.bench.gen_forest(7000 + run)
        discs = tuple(C.world.Geometry(C.world.SPHERE, C.world.RigidTransform.planar(c[0], c[1]), radius=scene.radius)
                      for c in scene.centers)
        world = C.world.World(C.bench.point_robot_model(), static=discs)
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
        rep = C.inflation.inflate_edge(C.inflation.Segment(v1, v2), domain, params, world.checker(),
                                       seed=child_seed(77, run))
        poly = rep.polytope
        mc = np.random.default_rng(child_seed(99, run))
        kept, need = [], 50_000
        while need > 0:
            draw = mc.uniform(-5, 5, size=(200_000, 2))
            take = draw[poly.contains_many(draw)][:need]
            kept.append(take)
            need -= take.shape[0]
        frac = float(np.mean(~world.checker().check_batch(np.concatenate(kept))))
        out[f"r{run}_A"], out[f"r{run}_b"], out[f"r{run}_v"] = poly.A, poly.b, np.stack([v1, v2])
        out[f"r{run}_centers"] = scene.centers
        recs.append([rep.iterations, rep.hyperplanes_added, rep.collision_checks,
                     int(rep.terminated_by == "test_accepted"), child_seed(77, run)])
        out[f"r{run}_frac"] = frac
    out["recs"] = np.array(recs, dtype=np.uint64)
    out["radius"] = scene.radius
    exceed = sum(float(out[f"r{r}_frac"]) > 0.01 for r in range(100))
    np.savez_compressed(GOLDEN / "criterion3.npz", **out)
    print(f"criterion3: {exceed}/100 exceed eps in {time.perf_counter() - t0:.0f}s")


def oblique_world():
    """Revolute, 3-D prismatic and oblique-axis joints (Rodrigues about a non-z axis, world.py:64-69,
    174-192) among a static sphere, a static box and the 10k-voxel cloud."""
    from oracle.make_scenes import pose
    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.model import (BOX, PRISMATIC, REVOLUTE, SPHERE, Geometry, Joint, Link,
                                             RigidTransform, RobotModel)
    from paper_2504_10783_b200.scene import World

    sph = lambda *p: Geometry(SPHERE, pose(p), radius=0.06)  # noqa: E731
    joints = (Joint(REVOLUTE, -1, pose((-0.2, 0.0, 0.2)), axis=np.array([0.0, 0.0, 1.0])),
              Joint(PRISMATIC, 0, pose((0.0, 0.0, 0.3), (0.3, 0.0, 0.0)), axis=np.array([0.3, 0.2, 0.93])),
              Joint(REVOLUTE, 1, pose((0.2, 0.0, 0.1), (0.0, 0.4, 0.0)), axis=np.array([0.6, -0.64, 0.48])),
              Joint(REVOLUTE, 2, pose((0.45, 0.0, 0.0), (0.2, -0.3, 0.5)), axis=np.array([-0.36, 0.48, 0.8])))
    links = (Link((sph(0, 0, 0.1), sph(0, 0, 0.25))), Link((sph(0, 0, 0), sph(0.1, 0, 0))),
             Link((sph(0.15, 0, 0), sph(0.3, 0, 0), sph(0.45, 0.05, 0))),
             Link((sph(0.1, 0, 0), sph(0.2, 0.02, 0.05))))
    model = RobotModel(3, joints, links, np.array([-3.0, -0.2, -3.0, -3.0]), np.array([3.0, 0.6, 3.0, 3.0]),
                       ((0, 5), (0, 6), (1, 6), (0, 7), (0, 8), (1, 8), (2, 8)))
    base = fx.franka7_world()
    static = (Geometry(SPHERE, RigidTransform(np.eye(3), np.array([-0.5, 0.2, 0.6])), radius=0.1),
              Geometry(BOX, RigidTransform(np.eye(3), np.array([0.3, -0.4, 0.2])), half_extents=np.array([0.1, 0.2, 0.15])))
    return World(model, static, base.vmap, model.lower, model.upper)


def gen_oblique(C):
    """Oblique revolute axes and a 3-D prismatic joint: the reference's FK and flags."""
    w = oblique_world()
    rw = _to_ref_world(w, C)
    rng = np.random.default_rng(4)
    Q = rng.uniform(w.lower, w.upper, size=(20_000, w.model.dof)).astype(np.float32)
    Qd = Q.astype(np.float64)
    free = rw.checker().check_batch(Qd)
    clr = _oracle_clearance(w, Qd)
    Qf = rng.uniform(w.lower, w.upper, size=(64, w.model.dof))
    rots, trans = C.world.fk_batch(rw.model, Qf)
    np.savez_compressed(GOLDEN / "check_oblique.npz", Q=Q, free=free, clearance=clr, margin=0.0,
                        fk_Q=Qf, fk_rot=np.stack(rots, axis=1), fk_trans=np.stack(trans, axis=1))
    print(f"check_oblique: free={free.mean():.3f} band={np.mean(np.abs(clr) < 1e-5):.2e}")


def main(which=None):
    GOLDEN.mkdir(parents=True, exist_ok=True)
    C = _import_reference()
    import corridor.bench, corridor.cpoly, corridor.drm, corridor.inflation, corridor.world  # noqa: E401,F401

    steps = {"checks": gen_checks, "fk": gen_fk, "hnr": gen_hnr, "inflate": gen_inflate,
             "voxelize": gen_voxelize, "drm": gen_drm, "corridor": gen_corridor, "boxes": gen_boxes,
             "config2": gen_config2, "region7": gen_region7, "criterion3": gen_criterion3,
             "oblique": gen_oblique}
    for name, fn in steps.items():
        if which and name not in which:
            continue
        fn(C)


if __name__ == "__main__":
    main(sys.argv[1:] or None)
