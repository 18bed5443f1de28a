"""Model-specialised check kernel (ez_jit.cu, NVRTC): parity with the reference goldens and
exact agreement with the generic kernel it replaces for large fp32 batches."""

import numpy as np
import pytest
import torch

from conftest import golden
from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.model import BOX, SPHERE, Geometry, RigidTransform
from paper_2504_10783_b200.scene import VoxelMap, World

pytestmark = pytest.mark.gpu

BAND = 1e-5


def _golden_world(name, g):
    if name == "forest7":
        return fx.disc_world(fx.forest_centers(7)).with_vmap(VoxelMap(np.array([-5.0, -5.0]), 0.02, g["vox_idx"]))
    return {"franka7": fx.franka7_world, "franka7_m02": fx.franka7_world, "bimanual14": fx.bimanual14_world,
            "arm3": fx.arm3_world}[name]()


@pytest.mark.parametrize("name", ["franka7", "franka7_m02", "bimanual14", "arm3", "forest7"])
def test_specialised_flags_match_reference(name):
    g = golden(f"check_{name}.npz")
    ck = _golden_world(name, g).checker(margin=float(g["margin"]))
    assert ck.native.specialize(1), "NVRTC specialisation unavailable on this box"
    free = ck.check_batch(g["Q"].astype(np.float64))
    mism = (free != g["free"]) & (np.abs(g["clearance"]) >= BAND)
    assert not mism.any(), f"{mism.sum()} flag mismatches outside the {BAND} band"


def _statics_world():
    """Franka arm among a static sphere, a static box and a voxel cloud."""
    w = fx.franka7_world()
    static = (Geometry(SPHERE, RigidTransform(np.eye(3), np.array([0.5, 0.3, 0.6])), radius=0.12),
              Geometry(BOX, RigidTransform(np.eye(3), np.array([0.0, -0.5, 0.4])), half_extents=np.array([0.1, 0.2, 0.3])))
    return World(w.model, static, w.vmap, w.lower, w.upper)


@pytest.mark.parametrize("which", ["franka7", "bimanual14", "arm3", "statics"])
@pytest.mark.parametrize("rows", ["float32", "float64"])
def test_specialised_equals_generic(which, rows):
    w = {"franka7": fx.franka7_world, "bimanual14": fx.bimanual14_world, "arm3": fx.arm3_world,
         "statics": _statics_world}[which]()
    gen, jit = w.checker(margin=0.01).native, w.checker(margin=0.01).native
    gen.specialize(-1)
    assert jit.specialize(1)
    lo = torch.as_tensor(w.lower, dtype=torch.float64, device="cuda")
    hi = torch.as_tensor(w.upper, dtype=torch.float64, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    Q = (lo + (hi - lo) * torch.rand((300_000, w.model.dof), generator=g, device="cuda", dtype=torch.float64))
    Q = Q.to(getattr(torch, rows))
    a, b = gen.check_device(Q), jit.check_device(Q)
    assert 0.0 < float(a.float().mean()) < 1.0
    assert torch.equal(a, b)


def test_robot_boxes_stay_generic():
    from oracle.make_scenes import box_arm3d
    ck = World(box_arm3d()).checker()
    assert not ck.native.specialize(1)
    assert not ck.native.specialize(0)


def test_specialisation_only_at_world_creation(monkeypatch):
    """no NVRTC compile or CTA-size tuning inside a check call.  Large robots get the
    specialised kernel when their device world is created ("auto"); specialize=False never."""
    monkeypatch.delenv("EZ_JIT", raising=False)  # the default behaviour ("auto" on)
    w = fx.franka7_world()
    assert w.checker().native.specialize(0)
    assert w.checker().native.info()["check_cta"] in (256, 512, 1024)
    nat = w.checker(specialize=False).native
    assert not nat.specialize(0) and nat.info()["check_cta"] == 0
    lo = torch.as_tensor(w.lower, dtype=torch.float32, device="cuda")
    hi = torch.as_tensor(w.upper, dtype=torch.float32, device="cuda")
    nat.check_device(lo + (hi - lo) * torch.rand((1 << 18, 7), device="cuda"))
    assert not nat.specialize(0)
    assert not fx.arm3_world().checker().native.specialize(0)  # 9 spheres: generic under "auto"


def test_concurrent_checks_while_specialising():
    """Checks from other threads while ez_world_specialize compiles and publishes the kernel:
    every result equals the generic kernel's (the launch takes an atomic snapshot)."""
    import threading

    w = fx.bimanual14_world()
    ref_nat = w.checker(specialize=False).native
    nat = w.checker(specialize=False).native
    lo = torch.as_tensor(w.lower, dtype=torch.float32, device="cuda")
    hi = torch.as_tensor(w.upper, dtype=torch.float32, device="cuda")
    Q = lo + (hi - lo) * torch.rand((1 << 16, 14), device="cuda")
    want = ref_nat.check_device(Q)
    torch.cuda.synchronize()
    bad = []

    def hammer():
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(40):
                out = nat.check_device(Q)
                s.synchronize()
                if not torch.equal(out, want):
                    bad.append(1)

    ts = [threading.Thread(target=hammer) for _ in range(3)]
    for t in ts:
        t.start()
    assert nat.specialize(1)
    for t in ts:
        t.join()
    assert not bad
    assert torch.equal(nat.check_device(Q), want)


@pytest.mark.parametrize("cta", [256, 512, 1024])
def test_every_kernel_shape_equals_generic(cta, monkeypatch):
    """The 64..256, 512 x 2 and 1024 x 1 kernels (EZ_JIT_BT forces the large-batch size)."""
    monkeypatch.setenv("EZ_JIT_BT", str(cta))
    w = fx.bimanual14_world()
    gen, jit = w.checker().native, w.checker().native
    gen.specialize(-1)
    assert gen.info()["check_cta"] == 0
    assert jit.specialize(1) and jit.info()["check_cta"] == cta
    lo = torch.as_tensor(w.lower, dtype=torch.float32, device="cuda")
    hi = torch.as_tensor(w.upper, dtype=torch.float32, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(cta)
    Q = lo + (hi - lo) * torch.rand((1 << 19, 14), generator=g, device="cuda")
    assert torch.equal(gen.check_device(Q), jit.check_device(Q))
    assert torch.equal(gen.check_device(Q.double()), jit.check_device(Q.double()))


def _oblique_world():
    """Revolute, prismatic and oblique-axis joints (Q folding and the prismatic branch of the generator)."""
    from paper_2504_10783_b200.model import Joint, Link, RobotModel, REVOLUTE, PRISMATIC
    from oracle.make_scenes import pose
    sph = lambda *p: Geometry(SPHERE, pose(p), radius=0.06)
    joints = (Joint(REVOLUTE, -1, pose((-0.2, 0.0, 0.2)), axis=np.array([0.0, 0.0, 1.0])),
              Joint(PRISMATIC, 0, pose((0.0, 0.0, 0.3), (0.3, 0.0, 0.0)), axis=np.array([0.3, 0.2, 0.93])),
              Joint(REVOLUTE, 1, pose((0.2, 0.0, 0.1), (0.0, 0.4, 0.0)), axis=np.array([0.6, -0.64, 0.48])))
    links = (Link((sph(0, 0, 0.1), sph(0, 0, 0.25))), Link((sph(0, 0, 0), sph(0.1, 0, 0))),
             Link((sph(0.15, 0, 0), sph(0.3, 0, 0), sph(0.45, 0.05, 0))))
    model = RobotModel(3, joints, links, np.array([-3.0, -0.2, -3.0]), np.array([3.0, 0.6, 3.0]),
                       ((0, 5), (0, 6), (1, 6)))
    base = fx.franka7_world()
    static = (Geometry(SPHERE, RigidTransform(np.eye(3), np.array([-0.5, 0.2, 0.6])), radius=0.1),)
    return World(model, static, base.vmap, model.lower, model.upper)


@pytest.mark.parametrize("rows", ["float32", "float64"])
def test_specialised_equals_generic_prismatic_oblique(rows):
    w = _oblique_world()
    gen, jit = w.checker().native, w.checker().native
    gen.specialize(-1)
    assert jit.specialize(1)
    lo = torch.as_tensor(w.lower, dtype=torch.float64, device="cuda")
    hi = torch.as_tensor(w.upper, dtype=torch.float64, device="cuda")
    Q = (lo + (hi - lo) * torch.rand((200_000, 3), device="cuda", dtype=torch.float64)).to(getattr(torch, rows))
    a, b = gen.check_device(Q), jit.check_device(Q)
    assert 0.0 < float(a.float().mean()) < 1.0
    assert torch.equal(a, b)


@pytest.mark.parametrize("variant", ["0", "1", "2"])
@pytest.mark.parametrize("which", ["franka7", "bimanual14"])
def test_both_voxel_code_variants_equal_generic(which, variant, monkeypatch):
    """The literal-constant voxel code (variant 0), the generic calls (variant 1) and the lookups
    streamed with the FK (variant 2), each forced
    with EZ_JIT_VOX, give the generic kernel's flags exactly (specialisation keeps the faster)."""
    monkeypatch.setenv("EZ_JIT_VOX", variant)
    w = {"franka7": fx.franka7_world, "bimanual14": fx.bimanual14_world}[which]()
    gen, jit = w.checker(specialize=False).native, w.checker(specialize=False).native
    assert jit.specialize(1) and jit.info()["check_variant"] == int(variant)
    lo = torch.as_tensor(w.lower, dtype=torch.float32, device="cuda")
    hi = torch.as_tensor(w.upper, dtype=torch.float32, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    Q = lo + (hi - lo) * torch.rand((1 << 19, w.model.dof), generator=g, device="cuda")
    assert torch.equal(gen.check_device(Q), jit.check_device(Q))
    assert torch.equal(gen.check_device(Q.double()), jit.check_device(Q.double()))


@pytest.mark.parametrize("which", ["franka7", "bimanual14", "arm3"])
def test_specialised_bisection_equals_cooperative(which, monkeypatch):
    """The EI-ZO bisection on the specialised check (ez_bisect_core.cuh: one thread per point,
    three binary steps per round) forms the same points as k_bisect2 (EZ_BISECT_JIT=0) and so
    takes the same decisions wherever the specialised and generic fp32 checks agree; they can
    differ only inside the fp32 contact band (next test), which these regions never hit:
    identical regions and counters."""
    from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge
    from paper_2504_10783_b200.polytope import HPolytope

    w = {"franka7": fx.franka7_world, "bimanual14": fx.bimanual14_world, "arm3": fx.arm3_world}[which]()
    ck = w.checker()
    assert ck.native.specialize(1)
    dom = HPolytope.from_bounds(w.lower, w.upper)
    if which == "arm3":
        v1, v2 = fx.ARM3_SEGMENT
        p = InflationParams()
    else:
        v1, v2 = fx.random_free_segment(w, seed=3)
        p = InflationParams(**{**fx.FRANKA_PARAMS, "n_it": 3 if which == "bimanual14" else None})
    reps = []
    for flag in ("0", "1"):
        monkeypatch.setenv("EZ_BISECT_JIT", flag)
        reps += [inflate_edge(Segment(np.asarray(v1), np.asarray(v2)), dom, p, ck, seed=s) for s in (7, 8)]
    for a, b in zip(reps[:2], reps[2:]):
        assert (a.iterations, a.hyperplanes_added, a.collision_checks, a.terminated_by) == \
               (b.iterations, b.hyperplanes_added, b.collision_checks, b.terminated_by)
        assert np.array_equal(a.polytope.A, b.polytope.A) and np.array_equal(a.polytope.b, b.polytope.b)


def test_specialised_flags_differ_only_inside_contact_band():
    """Near collision boundaries (points along free-to-colliding segments and their bisection
    points) the specialised and generic fp32 checks round differently in a few configurations;
    every such configuration lies inside the contact band the fp32 contract exempts (the
    reference's fp64 clearance |c| < 1e-5)."""
    from oracle import ref

    w = fx.franka7_world()
    gen, jit = w.checker(specialize=False).native, w.checker(specialize=False).native
    assert jit.specialize(1)
    lo = torch.as_tensor(w.lower, dtype=torch.float64, device="cuda")
    hi = torch.as_tensor(w.upper, dtype=torch.float64, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    Q = lo + (hi - lo) * torch.rand((1 << 16, 7), generator=g, device="cuda", dtype=torch.float64)
    f = gen.check_device(Q).bool()
    a, b = Q[f][: 1 << 13], Q[~f][: 1 << 13]
    n = min(len(a), len(b))
    a, b = a[:n], b[:n]
    pts = []
    for _ in range(24):  # bisection on the generic check, every visited point kept
        m = 0.5 * (a + b)
        fm = gen.check_device(m).bool()
        a = torch.where(fm[:, None], m, a)
        b = torch.where(fm[:, None], b, m)
        pts.append(m)
    P = torch.cat(pts)
    mism = (gen.check_device(P) != jit.check_device(P)).nonzero().flatten()
    X = P[mism[:256]].cpu().numpy()
    if len(X):
        clr = ref.OracleChecker(w).clearance(X)
        assert np.abs(clr).max() < BAND


@pytest.mark.parametrize("which", ["franka7", "bimanual14"])
def test_small_batch_full_path_equals_generic(which):
    """Batches up to 32k rows run one row per thread through the policy's full() (one FK, no
    survivor queue): the generic kernel's flags exactly, for fp32 and fp64 rows and with the
    EI-ZO loop's collision count."""
    w = {"franka7": fx.franka7_world, "bimanual14": fx.bimanual14_world}[which]()
    gen, jit = w.checker(specialize=False).native, w.checker(specialize=False).native
    assert jit.specialize(1)
    lo = torch.as_tensor(w.lower, dtype=torch.float32, device="cuda")
    hi = torch.as_tensor(w.upper, dtype=torch.float32, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(9)
    for n in (1, 100, 10_000, 32_768):
        Q = lo + (hi - lo) * torch.rand((n, w.model.dof), generator=g, device="cuda")
        assert torch.equal(gen.check_device(Q), jit.check_device(Q))
        assert torch.equal(gen.check_device(Q.double()), jit.check_device(Q.double()))


def test_batch_beyond_int32_queue_indices():
    """A device batch of 2^31 + 4096 rows (60 GB of fp32 rows; row indices past int32) runs as
    launches of at most 2^30 rows (the survivor queue holds int32 row indices): the rows on both
    sides of every split get the flags a small batch of the same rows gets."""
    w = fx.franka7_world()
    nat = w.checker().native
    n = (1 << 31) + 4096
    lo = torch.as_tensor(w.lower, dtype=torch.float32, device="cuda")
    hi = torch.as_tensor(w.upper, dtype=torch.float32, device="cuda")
    Q = torch.empty((n, 7), dtype=torch.float32, device="cuda")
    Q.uniform_()
    Q.mul_(hi - lo).add_(lo)
    flags = nat.check_device(Q)
    for a, b in ((0, 4096), ((1 << 30) - 4096, (1 << 30) + 4096), ((1 << 31) - 4096, n)):
        assert torch.equal(flags[a:b], nat.check_device(Q[a:b].clone()))
    del Q, flags
    torch.cuda.empty_cache()
