"""Benchmark and test scenes (BASELINE.json configs).

* config 1: the reference's planar three-link table-top arm
  (``corridor/bench.py:120-150``) with three disc obstacles;
* configs 2/3: Franka-like 7-DOF sphere model vs a 10k-voxel cloud
  (``scenes/franka7.json`` + ``scenes/cloud10k.npz``, frozen by
  ``oracle/make_scenes.py``);
* config 4: the 14-DOF bimanual model (``scenes/bimanual14.json``);
* the Forest point-robot scenes (``corridor/bench.py:30-117``).
"""

from __future__ import annotations

import math
from functools import lru_cache
from pathlib import Path

import numpy as np

from .model import BOX, PRISMATIC, REVOLUTE, SPHERE, Geometry, Joint, Link, RigidTransform, RobotModel
from .scene import VoxelMap, World, load_scene, voxelize_point_cloud

SCENES = Path(__file__).resolve().parents[1] / "scenes"

# Franka EI-ZO parameters and the Forest defaults
FRANKA_PARAMS = dict(delta=0.005, eps=0.005, n_p=10_000, n_f=10, n_ms=60, delta_max=0.01)
HOME7 = np.array([0.0, -0.785, 0.0, -2.356, 0.0, 1.571, 0.785])


@lru_cache(maxsize=None)
def cloud10k() -> VoxelMap:
    z = np.load(SCENES / "cloud10k.npz")
    return VoxelMap(z["origin"], float(z["side"]), z["idx"])


def franka7_world(cloud: bool = True) -> World:
    w = load_scene(SCENES / "franka7.json")
    return w.with_vmap(cloud10k()) if cloud else w


def bimanual14_world(cloud: bool = True) -> World:
    w = load_scene(SCENES / "bimanual14.json")
    return w.with_vmap(cloud10k()) if cloud else w


CONFIG2_ROWS = 1 << 20


def config2_rows(n: int = CONFIG2_ROWS, seed: int = 0) -> np.ndarray:
    """Config 2's configurations: U(joint limits) from ``default_rng(seed)``, cast
    to fp32.  Seed 0 is the set the reference's flags were computed on (tests/golden/config2_1m.npz)."""
    w = load_scene(SCENES / "franka7.json")
    return np.random.default_rng(seed).uniform(w.lower, w.upper, size=(n, w.model.dof)).astype(np.float32)


# ---------------------------------------------------------------------------
# planar scenes
# ---------------------------------------------------------------------------
ARM_LINKS = (0.9, 0.7, 0.5)
ARM_SPHERE_RADIUS = 0.07
ARM_TABLE = Geometry(BOX, RigidTransform.planar(0.0, -0.2), half_extents=np.array([2.5, 0.1]))
ARM_DISCS = ((0.9, 1.2), (-0.8, 1.0), (0.2, 1.8))


def three_link_arm_model() -> RobotModel:
    """Planar arm: three revolute joints, three spheres per link, base-vs-distal self pairs."""
    def chain(length):
        return tuple(Geometry(SPHERE, RigidTransform.planar(f * length, 0.0), radius=ARM_SPHERE_RADIUS)
                     for f in (1 / 6, 3 / 6, 5 / 6))

    l0, l1, l2 = ARM_LINKS
    joints = (Joint(REVOLUTE, -1, RigidTransform.identity(2)),
              Joint(REVOLUTE, 0, RigidTransform.planar(l0, 0.0)),
              Joint(REVOLUTE, 1, RigidTransform.planar(l1, 0.0)),
              Joint("fixed", 2, RigidTransform.planar(l2, 0.0)))
    links = (Link(chain(l0)), Link(chain(l1)), Link(chain(l2)), Link())
    pairs = tuple((i, j) for i in range(3) for j in range(6, 9))
    return RobotModel(2, joints, links, np.array([0.2, -2.2, -2.2]), np.array([math.pi - 0.2, 2.2, 2.2]), pairs)


def arm3_world() -> World:
    """Config 1: the arm over its table with three disc obstacles (r = 0.15)."""
    discs = tuple(Geometry(SPHERE, RigidTransform.planar(x, y), radius=0.15) for x, y in ARM_DISCS)
    return World(three_link_arm_model(), static=(ARM_TABLE,) + discs)


# free with margin 0.02 at step 0.01 (rejection-sampled once with default_rng(3), length 0.6)
ARM3_SEGMENT = (np.array([2.09001041, -0.35481385, -0.32738464]), np.array([2.03563355, -0.19406005, 0.24811634]))

DOMAIN_HALF = 5.0
CENTER_HALF = 3.5


def point_robot_model(lower=(-DOMAIN_HALF, -DOMAIN_HALF), upper=(DOMAIN_HALF, DOMAIN_HALF)) -> RobotModel:
    """Two prismatic joints carrying a radius-zero sphere."""
    joints = (Joint(PRISMATIC, -1, RigidTransform.identity(2), axis=np.array([1.0, 0.0])),
              Joint(PRISMATIC, 0, RigidTransform.identity(2), axis=np.array([0.0, 1.0])))
    links = (Link(), Link((Geometry(SPHERE, RigidTransform.identity(2), radius=0.0),)))
    return RobotModel(2, joints, links, np.asarray(lower, float), np.asarray(upper, float))


def disc_world(centers, radius=0.35, lower=(-5.0, -5.0), upper=(5.0, 5.0)) -> World:
    model = point_robot_model(lower, upper)
    discs = tuple(Geometry(SPHERE, RigidTransform.planar(c[0], c[1]), radius=radius)
                  for c in np.atleast_2d(np.asarray(centers, dtype=float)))
    return World(model, static=discs)


def forest_centers(seed: int) -> np.ndarray:
    """15 disc centres uniform in the side-7 centre square (bench.py:63-67)."""
    return np.random.default_rng(seed).uniform(-CENTER_HALF, CENTER_HALF, size=(15, 2))


def disc_point_cloud(centers, radius=0.35, spacing=0.01) -> np.ndarray:
    g = np.arange(-radius, radius + spacing / 2, spacing)
    xx, yy = np.meshgrid(g, g)
    m = xx ** 2 + yy ** 2 <= radius ** 2
    disc = np.stack([xx[m], yy[m]], axis=1)
    return np.concatenate([disc + c for c in centers])


def forest_scene_world(seed: int, bin_side: float = 0.02) -> World:
    """Exact discs plus their voxelised point cloud (bench.py:103-110); voxelised on the GPU."""
    c = forest_centers(seed)
    vmap = voxelize_point_cloud(disc_point_cloud(c), bin_side, np.array([-DOMAIN_HALF, -DOMAIN_HALF]))
    w = disc_world(c)
    return w.with_vmap(vmap)


def random_free_segment(world, seed: int = 3, length: float = 0.6, margin: float = 0.02, step: float = 0.01,
                        inner: float = 0.3, max_tries: int = 100_000):
    """Seeded rejection sampling of a segment that is free with ``margin`` at spacing ``step``.

    v1 ~ U(middle of the domain box), v2 = v1 + length * random unit direction
    (SURVEY.md §8(d) config 4); every check runs on the GPU checker.
    """
    ck = world.checker(margin=margin)
    rng = np.random.default_rng(seed)
    lo, hi = world.lower, world.upper
    for _ in range(max_tries):
        v1 = rng.uniform(lo + inner * (hi - lo), hi - inner * (hi - lo))
        if not ck.check(v1):
            continue
        d = rng.normal(size=v1.shape[0])
        d /= np.linalg.norm(d)
        v2 = v1 + d * length
        if np.all(v2 > lo) and np.all(v2 < hi) and ck.check_segment(v1, v2, step):
            return v1, v2
    raise RuntimeError("no free segment found")


def random_free_path(world, n_segments: int = 10, seed: int = 3, length: float = 0.6, margin: float = 0.02,
                     step: float = 0.01, max_tries: int = 100_000) -> np.ndarray:
    """Knots of a chain of ``n_segments`` segments, each free with ``margin`` at spacing ``step`` (config 3)."""
    v1, v2 = random_free_segment(world, seed=seed, length=length, margin=margin, step=step)
    knots = [v1, v2]
    ck = world.checker(margin=margin)
    rng = np.random.default_rng(seed + 1)
    lo, hi = world.lower, world.upper
    tries = 0
    while len(knots) < n_segments + 1:
        tries += 1
        if tries > max_tries:
            raise RuntimeError("could not extend the path")
        d = rng.normal(size=lo.shape[0])
        nxt = knots[-1] + d / np.linalg.norm(d) * length
        if np.all(nxt > lo) and np.all(nxt < hi) and ck.check_segment(knots[-1], nxt, step):
            knots.append(nxt)
    return np.array(knots)
