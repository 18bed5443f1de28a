"""Freeze the benchmark scenes of SURVEY.md Appendix A — TEST INFRASTRUCTURE.

Writes ``scenes/franka7.json``, ``scenes/bimanual14.json`` (robot scene JSON
in the reference's format, world.py:659-711) and ``scenes/cloud10k.npz``
(occupied voxel indices of the 10k-voxel point-cloud map).  The self-pair
lists depend on FK at the HOME configuration, evaluated with the oracle.

    python -m oracle.make_scenes
"""

from __future__ import annotations

import math
from pathlib import Path

import numpy as np

from paper_2504_10783_b200.model import (SPHERE, Geometry, Joint, Link, RigidTransform, RobotModel,
                                         rotation_about_axis)
from paper_2504_10783_b200.scene import World, save_scene

from . import ref

ROOT = Path(__file__).resolve().parents[1]
SCENES = ROOT / "scenes"

HALF_PI = math.pi / 2
# Franka-Panda-like joint origins (xyz; rpy), revolute about local z (Appendix A)
ORIGINS = [((0, 0, 0.333), (0, 0, 0)), ((0, 0, 0), (-HALF_PI, 0, 0)), ((0, -0.316, 0), (HALF_PI, 0, 0)),
           ((0.0825, 0, 0), (HALF_PI, 0, 0)), ((-0.0825, 0.384, 0), (-HALF_PI, 0, 0)),
           ((0, 0, 0), (HALF_PI, 0, 0)), ((0.088, 0, 0), (HALF_PI, 0, 0))]
FLANGE = (0, 0, 0.107)
LOWER = [-2.8973, -1.7628, -2.8973, -3.0718, -2.8973, -0.0175, -2.8973]
UPPER = [2.8973, 1.7628, 2.8973, -0.0698, 2.8973, 3.7525, 2.8973]
HOME = np.array([0.0, -0.785, 0.0, -2.356, 0.0, 1.571, 0.785])
SPHERES_PER_LINK = [5, 4, 5, 4, 6, 4, 3, 2]
RADIUS = 0.055


def pose(xyz=(0, 0, 0), rpy=(0, 0, 0)) -> RigidTransform:
    r, p, y = rpy
    R = rotation_about_axis([0, 0, 1], y) @ rotation_about_axis([0, 1, 0], p) @ rotation_about_axis([1, 0, 0], r)
    return RigidTransform(R, np.asarray(xyz, dtype=float))


def _link_spheres(i, n):
    """n spheres at fractions linspace(0.15, 0.85) from the link origin to the next joint origin."""
    nxt = [o[0] for o in ORIGINS[1:]] + [FLANGE, (0, 0, 0.10)]
    a = np.zeros(3)
    b = np.asarray(nxt[i], dtype=float)
    if np.linalg.norm(b) < 1e-9:  # zero-length link
        a, b = np.array([0.0, 0.0, -0.05]), np.array([0.0, 0.0, 0.10])
    return tuple(Geometry(SPHERE, pose(tuple(a + (b - a) * f)), radius=RADIUS) for f in np.linspace(0.15, 0.85, n))


def _arm(base_xyz, link_offset):
    joints = []
    for i, (xyz, rpy) in enumerate(ORIGINS):
        if i == 0:
            xyz = tuple(np.add(xyz, base_xyz))
        joints.append(Joint("revolute", -1 if i == 0 else link_offset + i - 1, pose(xyz, rpy),
                            axis=np.array([0.0, 0.0, 1.0])))
    joints.append(Joint("fixed", link_offset + 6, pose(FLANGE)))
    links = [Link(_link_spheres(i, n)) for i, n in enumerate(SPHERES_PER_LINK)]
    return joints, links


def _separated_pairs(model, home, candidates):
    _, tr = ref.geometry_poses(model, home[None, :])
    geoms = model.geometries()
    keep = []
    for i, j in candidates:
        if np.linalg.norm(tr[i][0] - tr[j][0]) > geoms[i].radius + geoms[j].radius + 0.01:
            keep.append((i, j))
    return keep


def franka7() -> RobotModel:
    joints, links = _arm((0, 0, 0), 0)
    bare = RobotModel(3, joints, links, LOWER, UPPER)
    owner = bare.geometry_links()
    n = len(owner)
    cand = [(i, j) for i in range(n) for j in range(i + 1, n) if owner[j] - owner[i] >= 3]
    return RobotModel(3, joints, links, LOWER, UPPER, tuple(_separated_pairs(bare, HOME, cand)))


def bimanual14() -> RobotModel:
    ja, la = _arm((0, -0.45, 0), 0)
    jb, lb = _arm((0, 0.45, 0), len(ja))
    joints, links = ja + jb, la + lb
    bare = RobotModel(3, joints, links, LOWER + LOWER, UPPER + UPPER)
    owner = bare.geometry_links()
    n = len(owner)
    h = n // 2
    home = np.concatenate([HOME, HOME])
    within = [(i, j) for lo, hi in ((0, h), (h, n)) for i in range(lo, hi) for j in range(i + 1, hi)
              if owner[j] - owner[i] >= 3]
    cross = [(i, j) for i in range(SPHERES_PER_LINK[0], h) for j in range(h + SPHERES_PER_LINK[0], n)]
    pairs = _separated_pairs(bare, home, within) + _separated_pairs(bare, home, cross)
    return RobotModel(3, joints, links, LOWER + LOWER, UPPER + UPPER, tuple(pairs))


def cloud_voxels(n_vox=10_000, side=0.02, seed=0):
    """Occupied voxels of Gaussian blobs in front of the robot (Appendix A, 'stop mid-blob')."""
    rng = np.random.default_rng(seed)
    origin = np.array([-1.0, -1.0, 0.0])
    occ = {}
    while len(occ) < n_vox:
        c = rng.uniform([0.3, -0.6, 0.0], [0.9, 0.6, 1.0])
        r = rng.uniform(0.03, 0.10)
        pts = c + rng.normal(size=(400, 3)) * r / 2
        for t in map(tuple, np.floor((pts - origin) / side).astype(np.int64)):
            occ.setdefault(t, None)
            if len(occ) >= n_vox:
                break
    return origin, side, np.array(sorted(occ), dtype=np.int64)


def main():
    SCENES.mkdir(exist_ok=True)
    save_scene(SCENES / "franka7.json", World(franka7()))
    save_scene(SCENES / "bimanual14.json", World(bimanual14()))
    origin, side, idx = cloud_voxels()
    np.savez_compressed(SCENES / "cloud10k.npz", origin=origin, side=side, idx=idx)
    for name in ("franka7", "bimanual14"):
        from paper_2504_10783_b200.scene import load_scene

        m = load_scene(SCENES / f"{name}.json").model
        print(name, "dof", m.dof, "spheres", len(m.geometries()), "pairs", len(m.self_pairs))
    print("cloud voxels", idx.shape[0])


if __name__ == "__main__":
    main()


def box_arm3d() -> RobotModel:
    """Franka-like chain with one box per link plus a tool sphere (robot box geometry tests)."""
    joints, _ = _arm((0, 0, 0), 0)
    nxt = [o[0] for o in ORIGINS[1:]] + [FLANGE, (0, 0, 0.10)]
    links = []
    for i in range(len(joints)):
        b = np.asarray(nxt[i], dtype=float)
        if np.linalg.norm(b) < 1e-9:
            b = np.array([0.0, 0.0, 0.10])
        mid = 0.5 * b
        L = float(np.linalg.norm(b))
        # box aligned with the link segment: local z along b
        z = b / L
        x = np.cross([0.0, 1.0, 0.0], z) if abs(z[1]) < 0.9 else np.cross([1.0, 0.0, 0.0], z)
        x /= np.linalg.norm(x)
        y = np.cross(z, x)
        R = np.stack([x, y, z], axis=1)
        geoms = [Geometry("box", RigidTransform(R, mid), half_extents=np.array([0.045, 0.045, 0.5 * L + 0.03]))]
        if i == len(joints) - 1:
            geoms.append(Geometry(SPHERE, pose((0, 0, 0.12)), radius=0.05))
        links.append(Link(tuple(geoms)))
    owner = [li for li, l in enumerate(links) for _ in l.geometries]
    n = len(owner)
    pairs = tuple((i, j) for i in range(n) for j in range(i + 1, n) if owner[j] - owner[i] >= 3)
    return RobotModel(3, joints, links, LOWER, UPPER, pairs)


def box_arm2d() -> RobotModel:
    """Planar 3-link arm with box links and sphere tips; box-box and sphere-box self pairs."""
    lengths = (0.9, 0.7, 0.5)
    joints = (Joint("revolute", -1, RigidTransform.identity(2)),
              Joint("revolute", 0, RigidTransform.planar(lengths[0], 0.0)),
              Joint("revolute", 1, RigidTransform.planar(lengths[1], 0.0)),
              Joint("fixed", 2, RigidTransform.planar(lengths[2], 0.0)))
    links = []
    for L in lengths:
        links.append(Link((Geometry("box", RigidTransform.planar(0.5 * L, 0.0, 0.1), half_extents=np.array([0.5 * L, 0.05])),
                           Geometry(SPHERE, RigidTransform.planar(L, 0.0), radius=0.06))))
    links.append(Link())
    # geometries: 0 box0, 1 sph0, 2 box1, 3 sph1, 4 box2, 5 sph2
    pairs = ((0, 4), (0, 5), (1, 4), (1, 5))
    return RobotModel(2, joints, tuple(links), np.array([0.2, -2.6, -2.6]), np.array([math.pi - 0.2, 2.6, 2.6]), pairs)
