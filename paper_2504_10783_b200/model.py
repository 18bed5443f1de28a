"""Robot description types of the drop-in API.

Host-side data mirroring the reference's ``RigidTransform``, ``Geometry``,
``Joint``, ``Link`` and ``RobotModel`` (``corridor/world.py:37-167``): a
kinematic tree given as joints in chain order (joint *j* moves link *j*;
``parent`` is a link index, -1 = world), sphere/box geometries per link and
self-collision pairs over link-major global geometry indices.  Kinematics is
evaluated on the GPU (:func:`fk_batch`, ``ez_fk_batch``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import DimensionMismatch

SPHERE = "sphere"
BOX = "box"
REVOLUTE = "revolute"
PRISMATIC = "prismatic"
FIXED = "fixed"

JOINT_CODES = {FIXED: 0, REVOLUTE: 1, PRISMATIC: 2}
GEOM_CODES = {SPHERE: 0, BOX: 1}


def rotation_about_axis(axis, angle: float) -> np.ndarray:
    """Rotation matrix of ``angle`` about a 3-D axis (Rodrigues' formula)."""
    u = np.asarray(axis, dtype=float)
    u = u / np.linalg.norm(u)
    x, y, z = u
    skew = np.array([[0.0, -z, y], [z, 0.0, -x], [-y, x, 0.0]])
    return np.eye(3) + math.sin(angle) * skew + (1.0 - math.cos(angle)) * (skew @ skew)


@dataclass(frozen=True, eq=False)
class RigidTransform:
    """Rotation + translation in 2-D or 3-D task space."""

    rot: np.ndarray
    trans: np.ndarray

    @staticmethod
    def identity(dim: int) -> "RigidTransform":
        return RigidTransform(np.eye(dim), np.zeros(dim))

    @staticmethod
    def planar(x: float = 0.0, y: float = 0.0, angle: float = 0.0) -> "RigidTransform":
        c, s = math.cos(angle), math.sin(angle)
        return RigidTransform(np.array([[c, -s], [s, c]]), np.array([float(x), float(y)]))

    def compose(self, other: "RigidTransform") -> "RigidTransform":
        return RigidTransform(self.rot @ other.rot, self.rot @ other.trans + self.trans)

    def apply(self, points: np.ndarray) -> np.ndarray:
        return np.asarray(points, dtype=float) @ self.rot.T + self.trans

    @property
    def dim(self) -> int:
        return int(self.trans.shape[0])


@dataclass(frozen=True, eq=False)
class Geometry:
    """Sphere (radius >= 0; 0 models a point robot) or box (half extents > 0)."""

    kind: str
    local_pose: RigidTransform
    radius: float = 0.0
    half_extents: np.ndarray | None = None

    def __post_init__(self):
        if self.kind not in GEOM_CODES:
            raise ValueError(f"unknown geometry kind {self.kind!r}")
        if self.kind == SPHERE and self.radius < 0.0:
            raise ValueError("sphere radius must be >= 0")
        if self.kind == BOX:
            he = np.asarray(self.half_extents, dtype=float)
            if he.ndim != 1 or np.any(he <= 0.0):
                raise ValueError("box half extents must be positive")
            object.__setattr__(self, "half_extents", he)


@dataclass(frozen=True, eq=False)
class Joint:
    kind: str            # revolute | prismatic | fixed
    parent: int          # parent link index, -1 = world frame
    origin: RigidTransform
    axis: np.ndarray | None = None

    def __post_init__(self):
        if self.kind not in JOINT_CODES:
            raise ValueError(f"unknown joint kind {self.kind!r}")
        if self.axis is not None:
            object.__setattr__(self, "axis", np.asarray(self.axis, dtype=float))


@dataclass(frozen=True, eq=False)
class Link:
    geometries: tuple = ()


@dataclass(frozen=True, eq=False)
class RobotModel:
    """Kinematic tree + collision geometry + self-collision pairs."""

    dim: int
    joints: tuple
    links: tuple
    lower: np.ndarray
    upper: np.ndarray
    self_pairs: tuple = ()
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        lo = np.asarray(self.lower, dtype=float)
        hi = np.asarray(self.upper, dtype=float)
        object.__setattr__(self, "lower", lo)
        object.__setattr__(self, "upper", hi)
        object.__setattr__(self, "joints", tuple(self.joints))
        object.__setattr__(self, "links", tuple(self.links))
        object.__setattr__(self, "self_pairs", tuple(tuple(int(v) for v in p) for p in self.self_pairs))
        if len(self.joints) != len(self.links):
            raise ValueError("need one link per joint")
        if lo.shape != hi.shape or lo.shape[0] != self.dof:
            raise DimensionMismatch("joint limits must match the number of actuated joints")
        if np.any(lo >= hi):
            raise ValueError("joint limits must satisfy lower < upper componentwise")
        owner = self.geometry_links()
        for a, b in self.self_pairs:
            if owner[a] == owner[b]:
                raise ValueError("self-collision pair on a single link")

    @property
    def dof(self) -> int:
        return sum(1 for j in self.joints if j.kind != FIXED)

    def geometry_links(self) -> list[int]:
        return [li for li, link in enumerate(self.links) for _ in link.geometries]

    def geometries(self) -> list[Geometry]:
        return [g for link in self.links for g in link.geometries]


# ---------------------------------------------------------------------------
# kinematics (GPU)
# ---------------------------------------------------------------------------

def _kinematic_world(model: RobotModel):
    from .native_world import NativeWorld

    key = ("kin",)
    w = model._cache.get(key)
    if w is None:
        w = NativeWorld(model, (), None, 0.0)
        model._cache[key] = w
    return w


def fk_batch(model: RobotModel, Q):
    """Link frames for a batch (GPU): lists of (B, dim, dim) rotations and (B, dim) translations.

    Replaces ``corridor/world.py:195-223``.
    """
    Q = np.atleast_2d(np.asarray(Q, dtype=float))
    if Q.shape[1] != model.dof:
        raise DimensionMismatch(f"configuration has {Q.shape[1]} values, robot has {model.dof} dof")
    frames = _kinematic_world(model).link_frames(Q)  # (B, L, 12)
    d = model.dim
    rots = [np.ascontiguousarray(frames[:, j, :9].reshape(-1, 3, 3)[:, :d, :d]) for j in range(len(model.links))]
    trans = [np.ascontiguousarray(frames[:, j, 9:9 + d]) for j in range(len(model.links))]
    return rots, trans


def forward_kinematics(model: RobotModel, q):
    """World pose of every geometry plus the end-effector (last link) pose."""
    q = np.asarray(q, dtype=float)
    if q.ndim != 1 or q.shape[0] != model.dof:
        raise DimensionMismatch(f"configuration has {q.size} values, robot has {model.dof} dof")
    rots, trans = fk_batch(model, q[None, :])
    poses = []
    for li, link in enumerate(model.links):
        R, t = rots[li][0], trans[li][0]
        for g in link.geometries:
            poses.append(RigidTransform(R @ g.local_pose.rot, R @ g.local_pose.trans + t))
    return poses, RigidTransform(rots[-1][0], trans[-1][0])


def pose_vector(tf: RigidTransform) -> np.ndarray:
    """(x, y, theta) in 2-D; (x, y, z, qw, qx, qy, qz) in 3-D."""
    if tf.dim == 2:
        return np.array([tf.trans[0], tf.trans[1], math.atan2(tf.rot[1, 0], tf.rot[0, 0])])
    R = tf.rot
    w = 0.5 * math.sqrt(max(0.0, 1.0 + np.trace(R)))
    if w > 1e-9:
        q = np.array([w, (R[2, 1] - R[1, 2]) / (4 * w), (R[0, 2] - R[2, 0]) / (4 * w),
                      (R[1, 0] - R[0, 1]) / (4 * w)])
    else:
        i = int(np.argmax(np.diag(R)))
        j, k = (i + 1) % 3, (i + 2) % 3
        s = math.sqrt(max(1e-18, 1.0 + R[i, i] - R[j, j] - R[k, k]))
        q = np.zeros(4)
        q[1 + i] = 0.5 * s
        q[0] = (R[k, j] - R[j, k]) / (2 * s)
        q[1 + j] = (R[j, i] + R[i, j]) / (2 * s)
        q[1 + k] = (R[k, i] + R[i, k]) / (2 * s)
    return np.concatenate([tf.trans, q])
