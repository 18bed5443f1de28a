"""Scenes: voxel maps, the ``World`` container, scene JSON and point-cloud files.

Drop-in counterparts of ``VoxelMap``/``voxelize_point_cloud``/``World`` and the
scene/point-cloud I/O of the reference (``corridor/world.py:287-391,
619-711``).  Occupied voxels are held as a lexicographically sorted int array
(the order of ``sorted(occupied)``); the ``occupied`` frozenset view is
materialised only when asked for.  Voxelisation runs on the GPU.
"""

from __future__ import annotations

import ctypes as C
import json
import math
import struct

import numpy as np

from . import _native as N
from ._device import require_cuda, stream_handle, torch_device
from .model import (BOX, SPHERE, Geometry, Joint, Link, RigidTransform, RobotModel,
                    rotation_about_axis)


class VoxelMap:
    """Occupied bins of a regular grid; each bin collides as its circumscribing sphere."""

    def __init__(self, origin, side: float, occupied=()):
        self.origin = np.asarray(origin, dtype=float)
        self.side = float(side)
        dim = self.origin.shape[0]
        if isinstance(occupied, np.ndarray):
            arr = np.asarray(occupied, dtype=np.int64).reshape(-1, dim)
            self._idx = np.unique(arr, axis=0) if arr.shape[0] else arr
            self._set = None
        else:
            s = frozenset(tuple(int(i) for i in v) for v in occupied)
            self._set = s
            arr = np.array(sorted(s), dtype=np.int64).reshape(-1, dim)
            self._idx = arr

    @classmethod
    def _from_sorted(cls, origin, side, idx: np.ndarray) -> "VoxelMap":
        vm = cls.__new__(cls)
        vm.origin = np.asarray(origin, dtype=float)
        vm.side = float(side)
        vm._idx = idx
        vm._set = None
        return vm

    @classmethod
    def _from_device(cls, origin, side, d_idx) -> "VoxelMap":
        """Map whose sorted indices live in a CUDA int32 tensor (voxelize_point_cloud); the host
        copy is made on first use, so voxelize -> collision_set never leaves the device."""
        vm = cls._from_sorted(origin, side, None)
        vm._dev = d_idx
        vm._n = int(d_idx.shape[0])
        return vm

    def _host_idx(self) -> np.ndarray:
        if self._idx is None:
            self._idx = self._dev.cpu().numpy().astype(np.int64)
        return self._idx

    def device_index(self):
        """Sorted indices as a CUDA int32 tensor, if the map was made on the device (else None)."""
        return getattr(self, "_dev", None)

    @property
    def occupied(self) -> frozenset:
        if self._set is None:
            self._set = frozenset(map(tuple, self._host_idx().tolist()))
        return self._set

    @property
    def n_occupied(self) -> int:
        return self._n if self._idx is None else int(self._idx.shape[0])

    def index_array(self) -> np.ndarray:
        """(n, dim) int64 occupied indices in sorted (lexicographic) order."""
        return self._host_idx()

    @property
    def dim(self) -> int:
        return int(self.origin.shape[0])

    @property
    def sphere_radius(self) -> float:
        return 0.5 * self.side * math.sqrt(self.dim)

    def centers(self) -> np.ndarray:
        idx = self._host_idx()
        if idx.shape[0] == 0:
            return np.zeros((0, self.dim))
        return self.origin + (idx.astype(float) + 0.5) * self.side


def voxelize_point_cloud(points, bin_side: float, origin) -> VoxelMap:
    """Occupied bins floor((p - origin) / side) of a point cloud, computed on the GPU.

    Replaces ``corridor/world.py:315-328`` (ez_voxelize): same floor-based
    indexing in fp64, so a point on a bin boundary lands in the higher bin.
    """
    if bin_side <= 0.0:
        raise ValueError("bin side must be positive")
    origin = np.asarray(origin, dtype=float)
    dim = origin.shape[0]
    pts = np.asarray(points, dtype=np.float64).reshape(-1, dim)
    if pts.shape[0] == 0:
        return VoxelMap._from_sorted(origin, bin_side, np.zeros((0, dim), dtype=np.int64))
    require_cuda()
    import torch

    dev = torch_device()
    d_pts = torch.as_tensor(np.ascontiguousarray(pts), device=dev)
    d_idx = torch.empty((pts.shape[0], dim), dtype=torch.int32, device=dev)
    n_out = C.c_int64(0)
    org = np.ascontiguousarray(origin)
    N.check(N.lib().ez_voxelize(d_pts.data_ptr(), pts.shape[0], dim, N.ptr(org), float(bin_side),
                                d_idx.data_ptr(), C.byref(n_out), stream_handle()))
    return VoxelMap._from_device(origin, bin_side, d_idx[: n_out.value])


# ---------------------------------------------------------------------------
# point clouds (whitespace XYZ text or PCB1 binary: "PCB1", u64 count, 4 pad bytes, f32 xyz)
# ---------------------------------------------------------------------------
_PCB = b"PCB1"


def load_point_cloud(path) -> np.ndarray:
    with open(path, "rb") as fh:
        raw = fh.read()
    if raw[:4] == _PCB:
        (count,) = struct.unpack_from("<Q", raw, 4)
        body = np.frombuffer(raw, dtype="<f4", offset=16)
        if body.shape[0] < count * 3:
            raise ValueError("truncated point cloud file")
        return body[: count * 3].reshape(count, 3).astype(np.float64)
    vals = np.array(raw.split(), dtype=np.float64)
    if vals.size % 3:
        raise ValueError("text point cloud must contain XYZ triples")
    return vals.reshape(-1, 3)


def save_point_cloud(path, points, binary: bool = False) -> None:
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    if binary:
        with open(path, "wb") as fh:
            fh.write(_PCB + struct.pack("<Q", pts.shape[0]) + b"\0\0\0\0")
            fh.write(pts.astype("<f4").tobytes())
    else:
        np.savetxt(path, pts, fmt="%.9g")


# ---------------------------------------------------------------------------
# world
# ---------------------------------------------------------------------------
class World:
    """A robot in a scene: static geometry, an optional voxel map and the domain box."""

    def __init__(self, model: RobotModel, static=(), vmap: VoxelMap | None = None, lower=None, upper=None):
        self.model = model
        self.static = tuple(static)
        self.vmap = vmap
        self.lower = np.asarray(model.lower if lower is None else lower, dtype=float).copy()
        self.upper = np.asarray(model.upper if upper is None else upper, dtype=float).copy()

    def with_vmap(self, vmap: VoxelMap | None) -> "World":
        return World(self.model, self.static, vmap, self.lower, self.upper)

    def checker(self, margin: float = 0.0, precision: str = "fp32", specialize="auto"):
        from .checker import CollisionChecker

        return CollisionChecker(self, margin=margin, precision=precision, specialize=specialize)


# ---------------------------------------------------------------------------
# scene JSON (format of corridor/world.py:619-711)
# ---------------------------------------------------------------------------
def _tf_json(tf: RigidTransform) -> dict:
    out = {"translation": [float(v) for v in tf.trans]}
    if tf.dim == 2:
        out["angle"] = float(math.atan2(tf.rot[1, 0], tf.rot[0, 0]))
    else:
        out["matrix"] = [[float(v) for v in row] for row in tf.rot]
    return out


def _tf_parse(obj: dict, dim: int) -> RigidTransform:
    t = np.asarray(obj.get("translation", np.zeros(dim)), dtype=float)
    if dim == 2:
        a = float(obj.get("angle", 0.0))
        return RigidTransform(np.array([[math.cos(a), -math.sin(a)], [math.sin(a), math.cos(a)]]), t)
    if "matrix" in obj:
        return RigidTransform(np.asarray(obj["matrix"], dtype=float), t)
    R = np.eye(3)
    if "rpy" in obj:
        r, p, y = obj["rpy"]
        R = rotation_about_axis([0, 0, 1], y) @ rotation_about_axis([0, 1, 0], p) @ rotation_about_axis([1, 0, 0], r)
    return RigidTransform(R, t)


def _geom_json(g: Geometry) -> dict:
    out = {"kind": g.kind, "pose": _tf_json(g.local_pose)}
    if g.kind == SPHERE:
        out["radius"] = float(g.radius)
    else:
        out["half_extents"] = [float(v) for v in g.half_extents]
    return out


def _geom_parse(obj: dict, dim: int) -> Geometry:
    pose = _tf_parse(obj.get("pose", {}), dim)
    if obj["kind"] == SPHERE:
        return Geometry(SPHERE, pose, radius=float(obj["radius"]))
    return Geometry(BOX, pose, half_extents=np.asarray(obj["half_extents"], dtype=float))


def world_to_json(world: World) -> dict:
    m = world.model
    joints = []
    for j in m.joints:
        rec = {"type": j.kind, "parent": j.parent, "offset": _tf_json(j.origin)}
        if j.axis is not None:
            rec["axis"] = [float(v) for v in j.axis]
        joints.append(rec)
    return {
        "robot": {
            "dim": m.dim,
            "joints": joints,
            "links": [{"geometries": [_geom_json(g) for g in link.geometries]} for link in m.links],
            "limits": {"lower": [float(v) for v in m.lower], "upper": [float(v) for v in m.upper]},
            "self_pairs": [list(p) for p in m.self_pairs],
        },
        "static": [_geom_json(g) for g in world.static],
        "domain": {"lower": [float(v) for v in world.lower], "upper": [float(v) for v in world.upper]},
    }


def world_from_json(obj: dict) -> World:
    rb = obj["robot"]
    dim = int(rb.get("dim", len(obj["domain"]["lower"])))
    joints = tuple(
        Joint(j["type"], int(j.get("parent", i - 1)), _tf_parse(j.get("offset", {}), dim),
              axis=np.asarray(j["axis"], dtype=float) if "axis" in j else None)
        for i, j in enumerate(rb["joints"]))
    links = tuple(Link(tuple(_geom_parse(g, dim) for g in link.get("geometries", []))) for link in rb["links"])
    model = RobotModel(dim, joints, links, np.asarray(rb["limits"]["lower"], dtype=float),
                       np.asarray(rb["limits"]["upper"], dtype=float),
                       tuple(tuple(p) for p in rb.get("self_pairs", [])))
    static = tuple(_geom_parse(g, dim) for g in obj.get("static", []))
    return World(model, static, lower=np.asarray(obj["domain"]["lower"], dtype=float),
                 upper=np.asarray(obj["domain"]["upper"], dtype=float))


def load_scene(path) -> World:
    with open(path) as fh:
        return world_from_json(json.load(fh))


def save_scene(path, world: World) -> None:
    with open(path, "w") as fh:
        json.dump(world_to_json(world), fh, indent=2)
        fh.write("\n")
