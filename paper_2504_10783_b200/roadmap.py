"""Dynamic-roadmap structures and the online collision-set prune (GPU).

``Grid``/``Drm``/``CollisionSet`` mirror ``corridor/drm.py:27-131``; the DRM1
file format is ``drm.py:501-556``.  :func:`collision_set` replaces
``drm.py:262-296``: the voxel->node CSR map lives on the device
(``ez_roadmap_create``, uploaded once per roadmap) and the union over active
voxels is a bitmap OR (``ez_collision_set``).  The blocked set is returned
as a lazily materialised frozenset view over a sorted id array.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._device import device_index, require_cuda, stream_handle, torch_device
from .errors import DimensionMismatch, GridMismatch
from .scene import VoxelMap


@dataclass(frozen=True, eq=False)
class Grid:
    """Fixed task-space voxel grid; ids are row-major with x fastest."""

    origin: np.ndarray
    side: float
    extents: tuple

    def __post_init__(self):
        object.__setattr__(self, "origin", np.asarray(self.origin, dtype=float))
        object.__setattr__(self, "extents", tuple(int(e) for e in self.extents))
        if len(self.extents) != self.origin.shape[0]:
            raise DimensionMismatch("grid extents/origin dimension mismatch")

    @property
    def dim(self) -> int:
        return len(self.extents)

    @property
    def n_voxels(self) -> int:
        return int(np.prod(self.extents))

    @property
    def sphere_radius(self) -> float:
        return 0.5 * self.side * float(np.sqrt(self.dim))

    def voxel_id(self, idx) -> int:
        vid = 0
        for ax in range(self.dim - 1, -1, -1):
            vid = vid * self.extents[ax] + int(idx[ax])
        return vid

    def ids_of(self, indices) -> np.ndarray:
        I = np.atleast_2d(np.asarray(indices, dtype=np.int64))
        strides = np.cumprod((1,) + self.extents[:-1]).astype(np.int64)
        return I @ strides

    def in_bounds(self, indices) -> np.ndarray:
        I = np.atleast_2d(np.asarray(indices, dtype=np.int64))
        return np.all((I >= 0) & (I < np.asarray(self.extents)), axis=1)

    def all_centers(self) -> np.ndarray:
        axes = [self.origin[a] + (np.arange(self.extents[a]) + 0.5) * self.side for a in range(self.dim)]
        mesh = np.meshgrid(*axes, indexing="ij")
        return np.stack([m.ravel(order="F") for m in mesh], axis=1)


class CollisionSet:
    """Blocked roadmap nodes; ``blocked`` is the frozenset view of ``ids`` (sorted int64)."""

    def __init__(self, blocked=(), ids: np.ndarray | None = None):
        if ids is None:
            ids = np.array(sorted(int(i) for i in blocked), dtype=np.int64)
        self.ids = np.asarray(ids, dtype=np.int64)
        self._set = None

    @property
    def blocked(self) -> frozenset:
        if self._set is None:
            self._set = frozenset(self.ids.tolist())
        return self._set

    def __len__(self) -> int:
        return int(self.ids.shape[0])


@dataclass(eq=False)
class PwlPath:
    knots: np.ndarray

    def __post_init__(self):
        self.knots = np.atleast_2d(np.asarray(self.knots, dtype=float))

    @property
    def length(self) -> float:
        return float(np.sum(np.linalg.norm(np.diff(self.knots, axis=0), axis=1)))

    @property
    def n_segments(self) -> int:
        return self.knots.shape[0] - 1


@dataclass(eq=False)
class Drm:
    nodes: np.ndarray          # (n, dof)
    adj_offsets: np.ndarray    # (n+1,) int64
    adj_ids: np.ndarray        # (nnz,) int32
    cmap_offsets: np.ndarray   # (n_voxels+1,) int64
    cmap_ids: np.ndarray       # (nnz,) int32 sorted per voxel
    poses: np.ndarray
    grid: Grid
    d_cs: float | None = None
    d_ts: float | None = None
    _device: dict = field(default_factory=dict, repr=False)

    @property
    def n_nodes(self) -> int:
        return int(self.nodes.shape[0])

    @property
    def dof(self) -> int:
        return int(self.nodes.shape[1])

    def neighbors(self, i: int) -> np.ndarray:
        return self.adj_ids[self.adj_offsets[i]:self.adj_offsets[i + 1]]

    def colliding_nodes(self, voxel_id: int) -> np.ndarray:
        return self.cmap_ids[self.cmap_offsets[voxel_id]:self.cmap_offsets[voxel_id + 1]]

    def device_map(self) -> "DeviceRoadmap":
        dev = device_index()
        rm = self._device.get(dev)
        if rm is None:
            rm = DeviceRoadmap(self, dev)
            self._device[dev] = rm
        return rm


class DeviceRoadmap:
    """``ez_roadmap`` handle: the CSR collision map resident on one device."""

    @classmethod
    def build(cls, world_or_model, nodes, grid: Grid) -> "DeviceRoadmap":
        """Collision map of ``nodes`` on ``grid`` computed on the GPU (ez_roadmap_build).

        Replaces the node x voxel sweep of ``build_drm`` (drm.py:170-204,
        250-251): voxel v lists every node whose spheres touch v's
        circumscribing sphere (fp64, no margin), ids ascending.
        """
        import torch

        from .native_world import NativeWorld
        from .scene import World

        model = getattr(world_or_model, "model", world_or_model)
        nw = NativeWorld(model, (), None, 0.0)
        dev = torch_device()
        q = torch.as_tensor(np.ascontiguousarray(nodes, dtype=np.float64), device=dev)
        if q.dim() != 2 or q.shape[1] != model.dof:
            raise DimensionMismatch("node rows must have one value per degree of freedom")
        org = np.ascontiguousarray(grid.origin, dtype=np.float64)
        ext = np.ascontiguousarray(grid.extents, dtype=np.int32)
        h = C.c_void_p()
        N.check(N.lib().ez_roadmap_build(nw.handle, q.data_ptr(), q.shape[0], grid.dim, N.ptr(org), float(grid.side),
                                         N.ptr(ext, C.c_int32), stream_handle(), C.byref(h)))
        self = cls.__new__(cls)
        self._h = h
        self.n_nodes = int(q.shape[0])
        self.grid = grid
        return self

    def export(self):
        """(cmap_offsets int64 [n_voxels+1], cmap_ids int32 [nnz]) on the host."""
        nv, nn, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        N.check(N.lib().ez_roadmap_info(self._h, C.byref(nv), C.byref(nn), C.byref(nnz)))
        off = np.empty(nv.value + 1, dtype=np.int64)
        ids = np.empty(nnz.value, dtype=np.int32)
        N.check(N.lib().ez_roadmap_export(self._h, N.ptr(off, C.c_int64), N.ptr(ids, C.c_int32)))
        return off, ids

    def __init__(self, drm: Drm, device: int):
        require_cuda()
        g = drm.grid
        off = np.ascontiguousarray(drm.cmap_offsets, dtype=np.int64)
        ids = np.ascontiguousarray(drm.cmap_ids, dtype=np.int32)
        org = np.ascontiguousarray(g.origin, dtype=np.float64)
        ext = np.ascontiguousarray(g.extents, dtype=np.int32)
        h = C.c_void_p()
        N.check(N.lib().ez_roadmap_create(N.ptr(off, C.c_int64), N.ptr(ids, C.c_int32), g.n_voxels, drm.n_nodes,
                                          g.dim, N.ptr(org), float(g.side), N.ptr(ext, C.c_int32), device,
                                          C.byref(h)))
        self._h = h
        self.n_nodes = drm.n_nodes
        self.grid = g

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                N.lib().ez_roadmap_destroy(h)
            except Exception:
                pass

    def blocked_bits(self, vmap: VoxelMap, same: bool, count: bool = True):
        """Blocked-node bitmap (CUDA uint32 tensor) and its popcount (None if not ``count``:
        then the call does not synchronise)."""
        import torch

        dev = torch_device()
        idx = vmap.device_index()  # voxelize_point_cloud keeps its indices on the device
        if idx is None or idx.device != dev:
            idx = torch.as_tensor(np.ascontiguousarray(vmap.index_array(), dtype=np.int32), device=dev)
        bits = torch.empty(max(1, (self.n_nodes + 31) // 32), dtype=torch.int32, device=dev)
        n_blocked = C.c_int64(0)
        vorg = np.ascontiguousarray(vmap.origin, dtype=np.float64)
        N.check(N.lib().ez_collision_set(self._h, idx.data_ptr(), vmap.n_occupied, N.ptr(vorg), float(vmap.side),
                                         1 if same else 0, bits.data_ptr(), C.byref(n_blocked) if count else None,
                                         stream_handle()))
        return bits, (n_blocked.value if count else None)

    def blocked_ids(self, vmap: VoxelMap, same: bool) -> np.ndarray:
        """Blocked node ids, ascending (int64 host array), via ez_collision_set_ids."""
        import torch

        dev = torch_device()
        idx = vmap.device_index()
        if idx is None or idx.device != dev:
            idx = torch.as_tensor(np.ascontiguousarray(vmap.index_array(), dtype=np.int32), device=dev)
        bits = torch.empty(max(1, (self.n_nodes + 31) // 32), dtype=torch.int32, device=dev)
        ids = torch.empty(max(1, self.n_nodes), dtype=torch.int32, device=dev)
        n = C.c_int64(0)
        vorg = np.ascontiguousarray(vmap.origin, dtype=np.float64)
        N.check(N.lib().ez_collision_set_ids(self._h, idx.data_ptr(), vmap.n_occupied, N.ptr(vorg), float(vmap.side),
                                             1 if same else 0, bits.data_ptr(), ids.data_ptr(), C.byref(n),
                                             stream_handle()))
        return ids[: n.value].cpu().numpy().astype(np.int64)


def build_collision_map(world_or_model, nodes, grid: Grid):
    """(cmap_offsets, cmap_ids) of ``nodes`` on ``grid``, computed on the GPU."""
    return DeviceRoadmap.build(world_or_model, nodes, grid).export()


def sample_free_configurations(checker, lower, upper, count: int, rng, budget_factor: int = 1000) -> np.ndarray:
    """Uniform rejection sampling of free configurations, draw for draw the reference's
    (drm.py:147-167): the same ``rng.uniform`` chunks, each chunk checked in one
    ``checker.check_batch`` call (one GPU launch for a GPU checker)."""
    lower = np.asarray(lower, dtype=float)
    upper = np.asarray(upper, dtype=float)
    out, have, drawn = [], 0, 0
    budget = budget_factor * count
    while have < count:
        chunk = min(max(count - have, 256) * 2, budget - drawn)
        if chunk <= 0:
            from .errors import SamplingExhausted

            raise SamplingExhausted(f"rejection budget {budget} exhausted with {have}/{count} samples")
        Q = rng.uniform(lower, upper, size=(chunk, lower.shape[0]))
        drawn += chunk
        good = Q[np.asarray(checker.check_batch(Q), dtype=bool)]
        out.append(good)
        have += good.shape[0]
    return np.concatenate(out)[:count]


def pose_rows(model, nodes: np.ndarray) -> np.ndarray:
    """``pose_vector(forward_kinematics(model, q)[1])`` for every node (drm.py:217), the
    end-effector (last link) frames from one batched GPU FK launch."""
    from .model import fk_batch

    rots, trans = fk_batch(model, nodes)
    R, t = rots[-1], trans[-1]
    if model.dim == 2:
        return np.concatenate([t, np.arctan2(R[:, 1, 0], R[:, 0, 0])[:, None]], axis=1)
    tr = R[:, 0, 0] + R[:, 1, 1] + R[:, 2, 2]
    w = 0.5 * np.sqrt(np.maximum(0.0, 1.0 + tr))
    with np.errstate(divide="ignore", invalid="ignore"):
        q = np.stack([w, (R[:, 2, 1] - R[:, 1, 2]) / (4 * w), (R[:, 0, 2] - R[:, 2, 0]) / (4 * w),
                      (R[:, 1, 0] - R[:, 0, 1]) / (4 * w)], axis=1)
    near_pi = ~(w > 1e-9)
    if near_pi.any():  # the reference's dominant-diagonal branch (world.py:253-262), row by row
        from .model import RigidTransform, pose_vector

        for r in np.flatnonzero(near_pi):
            q[r] = pose_vector(RigidTransform(R[r], t[r]))[3:]
    return np.concatenate([t, q], axis=1)


def build_drm(model, base_checker, lower, upper, n_nodes: int, k: int, d_cs: float, d_ts: float, grid: Grid,
              seed: int = 0) -> Drm:
    """Drop-in for ``corridor.drm.build_drm`` (drm.py:207-255), every bulk step on the GPU.

    * nodes: ``sample_free_configurations`` with ``default_rng(seed)`` (the reference's draws;
      each rejection chunk is one check launch of ``base_checker``);
    * poses: end-effector pose rows from one FK launch (``pose_rows``);
    * adjacency: ``ez_roadmap_adjacency`` (nearest 4k+1 by configuration distance, d_cs / d_ts
      filters, k per node, symmetrised CSR);
    * collision map: ``ez_roadmap_build`` (node x voxel sweep, CSR by voxel).
    """
    import torch

    if n_nodes < 2:
        raise ValueError("need at least two nodes")
    if k < 1:
        raise ValueError("k must be >= 1")
    rng = np.random.default_rng(seed)
    nodes = sample_free_configurations(base_checker, lower, upper, n_nodes, rng)
    poses = pose_rows(model, nodes)
    dev = torch_device()
    dn = torch.as_tensor(np.ascontiguousarray(nodes, dtype=np.float64), device=dev)
    de = torch.as_tensor(np.ascontiguousarray(poses[:, :model.dim], dtype=np.float64), device=dev)
    off = torch.empty(n_nodes + 1, dtype=torch.int64, device=dev)
    ids = torch.empty(max(1, 2 * k * n_nodes), dtype=torch.int32, device=dev)
    nnz = C.c_int64(0)
    N.check(N.lib().ez_roadmap_adjacency(dn.data_ptr(), n_nodes, model.dof, de.data_ptr(), model.dim, int(k),
                                         float(d_cs), float(d_ts), off.data_ptr(), ids.data_ptr(), C.byref(nnz),
                                         stream_handle()))
    adj_off = off.cpu().numpy()
    adj_ids = ids[: nnz.value].cpu().numpy()
    cmap_off, cmap_ids = DeviceRoadmap.build(model, nodes, grid).export()
    return Drm(nodes, adj_off, adj_ids, cmap_off, cmap_ids, poses, grid, d_cs=d_cs, d_ts=d_ts)


def sample_free_nodes(world, n: int, seed: int = 0, batch: int = 1 << 20) -> np.ndarray:
    """Uniform collision-free configurations of ``world`` (rejection sampling, GPU checks).

    Same distribution as ``sample_free_configurations`` (drm.py:147-167);
    the stream is torch's Philox, not numpy's.
    """
    import torch

    dev = torch_device()
    ck = world.checker()
    lo = torch.as_tensor(world.lower, dtype=torch.float64, device=dev)
    hi = torch.as_tensor(world.upper, dtype=torch.float64, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed))
    out, have = [], 0
    for _ in range(1000):
        Q = lo + (hi - lo) * torch.rand((batch, lo.shape[0]), generator=g, device=dev, dtype=torch.float64)
        free = ck.check_batch(Q)
        good = Q[free]
        out.append(good)
        have += int(good.shape[0])
        if have >= n:
            break
    else:
        from .errors import SamplingExhausted

        raise SamplingExhausted(f"only {have}/{n} free configurations found")
    return torch.cat(out)[:n].cpu().numpy()


def collision_set(drm: Drm, vmap: VoxelMap) -> CollisionSet:
    """Union of the collision-map entries of the occupied voxels (GPU).

    A voxel map on the roadmap grid is used directly; a finer or offset map
    activates every roadmap voxel its cubes overlap (drm.py:273-289).
    """
    if vmap.dim != drm.grid.dim:
        raise GridMismatch("voxel map dimension differs from roadmap grid")
    if vmap.n_occupied == 0:
        return CollisionSet(ids=np.zeros(0, dtype=np.int64))
    same = bool(np.allclose(vmap.origin, drm.grid.origin) and np.isclose(vmap.side, drm.grid.side))
    return CollisionSet(ids=drm.device_map().blocked_ids(vmap, same))


# ---------------------------------------------------------------------------
# DRM1 binary roadmap format (drm.py:501-556)
# ---------------------------------------------------------------------------
_MAGIC = b"DRM1"


def save_drm(drm: Drm, path) -> None:
    g = drm.grid
    o3 = np.zeros(3)
    o3[: g.dim] = g.origin
    e3 = np.ones(3, dtype=np.uint32)
    e3[: g.dim] = g.extents
    with open(path, "wb") as fh:
        fh.write(_MAGIC + struct.pack("<II", 1, drm.dof) + struct.pack("<QQ", drm.n_nodes, g.n_voxels))
        fh.write(o3.astype("<f8").tobytes() + struct.pack("<d", g.side) + e3.astype("<u4").tobytes())
        for arr, dt in ((drm.nodes, "<f8"), (drm.adj_offsets, "<u8"), (drm.adj_ids, "<u4"),
                        (drm.cmap_offsets, "<u8"), (drm.cmap_ids, "<u4"), (drm.poses, "<f8")):
            fh.write(np.asarray(arr).astype(dt).tobytes())


def load_drm(path) -> Drm:
    with open(path, "rb") as fh:
        data = fh.read()
    if data[:4] != _MAGIC:
        raise ValueError("not a roadmap file")
    version, dof = struct.unpack_from("<II", data, 4)
    if version != 1:
        raise ValueError(f"unsupported roadmap version {version}")
    n_nodes, n_vox = struct.unpack_from("<QQ", data, 12)
    pos = 28

    def take(dt, count):
        nonlocal pos
        arr = np.frombuffer(data, dt, count, pos)
        pos += count * np.dtype(dt).itemsize
        return arr

    o3 = take("<f8", 3)
    (side,) = struct.unpack_from("<d", data, pos)
    pos += 8
    e3 = take("<u4", 3)
    nodes = take("<f8", n_nodes * dof).reshape(n_nodes, dof).copy()
    adj_off = take("<u8", n_nodes + 1).astype(np.int64)
    adj_ids = take("<u4", int(adj_off[-1])).astype(np.int32)
    cm_off = take("<u8", n_vox + 1).astype(np.int64)
    cm_ids = take("<u4", int(cm_off[-1])).astype(np.int32)
    rest = len(data) - pos
    psz = rest // (8 * n_nodes) if n_nodes else 0
    poses = np.frombuffer(data, "<f8", n_nodes * psz, pos).reshape(n_nodes, psz).copy()
    dim = 2 if psz == 3 else 3
    grid = Grid(o3[:dim].copy(), side, tuple(int(e) for e in e3[:dim]))
    if grid.n_voxels != n_vox:
        raise ValueError("grid extents disagree with the stored voxel count")
    return Drm(nodes, adj_off, adj_ids, cm_off, cm_ids, poses, grid)
