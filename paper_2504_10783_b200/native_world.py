"""Owner of one device-resident world (``ez_world``): robot, static obstacles,
voxel distance grid, for one checker margin.

Replaces the state the reference builds in ``CollisionChecker.__init__``
(``corridor/world.py:441-463``).  Inputs are translated once into the flat
arrays of ``ez_robot_desc`` / ``ez_scene_desc``; afterwards every call passes
device pointers (torch tensors) or host numpy buffers through the C ABI.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from ._device import device_index, require_cuda, stream_handle, torch_mod
from .model import BOX, GEOM_CODES, JOINT_CODES, SPHERE

PRECISIONS = {"fp32": 0, "fp64": 1, "float32": 0, "float64": 1}


def precision_code(p) -> int:
    if isinstance(p, int) and p in (0, 1):
        return p
    try:
        return PRECISIONS[str(p)]
    except KeyError:
        raise ValueError(f"precision must be 'fp32' or 'fp64', got {p!r}") from None


def _robot_arrays(model):
    d = model.dim
    nj = len(model.joints)
    kind = np.array([JOINT_CODES[j.kind] for j in model.joints], dtype=np.int32)
    parent = np.array([j.parent for j in model.joints], dtype=np.int32)
    rot = np.stack([np.asarray(j.origin.rot, dtype=float).reshape(d, d) for j in model.joints]).astype(np.float64)
    trans = np.stack([np.asarray(j.origin.trans, dtype=float).reshape(d) for j in model.joints]).astype(np.float64)
    axis = np.zeros((nj, d))
    for i, j in enumerate(model.joints):
        if j.axis is not None and j.kind != "fixed":
            a = np.asarray(j.axis, dtype=float).ravel()
            axis[i, : min(d, a.size)] = a[:d]
        elif j.kind == "revolute" and d == 3:
            raise ValueError("3-D revolute joint needs an axis")
        elif j.kind == "prismatic":
            raise ValueError("prismatic joint needs an axis")
    geoms = model.geometries()
    ng = len(geoms)
    glink = np.array(model.geometry_links(), dtype=np.int32)
    gkind = np.array([GEOM_CODES[g.kind] for g in geoms], dtype=np.int32)
    grot = np.stack([np.asarray(g.local_pose.rot, float).reshape(d, d) for g in geoms]) if ng else np.zeros((0, d, d))
    gtr = np.stack([np.asarray(g.local_pose.trans, float).reshape(d) for g in geoms]) if ng else np.zeros((0, d))
    grad = np.array([g.radius if g.kind == SPHERE else 0.0 for g in geoms], dtype=np.float64)
    ghalf = np.zeros((ng, d))
    for i, g in enumerate(geoms):
        if g.kind == BOX:
            ghalf[i] = np.asarray(g.half_extents, float)[:d]
    pairs = np.array(model.self_pairs, dtype=np.int32).reshape(-1, 2)
    arrs = dict(kind=kind, parent=parent, rot=np.ascontiguousarray(rot), trans=np.ascontiguousarray(trans),
                axis=np.ascontiguousarray(axis), glink=glink, gkind=gkind,
                grot=np.ascontiguousarray(grot, dtype=np.float64), gtr=np.ascontiguousarray(gtr, dtype=np.float64),
                grad=grad, ghalf=np.ascontiguousarray(ghalf), pairs=np.ascontiguousarray(pairs),
                lower=np.ascontiguousarray(model.lower, dtype=np.float64),
                upper=np.ascontiguousarray(model.upper, dtype=np.float64))
    desc = N.RobotDesc(
        d, nj, N.ptr(arrs["kind"], C.c_int32), N.ptr(arrs["parent"], C.c_int32), N.ptr(arrs["rot"]),
        N.ptr(arrs["trans"]), N.ptr(arrs["axis"]), ng, N.ptr(arrs["glink"], C.c_int32),
        N.ptr(arrs["gkind"], C.c_int32), N.ptr(arrs["grot"]), N.ptr(arrs["gtr"]), N.ptr(arrs["grad"]),
        N.ptr(arrs["ghalf"]), pairs.shape[0], N.ptr(arrs["pairs"], C.c_int32), N.ptr(arrs["lower"]),
        N.ptr(arrs["upper"]))
    return desc, arrs


def _scene_arrays(dim, static, vmap):
    ns = len(static)
    kind = np.array([GEOM_CODES[g.kind] for g in static], dtype=np.int32)
    rot = np.ascontiguousarray(np.stack([np.asarray(g.local_pose.rot, float).reshape(dim, dim) for g in static])
                               if ns else np.zeros((0, dim, dim)))
    tr = np.ascontiguousarray(np.stack([np.asarray(g.local_pose.trans, float).reshape(dim) for g in static])
                              if ns else np.zeros((0, dim)))
    rad = np.array([g.radius if g.kind == SPHERE else 0.0 for g in static], dtype=np.float64)
    half = np.zeros((ns, dim))
    for i, g in enumerate(static):
        if g.kind == BOX:
            half[i] = np.asarray(g.half_extents, float)[:dim]
    if vmap is not None and vmap.n_occupied:
        idx = np.ascontiguousarray(vmap.index_array(), dtype=np.int32)
        origin = np.ascontiguousarray(vmap.origin, dtype=np.float64)
        side = float(vmap.side)
        nv = idx.shape[0]
    else:
        idx = np.zeros((0, dim), dtype=np.int32)
        origin = np.zeros(dim)
        side = 1.0
        nv = 0
    arrs = dict(kind=kind, rot=rot, tr=tr, rad=rad, half=half, idx=idx, origin=origin)
    desc = N.SceneDesc(ns, N.ptr(kind, C.c_int32), N.ptr(rot), N.ptr(tr), N.ptr(rad), N.ptr(half),
                       nv, N.ptr(idx, C.c_int32), N.ptr(origin), side)
    return desc, arrs


class NativeWorld:
    """RAII wrapper of an ``ez_world`` handle on the calling rank's device."""

    def __init__(self, model, static=(), vmap=None, margin: float = 0.0, device: int | None = None):
        require_cuda()
        lib = N.lib()
        self.model = model
        self.dim = model.dim
        self.dof = model.dof
        self.device = device_index() if device is None else int(device)
        rdesc, self._rarrs = _robot_arrays(model)
        sdesc, self._sarrs = _scene_arrays(model.dim, tuple(static), vmap)
        h = C.c_void_p()
        N.check(lib.ez_world_create(C.byref(rdesc), C.byref(sdesc), float(margin), self.device, C.byref(h)))
        self._h = h
        self.margin = float(margin)

    @property
    def handle(self):
        return self._h

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                N.lib().ez_world_destroy(h)
            except Exception:
                pass
            self._h = C.c_void_p()

    def __del__(self):
        self.close()

    def info(self) -> dict:
        wi = N.WorldInfo()
        N.check(N.lib().ez_world_get_info(self._h, C.byref(wi)))
        return {"dof": wi.dof, "n_links": wi.n_links, "n_spheres": wi.n_spheres, "n_pairs": wi.n_pairs,
                "n_hot_pairs": wi.n_hot_pairs,
                "n_static": wi.n_static, "n_voxels": wi.n_voxels, "grid_dims": tuple(wi.grid_dims),
                "cell_side": wi.cell_side, "list_entries": wi.list_entries, "device_bytes": wi.device_bytes,
                "check_cta": wi.check_cta, "check_variant": wi.check_variant}

    # -- checking --------------------------------------------------------------
    def check_host(self, Q: np.ndarray, precision="fp32", out: np.ndarray | None = None) -> np.ndarray:
        """Free mask for host rows (fp32 rows stay fp32 on the wire, anything else is fp64);
        pinned or pageable, pipelined H2D / kernel / D2H inside the library."""
        Q = np.asarray(Q)
        if Q.dtype != np.float32:
            Q = np.asarray(Q, dtype=np.float64)
        if Q.ndim != 2 or Q.strides[1] != Q.itemsize or Q.strides[0] % Q.itemsize:
            Q = np.ascontiguousarray(Q)
        n = Q.shape[0]
        # row stride in elements; numpy gives a single row any stride (e.g. 0 for q[None, :])
        ld = Q.strides[0] // Q.itemsize if n > 1 else Q.shape[1]
        if ld < Q.shape[1]:
            Q = Q.copy()
            ld = Q.shape[1]
        if out is None:
            out = np.empty(n, dtype=np.uint8)
        if n:
            N.check(N.lib().ez_check_batch_host(self._h, Q.ctypes.data, 0 if Q.dtype == np.float32 else 1, n,
                                                ld, out.ctypes.data,
                                                precision_code(precision)))
        return out

    def specialize(self, mode: int = 1) -> bool:
        """Model-specialised fp32 check kernel (``ez_world_specialize``).

        mode 1 compiles it (NVRTC, once per model and margin) and uses it for
        fp32 batches; 0 queries; -1 returns to the generic kernel for good.
        Returns True if the specialised kernel is in use.
        """
        st = N.lib().ez_world_specialize(self._h, int(mode))
        if st == 0:
            return mode >= 0
        if st == 10:  # EZ_UNSUPPORTED: robot boxes, NVRTC missing or disabled
            return False
        N.check(st)
        return False

    def check_device(self, Q, out=None, precision="fp32", stream: int | None = None):
        """Free mask (uint8 CUDA tensor) for a CUDA tensor of configurations (fp32 or fp64)."""
        torch = torch_mod()
        if not Q.is_cuda or Q.device.index != self.device:
            raise ValueError(f"configurations live on {Q.device}, this checker's world is on cuda:{self.device}")
        if Q.dim() != 2 or Q.shape[1] != self.dof:
            from .errors import DimensionMismatch

            raise DimensionMismatch(f"batch has {Q.shape[-1]} columns, robot has {self.dof} dof")
        if Q.dtype not in (torch.float32, torch.float64):
            Q = Q.to(torch.float64)
        if Q.stride(1) != 1:
            Q = Q.contiguous()
        n = Q.shape[0]
        if out is None:
            out = torch.empty(n, dtype=torch.uint8, device=Q.device)
        if n:
            dt = 0 if Q.dtype == torch.float32 else 1
            s = torch.cuda.current_stream(Q.device).cuda_stream if stream is None else stream
            N.check(N.lib().ez_check_batch(self._h, Q.data_ptr(), dt, n, Q.stride(0), out.data_ptr(),
                                           precision_code(precision), s))
        return out

    def link_frames(self, Q: np.ndarray) -> np.ndarray:
        torch = torch_mod()
        dev = torch.device("cuda", self.device)
        q = torch.as_tensor(np.ascontiguousarray(Q, dtype=np.float64), device=dev)
        n = q.shape[0]
        out = torch.empty((n, len(self.model.links), 12), dtype=torch.float64, device=dev)
        if n:
            N.check(N.lib().ez_fk_batch(self._h, q.data_ptr(), n, out.data_ptr(), stream_handle()))
        return out.cpu().numpy()
