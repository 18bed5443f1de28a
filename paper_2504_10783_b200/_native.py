"""ctypes binding of ``libcorridor_b200.so`` (C ABI in ``include/corridor_b200.h``).

This is exactly the binding a maintainer of the reference package would add
to route its hot path to the GPU.  There is no
fallback: if the library or a CUDA device is missing, every GPU entry point
raises :class:`NativeError`.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

from .errors import NativeError, raise_for_status

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libcorridor_b200.so"

c_i32, c_i64, c_u64, c_dbl, c_vp = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_void_p
P_i32, P_i64, P_dbl, P_u8, P_u32 = (C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                    C.POINTER(C.c_uint8), C.POINTER(C.c_uint32))


class RobotDesc(C.Structure):
    _fields_ = [("dim", c_i32), ("n_joints", c_i32),
                ("joint_kind", P_i32), ("joint_parent", P_i32), ("joint_rot", P_dbl),
                ("joint_trans", P_dbl), ("joint_axis", P_dbl),
                ("n_geoms", c_i32), ("geom_link", P_i32), ("geom_kind", P_i32), ("geom_rot", P_dbl),
                ("geom_trans", P_dbl), ("geom_radius", P_dbl), ("geom_half", P_dbl),
                ("n_pairs", c_i32), ("pairs", P_i32), ("joint_lower", P_dbl), ("joint_upper", P_dbl)]


class SceneDesc(C.Structure):
    _fields_ = [("n_static", c_i32), ("static_kind", P_i32), ("static_rot", P_dbl),
                ("static_trans", P_dbl), ("static_radius", P_dbl), ("static_half", P_dbl),
                ("n_voxels", c_i64), ("h_voxel_idx", P_i32), ("voxel_origin", P_dbl),
                ("voxel_side", c_dbl)]


class WorldInfo(C.Structure):
    _fields_ = [("dof", c_i32), ("n_links", c_i32), ("n_spheres", c_i32), ("n_pairs", c_i32),
                ("n_static", c_i32), ("n_hot_pairs", c_i32), ("n_voxels", c_i64), ("grid_dims", c_i32 * 3),
                ("cell_side", c_dbl), ("list_entries", c_i64), ("device_bytes", c_i64),
                ("check_cta", c_i32), ("check_variant", c_i32)]


class EizoParams(C.Structure):
    _fields_ = [("delta", c_dbl), ("eps", c_dbl), ("tau", c_dbl), ("delta_max", c_dbl), ("t_col", c_dbl),
                ("n_p", c_i32), ("n_f", c_i32), ("n_b", c_i32), ("n_ms", c_i32), ("n_it", c_i32)]


class EizoReport(C.Structure):
    _fields_ = [("iterations", c_i32), ("hyperplanes_added", c_i32), ("collision_checks", c_i64),
                ("terminated_by", c_i32), ("n_faces", c_i32), ("device_ms", c_dbl)]


# name -> (restype, argtypes); every symbol declared in include/corridor_b200.h
SIGNATURES = {
    "ez_abi_version": (c_i32, []),
    "ez_last_error": (C.c_char_p, []),
    "ez_device_count": (c_i32, []),
    "ez_fp32_peak": (c_i32, [c_i32, P_dbl, P_dbl]),
    "ez_fp64_tc_peak": (c_i32, [c_i32, P_dbl, P_dbl]),
    "ez_world_create": (c_i32, [C.POINTER(RobotDesc), C.POINTER(SceneDesc), c_dbl, c_i32, C.POINTER(c_vp)]),
    "ez_world_destroy": (c_i32, [c_vp]),
    "ez_world_get_info": (c_i32, [c_vp, C.POINTER(WorldInfo)]),
    "ez_world_specialize": (c_i32, [c_vp, c_i32]),
    "ez_check_batch": (c_i32, [c_vp, c_vp, c_i32, c_i64, c_i64, c_vp, c_i32, c_vp]),
    "ez_check_batch_host": (c_i32, [c_vp, c_vp, c_i32, c_i64, c_i64, c_vp, c_i32]),
    "ez_fk_batch": (c_i32, [c_vp, c_vp, c_i64, c_vp, c_vp]),
    "ez_hit_and_run": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_vp, c_i64, c_i64, c_i32, c_u64, c_u64, c_i32,
                               c_vp, c_vp]),
    "ez_inflate_edge": (c_i32, [c_vp, P_dbl, P_dbl, c_i32, P_dbl, P_dbl, c_i32, C.POINTER(EizoParams),
                                c_u64, c_i32, c_i32, C.POINTER(EizoReport), P_dbl, P_dbl, c_i32]),
    "ez_inflate_edge_result": (c_i32, [P_dbl, P_dbl, c_i32, P_i32]),
    "ez_eizo_session_begin": (c_i32, [c_vp, P_dbl, P_dbl, c_i32, P_dbl, P_dbl, c_i32, C.POINTER(EizoParams), c_u64,
                                      c_i32, c_i32, C.POINTER(c_vp)]),
    "ez_eizo_session_end": (c_i32, [c_vp]),
    "ez_eizo_session_sample": (c_i32, [c_vp, c_i32, c_u64, c_i64, c_i64, P_i32, P_i32]),
    "ez_eizo_session_prefetch": (c_i32, [c_vp, c_i32, c_u64, c_i64]),
    "ez_eizo_session_bisect": (c_i32, [c_vp, c_i32, c_i32, c_vp, c_vp, c_vp]),
    "ez_eizo_session_place": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_vp, c_i32, P_i32, P_i32]),
    "ez_eizo_session_result": (c_i32, [c_vp, P_dbl, P_dbl, c_i32, P_i32]),
    "ez_refine_set": (c_i32, [c_vp, P_dbl, P_dbl, c_i32, P_dbl, P_dbl, c_i32, P_dbl, c_i32, c_dbl, c_dbl, c_i32,
                              c_i32, P_dbl, P_dbl, c_i32, P_i32, P_i64]),
    "ez_voxelize": (c_i32, [c_vp, c_i64, c_i32, P_dbl, c_dbl, c_vp, P_i64, c_vp]),
    "ez_roadmap_create": (c_i32, [P_i64, P_i32, c_i64, c_i64, c_i32, P_dbl, c_dbl, P_i32, c_i32,
                                  C.POINTER(c_vp)]),
    "ez_roadmap_destroy": (c_i32, [c_vp]),
    "ez_roadmap_build": (c_i32, [c_vp, c_vp, c_i64, c_i32, P_dbl, c_dbl, P_i32, c_vp, C.POINTER(c_vp)]),
    "ez_roadmap_adjacency": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_i32, c_i32, c_dbl, c_dbl, c_vp, c_vp, P_i64,
                                     c_vp]),
    "ez_roadmap_info": (c_i32, [c_vp, P_i64, P_i64, P_i64]),
    "ez_roadmap_export": (c_i32, [c_vp, P_i64, P_i32]),
    "ez_collision_set": (c_i32, [c_vp, c_vp, c_i64, P_dbl, c_dbl, c_i32, c_vp, P_i64, c_vp]),
    "ez_collision_set_ids": (c_i32, [c_vp, c_vp, c_i64, P_dbl, c_dbl, c_i32, c_vp, c_vp, P_i64, c_vp]),
}

_lib = None
_lock = threading.Lock()


def load_library(path: Path | str | None = None) -> C.CDLL:
    """Load the shared library (no compute, works without a GPU)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise NativeError(
                f"native library {p} is missing; build it with `python -m paper_2504_10783_b200.build`")
        lib = C.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.ez_abi_version() != 3:
            raise NativeError("ABI version mismatch")
        if path is None:
            _lib = lib
        return lib


def lib() -> C.CDLL:
    return _lib if _lib is not None else load_library()


def check(status: int) -> None:
    """Raise the mapped exception for a non-OK status, with the native message."""
    if status != 0:
        msg = lib().ez_last_error()
        raise_for_status(status, msg.decode() if msg else "")


def ptr(arr, ctype=C.c_double):
    """ctypes pointer to a contiguous numpy array."""
    return arr.ctypes.data_as(C.POINTER(ctype))
