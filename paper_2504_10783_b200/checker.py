"""GPU collision checker: the drop-in for ``corridor.world.CollisionChecker``.

Same protocol as the reference (``corridor/world.py:430-501``): ``check``,
``check_batch`` (True = free, order independent), ``check_segment`` and the
``calls`` counter (one per configuration passed in).  Every call runs the
fused FK + collision kernel (``ez_check_batch`` / ``ez_check_batch_host``).

``precision="fp32"`` (default) evaluates kinematics and distances in fp32:
flags agree with the reference's fp64 oracle wherever the contact distance
exceeds 1e-5.  ``precision="fp64"`` uses the reference's fp64 arithmetic.
"""

from __future__ import annotations

import os

import numpy as np

from .errors import DimensionMismatch
from .native_world import NativeWorld, precision_code


def segment_samples(v1, v2, step: float) -> np.ndarray:
    """ceil(len/step)+1 evenly spaced configurations on conv{v1, v2} (world.py:568-582)."""
    v1 = np.asarray(v1, dtype=float)
    v2 = np.asarray(v2, dtype=float)
    if v1.shape != v2.shape:
        raise DimensionMismatch("segment endpoints differ in dimension")
    length = float(np.linalg.norm(v2 - v1))
    if length == 0.0:
        return v1[None, :]
    n = int(np.ceil(length / step))
    ts = np.linspace(0.0, 1.0, n + 1)
    return v1[None, :] + ts[:, None] * (v2 - v1)[None, :]


class CollisionChecker:
    """Conservative collision oracle for one world and margin, evaluated on the GPU."""

    # "auto" specialisation: robots with at least this many spheres get the
    # model-specialised kernel when the device world is created
    SPECIALIZE_MIN_SPHERES = 16

    def __init__(self, world, margin: float = 0.0, precision: str = "fp32", specialize="auto"):
        self.world = world
        self.model = world.model
        self.margin = float(margin)
        self.precision = precision
        precision_code(precision)
        if specialize not in ("auto", True, False):
            raise ValueError("specialize must be 'auto', True or False")
        self.specialize = specialize
        self.calls = 0
        self._native: NativeWorld | None = None

    @property
    def native(self) -> NativeWorld:
        """The device world, created on first use.  The model-specialised fp32 kernel
        (``ez_world_specialize``: NVRTC once per model and margin, cached in-process and on disk)
        is compiled here and only here, never inside a check call: always with
        ``specialize=True``, for robots of >= 16 spheres with ``"auto"``."""
        if self._native is None:
            nat = NativeWorld(self.model, self.world.static, self.world.vmap, self.margin)
            want = self.specialize is True or (
                self.specialize == "auto" and len(self.model.geometries()) >= self.SPECIALIZE_MIN_SPHERES
                and os.environ.get("EZ_JIT", "1") != "0")
            if want:
                nat.specialize(1)  # EZ_UNSUPPORTED (robot boxes, no NVRTC) keeps the generic kernel
            self._native = nat
        return self._native

    def check(self, q) -> bool:
        return bool(self.check_batch(np.asarray(q, dtype=float)[None, :])[0])

    def check_batch(self, Q):
        """Free mask of a batch.  numpy in -> numpy bool out; a CUDA tensor in -> CUDA bool tensor out."""
        if hasattr(Q, "is_cuda") and Q.is_cuda:
            Qt = Q if Q.dim() == 2 else Q.reshape(1, -1)
            if Qt.shape[0] == 0:
                return Qt.new_zeros((0,), dtype=bool)
            if Qt.shape[1] != self.model.dof:
                raise DimensionMismatch(
                    f"batch has {Qt.shape[1]} columns, robot has {self.model.dof} dof")
            self.calls += int(Qt.shape[0])
            return self.native.check_device(Qt, precision=self.precision).bool()
        Q = np.asarray(Q)
        if Q.dtype != np.float32:  # fp32 rows go to the device as they are (4 B per value)
            Q = np.asarray(Q, dtype=float)
        if Q.ndim != 2:
            Q = np.atleast_2d(Q)
        if Q.shape[0] == 0:
            return np.zeros(0, dtype=bool)
        if Q.shape[1] != self.model.dof:
            raise DimensionMismatch(f"batch has {Q.shape[1]} columns, robot has {self.model.dof} dof")
        self.calls += Q.shape[0]
        return self.native.check_host(Q, precision=self.precision).view(bool)

    def check_segments(self, V1, V2, step: float) -> np.ndarray:
        """Batched ``check_segment`` over many edges in one GPU check.

        Edge i is free iff all of its ceil(len_i / step) + 1 evenly spaced
        samples (``segment_samples``) are free; ``calls`` grows by the total
        sample count, as with one check_segment call per edge.
        """
        if step <= 0.0:
            raise ValueError("step must be positive")
        V1 = np.atleast_2d(np.asarray(V1, dtype=float))
        V2 = np.atleast_2d(np.asarray(V2, dtype=float))
        if V1.shape != V2.shape:
            raise DimensionMismatch("segment endpoints differ in dimension")
        if V1.shape[0] == 0:
            return np.zeros(0, dtype=bool)
        parts = [segment_samples(a, b, step) for a, b in zip(V1, V2)]
        counts = np.array([p.shape[0] for p in parts])
        free = self.check_batch(np.concatenate(parts))
        return np.logical_and.reduceat(free, np.concatenate([[0], np.cumsum(counts)[:-1]]))

    def check_segment(self, v1, v2, step: float) -> bool:
        """True iff every sample at spacing <= step (endpoints included) is free."""
        if step <= 0.0:
            raise ValueError("step must be positive")
        return bool(np.all(self.check_batch(segment_samples(v1, v2, step))))
