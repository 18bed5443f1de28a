"""EI-ZO: inflate a collision-free segment into a probabilistically collision-free polytope.

Drop-in for ``corridor/inflation.py``.  ``inflate_edge`` runs the whole loop
on the GPU (``ez_inflate_edge``): hit-and-run, the fused FK + collision
check, order-preserving candidate compaction, projection + fail-fast check +
N_b-round bisection, and the greedy step-back placement, with samples never
leaving device memory.  The small scalar primitives (projection, gradient,
step back, batch size) are host helpers of the public API.
"""

from __future__ import annotations

import ctypes as C
import functools
import math
import threading
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import DimensionMismatch, GradientUndefined, NativeError
from .polytope import HPolytope
from .rng import rng_mode

TERMINATED_ACCEPTED = "test_accepted"
TERMINATED_MAX_ITER = "max_iterations"


@dataclass(frozen=True, eq=False)
class Segment:
    v1: np.ndarray
    v2: np.ndarray

    def __post_init__(self):
        v1 = np.asarray(self.v1, dtype=float)
        v2 = np.asarray(self.v2, dtype=float)
        if v1.shape != v2.shape:
            raise DimensionMismatch("segment endpoints differ in dimension")
        object.__setattr__(self, "v1", v1)
        object.__setattr__(self, "v2", v2)

    @property
    def dim(self) -> int:
        return int(self.v1.shape[0])

    @property
    def length(self) -> float:
        return float(np.linalg.norm(self.v2 - self.v1))

    def point(self, alpha) -> np.ndarray:
        return self.v1 + np.multiply.outer(np.asarray(alpha), self.v2 - self.v1)


@dataclass(frozen=True)
class InflationParams:
    """(delta, eps, tau), step back, and the optimiser counts; defaults = paper Forest table."""

    delta: float = 0.05
    eps: float = 0.01
    tau: float = 0.5
    delta_max: float = 0.01
    n_p: int = 1000
    n_f: int = 10
    n_b: int | None = None
    n_ms: int = 30
    t_col: float = 1e-4
    n_it: int | None = None

    def __post_init__(self):
        for name in ("delta", "eps", "tau"):
            v = getattr(self, name)
            if not 0.0 < v < 1.0:
                raise ValueError("delta, eps, tau must lie in (0, 1)")
        if self.delta_max <= 0.0:
            raise ValueError("delta_max must be positive")
        if not 0.0 <= self.t_col < self.delta_max:
            raise ValueError("need 0 <= t_col < delta_max")
        for name in ("n_p", "n_f", "n_ms"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1")
        if self.n_b is not None and self.n_b < 1:
            raise ValueError("n_b must be >= 1")
        if self.n_it is not None and self.n_it < 1:
            raise ValueError("n_it must be >= 1")

    @staticmethod
    def from_dict(obj: dict) -> "InflationParams":
        names = InflationParams.__dataclass_fields__
        return InflationParams(**{k: v for k, v in obj.items() if k in names})

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k in self.__dataclass_fields__}


@dataclass
class InflationReport:
    polytope: HPolytope
    iterations: int
    hyperplanes_added: int
    collision_checks: int
    terminated_by: str
    device_ms: float = 0.0

    @property
    def guarantee_holds(self) -> bool:
        return self.terminated_by == TERMINATED_ACCEPTED


# ---------------------------------------------------------------------------
# distance-to-segment primitives (inflation.py:115-149)
# ---------------------------------------------------------------------------
def project_batch(C_, seg: Segment):
    Cm = np.atleast_2d(np.asarray(C_, dtype=float))
    if Cm.shape[1] != seg.dim:
        raise DimensionMismatch("point/segment dimension mismatch")
    e = seg.v2 - seg.v1
    ee = float(e @ e)
    if ee == 0.0:
        alpha = np.zeros(Cm.shape[0])
        proj = np.repeat(seg.v1[None, :], Cm.shape[0], axis=0)
    else:
        alpha = np.clip((Cm - seg.v1) @ e / ee, 0.0, 1.0)
        proj = seg.v1 + alpha[:, None] * e
    return proj, alpha, np.linalg.norm(Cm - proj, axis=1)


def project_to_segment(c, seg: Segment):
    """Closest point of the segment: (c_proj, alpha, dist)."""
    c = np.asarray(c, dtype=float)
    if c.shape[0] != seg.dim:
        raise DimensionMismatch("point/segment dimension mismatch")
    p, a, d = project_batch(c[None, :], seg)
    return p[0], float(a[0]), float(d[0])


def dist_to_segment(c, seg: Segment) -> float:
    return project_to_segment(c, seg)[2]


def dist_gradient(c, seg: Segment) -> np.ndarray:
    p, _, d = project_to_segment(c, seg)
    if d <= 1e-12:
        raise GradientUndefined("gradient undefined at distance <= 1e-12")
    return (np.asarray(c, dtype=float) - p) / d


# ---------------------------------------------------------------------------
# the statistical test (inflation.py:156-172)
# ---------------------------------------------------------------------------
def required_batch_size(k: int, params: InflationParams) -> int:
    if k < 1:
        raise ValueError("iterations count from 1")
    delta_k = 6.0 * params.delta / (math.pi ** 2 * k ** 2)
    return int(math.ceil(2.0 * math.log(1.0 / delta_k) / (params.eps * params.tau ** 2)))


def unadaptive_test(n_col_first_m: int, k: int, params: InflationParams):
    m = required_batch_size(k, params)
    return n_col_first_m <= m * (1.0 - params.tau) * params.eps, m


# ---------------------------------------------------------------------------
# candidate updates
# ---------------------------------------------------------------------------
def _bisection_batch(proj, col, n_b: int, checker):
    lo = np.array(proj, dtype=float, copy=True)
    hi = np.array(col, dtype=float, copy=True)
    for _ in range(n_b):
        mid = 0.5 * (lo + hi)
        free = np.asarray(checker.check_batch(mid), dtype=bool)
        hi = np.where(free[:, None], hi, mid)
        lo = np.where(free[:, None], mid, lo)
    return lo, hi


def bisection_update(c_col, seg: Segment, n_b: int, checker) -> np.ndarray:
    """n_b midpoint checks on [c_proj, c_col]; returns the colliding point closest to the projection."""
    c = np.asarray(c_col, dtype=float)
    p, _, _ = project_to_segment(c, seg)
    return _bisection_batch(p[None, :], c[None, :], n_b, checker)[1][0]


def compute_step_back(a, b_raw: float, seg: Segment, delta_max: float) -> float:
    a = np.asarray(a, dtype=float)
    r = max(float(a @ seg.v1), float(a @ seg.v2)) - b_raw + delta_max
    return delta_max - r if r > 0.0 else delta_max


def default_bisection_steps(domain: HPolytope, delta_max: float) -> int:
    """ceil(log2(L / delta_max)) with L the domain box diagonal (inflation.py:219-229)."""
    return _bisection_steps(domain.A.tobytes(), domain.b.tobytes(), domain.A.shape, float(delta_max))


@functools.lru_cache(maxsize=64)
def _bisection_steps(a_bytes: bytes, b_bytes: bytes, shape, delta_max: float) -> int:
    A = np.frombuffer(a_bytes, dtype=float).reshape(shape)
    b = np.frombuffer(b_bytes, dtype=float)
    with np.errstate(divide="ignore", invalid="ignore"):
        R = b[:, None] / A
    hi = np.where(A > 1e-12, R, np.inf).min(axis=0, initial=np.inf)
    lo = np.where(A < -1e-12, R, -np.inf).max(axis=0, initial=-np.inf)
    spans = np.where(np.isfinite(hi) & np.isfinite(lo), hi - lo, 1.0)
    diag = float(np.linalg.norm(spans))
    return max(1, int(math.ceil(math.log2(max(diag, 2.0 * delta_max) / delta_max))))


# ---------------------------------------------------------------------------
# the inflation loop (GPU)
# ---------------------------------------------------------------------------
_CALLS_LOCK = threading.Lock()

def inflate_edge(seg: Segment, domain: HPolytope, params: InflationParams, checker, seed: int = 0,
                 rng="counter") -> InflationReport:
    """Grow a polytope around a collision-free segment inside the domain, on the GPU.

    Same contract as ``corridor/inflation.py:262-325``: the segment is
    contained by construction; ``terminated_by == "test_accepted"`` carries
    the (eps, delta) guarantee.  Raises SeedOutsideDomain, SegmentInCollision,
    GradientUndefined, EmptyChord like the reference.  ``checker`` must be a
    GPU :class:`CollisionChecker` (there is no CPU path).
    """
    if seg.dim != domain.dim:
        raise DimensionMismatch("segment/domain dimension mismatch")
    native = getattr(checker, "native", None)
    if native is None:
        raise NativeError("inflate_edge needs a GPU CollisionChecker; generic checkers have no device path")
    if domain.slack(seg.v1) >= 0.0 or domain.slack(seg.v2) >= 0.0:
        from .errors import SeedOutsideDomain

        raise SeedOutsideDomain("seed segment must be strictly inside the domain")
    n_b = params.n_b if params.n_b is not None else default_bisection_steps(domain, params.delta_max)
    p = N.EizoParams(params.delta, params.eps, params.tau, params.delta_max, params.t_col, params.n_p,
                     params.n_f, n_b, params.n_ms, params.n_it or 0)
    d = seg.dim
    cap = domain.n_faces + params.n_f * (params.n_it if params.n_it else 1024)
    A_out = np.empty((cap, d))
    b_out = np.empty(cap)
    A0 = np.ascontiguousarray(domain.A)
    b0 = np.ascontiguousarray(domain.b)
    v1 = np.ascontiguousarray(seg.v1)
    v2 = np.ascontiguousarray(seg.v2)
    rep = N.EizoReport()
    from .native_world import precision_code

    st = N.lib().ez_inflate_edge(native.handle, N.ptr(v1), N.ptr(v2), d, N.ptr(A0), N.ptr(b0), domain.n_faces,
                                 C.byref(p), int(seed) & (2**64 - 1), precision_code(checker.precision),
                                 rng_mode(rng), C.byref(rep), N.ptr(A_out), N.ptr(b_out), cap)
    if st == 11 and rep.n_faces > cap:  # EZ_CAPACITY: count, then copy (the device run is not repeated)
        cap = rep.n_faces
        A_out, b_out = np.empty((cap, d)), np.empty(cap)
        nf = C.c_int32(0)
        st = N.lib().ez_inflate_edge_result(N.ptr(A_out), N.ptr(b_out), cap, C.byref(nf))
    N.check(st)
    with _CALLS_LOCK:  # inflations of several segments may run in threads
        checker.calls += int(rep.collision_checks)
    F = rep.n_faces
    poly = HPolytope._from_unit_rows(A_out[:F], b_out[:F])  # the device normalised them (cpoly.py:32-38)
    return InflationReport(poly, rep.iterations, rep.hyperplanes_added, int(rep.collision_checks),
                           TERMINATED_ACCEPTED if rep.terminated_by == 0 else TERMINATED_MAX_ITER,
                           float(rep.device_ms))
