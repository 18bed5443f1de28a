"""Corridor construction and repair around a polygonal path.

Drop-in counterparts of ``inflate_path``, ``find_path_collisions`` and
``refine_sets`` (``corridor/planner.py:103-224``), the direct callers of the
EI-ZO hot path.  Inflations run through ``ez_inflate_edge``, repairs through
``ez_refine_set`` (project / bisect / uncapped placement on the device), path
sampling checks through the GPU checker; the bookkeeping (skip rule,
coverage, set order) is host logic, as in the reference.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .checker import segment_samples
from .eizo import InflationParams, Segment, default_bisection_steps, inflate_edge
from .errors import NativeError
from .native_world import precision_code
from .polytope import HPolytope
from .rng import child_seed


@dataclass(eq=False)
class Scs:
    """Sequence of convex sets along a path: sets, per-segment coverage, seed segments."""

    sets: list
    coverage: list
    seeds: list
    path: object = None
    domain: HPolytope | None = None
    reports: list = field(default_factory=list)


def inflate_path(path, domain: HPolytope, params: InflationParams, checker, seed: int = 0, rng="counter") -> Scs:
    """Inflate path segments in order, skipping any already contained in an earlier set.

    Segment k is inflated with seed ``child_seed(seed, 0x5E7, len(sets))``
    (planner.py:103-130).
    """
    sets, seeds, coverage, reports = [], [], [], []
    knots = path.knots
    for k in range(knots.shape[0] - 1):
        v1, v2 = knots[k], knots[k + 1]
        covered = next((j for j, P in enumerate(sets) if P.contains_segment(v1, v2)), None)
        if covered is None:
            seg = Segment(v1, v2)
            rep = inflate_edge(seg, domain, params, checker, seed=child_seed(seed, 0x5E7, len(sets)), rng=rng)
            sets.append(rep.polytope)
            seeds.append(seg)
            reports.append(rep)
            covered = len(sets) - 1
        coverage.append(covered)
    return Scs(sets, coverage, seeds, path, domain=domain, reports=reports)


def find_path_collisions(scs: Scs, knots, checker, fine_step: float):
    """Colliding samples along a path, attributed to every containing set (planner.py:133-156)."""
    if fine_step <= 0.0:
        raise ValueError("fine_step must be positive")
    knots = np.atleast_2d(np.asarray(getattr(knots, "knots", knots), dtype=float))
    out, seen = [], set()
    for i in range(knots.shape[0] - 1):
        samples = segment_samples(knots[i], knots[i + 1], fine_step)
        free = checker.check_batch(samples)
        for c in samples[~free]:
            key = tuple(np.round(c, 12))
            if key in seen:
                continue
            seen.add(key)
            hit = False
            for j, P in enumerate(scs.sets):
                if P.contains(c):
                    out.append((j, c))
                    hit = True
            if not hit:
                out.append((int(np.argmin([P.slack(c) for P in scs.sets])), c))
    return out


def repair_set(poly: HPolytope, seg: Segment, cols, params: InflationParams, checker, n_b: int):
    """Exclude collisions ``cols`` from ``poly`` (device projection, bisection, uncapped placement)."""
    native = getattr(checker, "native", None)
    if native is None:
        raise NativeError("refine_sets needs a GPU CollisionChecker")
    cols = np.ascontiguousarray(np.atleast_2d(np.asarray(cols, dtype=np.float64)))
    d = seg.dim
    cap = poly.n_faces + cols.shape[0] + 1
    A_out, b_out = np.empty((cap, d)), np.empty(cap)
    nf = C.c_int32(0)
    checks = C.c_int64(0)
    A = np.ascontiguousarray(poly.A)
    b = np.ascontiguousarray(poly.b)
    N.check(N.lib().ez_refine_set(native.handle, N.ptr(np.ascontiguousarray(seg.v1)), N.ptr(np.ascontiguousarray(seg.v2)),
                                  d, N.ptr(A), N.ptr(b), poly.n_faces, N.ptr(cols), cols.shape[0],
                                  float(params.delta_max), float(params.t_col), int(n_b),
                                  precision_code(checker.precision), N.ptr(A_out), N.ptr(b_out), cap,
                                  C.byref(nf), C.byref(checks)))
    checker.calls += int(checks.value)
    return HPolytope(A_out[: nf.value], b_out[: nf.value])


def refine_sets(scs: Scs, collisions, seed_path, params: InflationParams, checker, seed: int = 0,
                rng="counter") -> Scs:
    """Exclude reported collisions from their sets, then restore path coverage (planner.py:159-224)."""
    if not collisions:
        raise ValueError("refine_sets needs at least one collision")
    by_set: dict[int, list] = {}
    for j, c in collisions:
        by_set.setdefault(int(j), []).append(np.asarray(c, dtype=float))
    sets = list(scs.sets)
    seeds = list(scs.seeds)
    domain = scs.domain if scs.domain is not None else sets[0]
    n_b = params.n_b if params.n_b is not None else default_bisection_steps(domain, params.delta_max)
    for j, cols in by_set.items():
        sets[j] = repair_set(sets[j], seeds[j], np.array(cols), params, checker, n_b)
    knots = seed_path.knots
    coverage = list(scs.coverage)
    for k in range(knots.shape[0] - 1):
        v1, v2 = knots[k], knots[k + 1]
        if sets[coverage[k]].contains_segment(v1, v2):
            continue
        found = next((j for j, P in enumerate(sets) if P.contains_segment(v1, v2)), None)
        if found is None:
            seg = Segment(v1, v2)
            rep = inflate_edge(seg, domain, params, checker, seed=child_seed(seed, 0x2EF, k), rng=rng)
            sets.append(rep.polytope)
            seeds.append(seg)
            found = len(sets) - 1
        coverage[k] = found
    order = []
    for c in coverage:
        if c not in order:
            order.append(c)
    order += [j for j in range(len(sets)) if j not in order]
    remap = {old: new for new, old in enumerate(order)}
    return Scs([sets[i] for i in order], [remap[c] for c in coverage], [seeds[i] for i in order], seed_path,
               domain=scs.domain)
