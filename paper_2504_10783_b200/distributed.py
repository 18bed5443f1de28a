"""Multi-GPU sharding of the EI-ZO path: one process per GPU.

Two levels:

* **Segments** (config 3): :func:`inflate_segments_sharded` gives rank r the
  path segments k = r, r + W, ...  Each segment is inflated speculatively with
  the segment-keyed seed ``child_seed(seed, 0x5E7, k)``.  The polytopes are
  all-gathered, and every rank replays the reference's sequential skip rule
  (``planner.py:116-120``): set k is kept iff segment k is not contained in an
  earlier kept set.  There is no data-path collective.
* **Samples inside one segment**: :func:`inflate_edge_sharded` splits each
  iteration's walk range [0, n_s) into contiguous shares (rank order is index
  order).  Per iteration it uses three small collectives: all_reduce of the
  first-M collision count, all_gather of the per-rank candidate counts, and
  all_gather of the bisected boundary points (star, projection, distance).
  Every rank then places the same faces.  Walk streams are keyed by the
  global walk index, so the result equals single-GPU ``inflate_edge`` for any
  world size.

Collectives go through a small :class:`Comm` interface.  :class:`TorchComm`
wraps ``torch.distributed`` (NCCL on GPU, gloo on CPU for tests).
``LocalComm`` (world size 1) lets one process drive several shards; the
shard-equivalence tests use it.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .eizo import (TERMINATED_ACCEPTED, TERMINATED_MAX_ITER, InflationParams, InflationReport, Segment,
                   default_bisection_steps, inflate_edge, required_batch_size)
from .errors import raise_for_status
from .polytope import HPolytope
from .rng import child_seed, rng_mode


def shard_range(n: int, world_size: int, rank: int) -> tuple[int, int]:
    """Contiguous share [lo, hi) of range(n) owned by ``rank``."""
    return n * rank // world_size, n * (rank + 1) // world_size


def shard_segments(n_segments: int, world_size: int, rank: int) -> list[int]:
    """Round-robin segment indices of ``rank``."""
    return list(range(rank, n_segments, world_size))


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------
class Comm:
    world_size = 1
    rank = 0

    def all_reduce_sum(self, x: int) -> int:
        return int(x)

    def all_reduce_max(self, x: int) -> int:
        return int(x)

    def all_gather_int(self, x: int) -> list:
        return [int(x)]

    def all_gather_rows(self, t):
        """Concatenate every rank's rows (rank order); variable row counts allowed."""
        return t

    def all_gather_object(self, obj) -> list:
        return [obj]


class LocalComm(Comm):
    """Single process (world size 1)."""


class TorchComm(Comm):
    """torch.distributed default group; tensors live on ``device`` (cuda for NCCL, cpu for gloo)."""

    def __init__(self, device=None):
        import torch
        import torch.distributed as dist

        self.dist = dist
        self.torch = torch
        self.world_size = dist.get_world_size()
        self.rank = dist.get_rank()
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else \
                torch.device("cpu")
        self.device = device

    def _t(self, vals, dtype=None):
        return self.torch.tensor(vals, dtype=dtype or self.torch.int64, device=self.device)

    def all_reduce_sum(self, x):
        t = self._t([int(x)])
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return int(t.item())

    def all_reduce_max(self, x):
        t = self._t([int(x)])
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return int(t.item())

    def all_gather_int(self, x):
        t = self._t([int(x)])
        out = [self.torch.empty_like(t) for _ in range(self.world_size)]
        self.dist.all_gather(out, t)
        return [int(o.item()) for o in out]

    def all_gather_rows(self, t):
        torch = self.torch
        n = self.all_gather_int(t.shape[0])
        width = max(n) if n else 0
        pad = torch.zeros((width,) + tuple(t.shape[1:]), dtype=t.dtype, device=self.device)
        if t.shape[0]:
            pad[: t.shape[0]] = t.to(self.device)
        outs = [torch.empty_like(pad) for _ in range(self.world_size)]
        self.dist.all_gather(outs, pad)
        return torch.cat([o[:k] for o, k in zip(outs, n)])

    def all_gather_object(self, obj):
        out = [None] * self.world_size
        self.dist.all_gather_object(out, obj)
        return out


# ---------------------------------------------------------------------------
# in-segment batch sharding
# ---------------------------------------------------------------------------
class EizoSession:
    """One rank's share of a sharded inflation (``ez_eizo_session``)."""

    def __init__(self, checker, seg: Segment, domain: HPolytope, params: InflationParams, n_b: int, seed: int,
                 rng="counter"):
        import torch

        from .native_world import precision_code

        self.torch = torch
        self.d = seg.dim
        self.n_p = params.n_p
        self.dev = torch.device("cuda", checker.native.device)
        p = N.EizoParams(params.delta, params.eps, params.tau, params.delta_max, params.t_col, params.n_p,
                         params.n_f, n_b, params.n_ms, params.n_it or 0)
        h = C.c_void_p()
        self._keep = [np.ascontiguousarray(x, dtype=np.float64) for x in (seg.v1, seg.v2, domain.A, domain.b)]
        v1, v2, A, b = self._keep
        N.check(N.lib().ez_eizo_session_begin(checker.native.handle, N.ptr(v1), N.ptr(v2), self.d, N.ptr(A),
                                              N.ptr(b), domain.n_faces, C.byref(p), int(seed) & (2 ** 64 - 1),
                                              precision_code(checker.precision), rng_mode(rng), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            N.lib().ez_eizo_session_end(self._h)
            self._h = C.c_void_p()

    __del__ = close

    def sample(self, k: int, walk_begin: int, count: int, m_local: int):
        ncm, nc = C.c_int32(), C.c_int32()
        st = N.lib().ez_eizo_session_sample(self._h, k, int(walk_begin), int(count), int(m_local), C.byref(ncm),
                                            C.byref(nc))
        return st, int(ncm.value), int(nc.value)

    def bisect(self, k: int, n_take: int):
        torch = self.torch
        star = torch.empty((n_take, self.d), dtype=torch.float64, device=self.dev)
        pstar = torch.empty((n_take, self.d), dtype=torch.float64, device=self.dev)
        dstar = torch.empty((n_take,), dtype=torch.float64, device=self.dev)
        st = N.lib().ez_eizo_session_bisect(self._h, k, int(n_take), star.data_ptr(), pstar.data_ptr(),
                                            dstar.data_ptr())
        return st, star, pstar, dstar

    def place(self, k: int, star, pstar, dstar):
        star, pstar, dstar = (x.to(self.dev).contiguous() for x in (star, pstar, dstar))
        placed, nf = C.c_int32(), C.c_int32()
        st = N.lib().ez_eizo_session_place(self._h, k, star.data_ptr(), pstar.data_ptr(), dstar.data_ptr(),
                                           int(star.shape[0]), C.byref(placed), C.byref(nf))
        return st, int(placed.value), int(nf.value)

    def result(self):
        nf = C.c_int32()
        N.lib().ez_eizo_session_result(self._h, None, None, 0, C.byref(nf))
        F = nf.value
        A = np.empty((F, self.d))
        b = np.empty(F)
        N.check(N.lib().ez_eizo_session_result(self._h, N.ptr(A), N.ptr(b), F, C.byref(nf)))
        return HPolytope(A, b)


def _agree(comm: Comm, statuses) -> None:
    """Raise the same error on every rank if any shard failed (no rank is left in a collective)."""
    worst = comm.all_reduce_max(max(statuses) if statuses else 0)
    if worst:
        msg = N.lib().ez_last_error()
        raise_for_status(worst, (msg.decode() if msg else "") or f"a shard failed with status {worst}")


def inflate_edge_sharded(seg: Segment, domain: HPolytope, params: InflationParams, checker, seed: int = 0,
                         comm: Comm | None = None, shards: int | None = None, rng="counter",
                         session_factory=None) -> InflationReport:
    """EI-ZO with each iteration's sample batch split over the ranks of ``comm``.

    ``shards`` > 1 with a single-process ``comm`` drives that many shards in
    this process (the equivalence tests use this).  The result equals
    ``inflate_edge`` exactly.
    """
    comm = comm or LocalComm()
    if seg.dim != domain.dim:
        from .errors import DimensionMismatch

        raise DimensionMismatch("segment/domain dimension mismatch")
    if domain.slack(seg.v1) >= 0.0 or domain.slack(seg.v2) >= 0.0:
        from .errors import SeedOutsideDomain

        raise SeedOutsideDomain("seed segment must be strictly inside the domain")
    n_b = params.n_b if params.n_b is not None else default_bisection_steps(domain, params.delta_max)
    local = shards or 1
    W = comm.world_size * local
    my_shards = [comm.rank * local + j for j in range(local)]
    make = session_factory or (lambda: EizoSession(checker, seg, domain, params, n_b, seed, rng))
    sessions = [make() for _ in my_shards]
    torch = None
    try:
        k, walk_offset, checks, hyper = 1, 0, 0, 0
        while True:
            m = required_batch_size(k, params)
            n_s = max(params.n_p, m)
            res = []
            for g, S in zip(my_shards, sessions):
                lo, hi = shard_range(n_s, W, g)
                res.append(S.sample(k, walk_offset + lo, hi - lo, max(0, min(hi, m) - lo)))
            _agree(comm, [r[0] for r in res])
            n_col_m = comm.all_reduce_sum(sum(r[1] for r in res))
            walk_offset += n_s
            checks += n_s
            if n_col_m <= m * (1.0 - params.tau) * params.eps:
                terminated = TERMINATED_ACCEPTED
                break
            counts = []
            for c in comm.all_gather_object([r[2] for r in res]):
                counts.extend(c)
            prefix = np.concatenate([[0], np.cumsum(counts)])
            rows, sts = [], []
            for g, S in zip(my_shards, sessions):
                take = int(max(0, min(counts[g], params.n_p - prefix[g])))
                st, star, pstar, dstar = S.bisect(k, take)
                sts.append(st)
                rows.append((star, pstar, dstar))
            _agree(comm, sts)
            import torch

            star = comm.all_gather_rows(torch.cat([r[0] for r in rows]))
            pstar = comm.all_gather_rows(torch.cat([r[1] for r in rows]))
            dstar = comm.all_gather_rows(torch.cat([r[2] for r in rows]))
            C_tot = int(star.shape[0])
            checks += C_tot * (1 + n_b)
            outs = [S.place(k, star, pstar, dstar) for S in sessions]
            _agree(comm, [o[0] for o in outs])
            hyper += outs[0][1]
            if params.n_it is not None and k >= params.n_it:
                terminated = TERMINATED_MAX_ITER
                break
            k += 1
        poly = sessions[0].result()
        checker.calls += checks
        return InflationReport(poly, k, hyper, checks, terminated)
    finally:
        for S in sessions:
            S.close()


# ---------------------------------------------------------------------------
# segment sharding
# ---------------------------------------------------------------------------
def inflate_segments_sharded(path, domain: HPolytope, params: InflationParams, checker, seed: int = 0,
                             comm: Comm | None = None, rng="counter", inflate_fn=None, concurrency: int = 6):
    """Inflate the path's segments round-robin over ranks, then replay the skip rule everywhere.

    A rank runs up to ``concurrency`` of its segments at once (host threads;
    each native inflation takes its own device workspace and stream, so
    several latency-bound regions share the GPU).  Returns ``(Scs,
    local_reports)``; every rank gets the same ``Scs``, whatever the
    concurrency (segment-keyed seeds).
    """
    from concurrent.futures import ThreadPoolExecutor

    from .corridor import Scs

    comm = comm or LocalComm()
    knots = path.knots
    n = knots.shape[0] - 1
    mine = {}
    inflate_fn = inflate_fn or inflate_edge
    own = list(shard_segments(n, comm.world_size, comm.rank))

    def one(k):
        rep = inflate_fn(Segment(knots[k], knots[k + 1]), domain, params, checker,
                         seed=child_seed(seed, 0x5E7, k), rng=rng)
        return k, (rep.polytope.A, rep.polytope.b, rep.iterations, rep.hyperplanes_added, rep.collision_checks)

    workers = max(1, min(int(concurrency), len(own)))
    if workers == 1:
        mine.update(one(k) for k in own)
    else:
        with ThreadPoolExecutor(max_workers=workers) as ex:
            mine.update(ex.map(one, own))
    allpolys = {}
    for part in comm.all_gather_object(mine):
        allpolys.update(part)
    sets, seeds, coverage = [], [], []
    for k in range(n):
        v1, v2 = knots[k], knots[k + 1]
        covered = next((j for j, P in enumerate(sets) if P.contains_segment(v1, v2)), None)
        if covered is None:
            A, b = allpolys[k][0], allpolys[k][1]
            sets.append(HPolytope(A, b))
            seeds.append(Segment(v1, v2))
            covered = len(sets) - 1
        coverage.append(covered)
    return Scs(sets, coverage, seeds, path, domain=domain), mine
