"""Multi-GPU sharding of the EI-ZO path: one process per GPU.

Three levels, none with a data-path collective except the in-segment one:

* **Paths** (config 3 throughput, "segments/s over a stream of paths"):
  :func:`inflate_paths_sharded` gives rank r the paths p = r, r + W, ...; each
  is inflated by the drop-in ``inflate_path`` (reference seeding and skip rule,
  planner.py:103-130), several in flight per GPU.  Results are identical to
  one GPU's.
* **Segments of one path** (config 3 latency): :func:`inflate_segments_sharded`
  gives rank r the path segments k = r, r + W, ...  Each is inflated
  speculatively with the seed it would get if no earlier segment were skipped,
  ``child_seed(seed, 0x5E7, k)``.  The polytopes are all-gathered once and
  every rank replays the reference's sequential skip rule (planner.py:116-120).
  With ``semantics="reference"`` (default) a kept set whose reference seed index
  ``len(sets)`` differs from k is re-inflated with that seed, so the corridor
  equals ``inflate_path``'s; ``semantics="segment"`` keeps the segment-keyed
  seeds (not a drop-in: a different, equally valid corridor).
* **Samples inside one segment**: :func:`inflate_edge_sharded` splits each
  iteration's walk range [0, n_s) into contiguous shares (rank order is index
  order).  Per iteration it uses two collectives: an int64 all-gather of each
  shard's (status, first-M collision count, candidate count) and an fp64
  all-gather of the bisected boundary points (star, projection, distance),
  sized from the gathered counts.  Every rank then places the same faces.
  Walk streams are keyed by the global walk index, so the result equals
  single-GPU ``inflate_edge`` for any world size.

Collectives go through a small :class:`Comm` interface.  :class:`TorchComm`
wraps ``torch.distributed`` (NCCL on GPU, gloo for host-staged tests).
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
    """Collectives the sharded paths need.  Every call is made by all ranks in the same order."""

    world_size = 1
    rank = 0

    def all_gather_i64(self, x) -> np.ndarray:
        """(world_size, len(x)) int64: every rank's vector, rank order."""
        return np.asarray(x, dtype=np.int64).reshape(1, -1)

    def all_gather_f64(self, x):
        """(world_size, len(x)) float64 torch tensor on the comm's device: equal lengths on all ranks."""
        return x.reshape(1, -1)

    def all_gather_object(self, obj) -> list:
        return [obj]


class LocalComm(Comm):
    """Single process (world size 1)."""


class TorchComm(Comm):
    """torch.distributed default group.  Tensors live on ``device``: cuda for NCCL, cpu for gloo
    (the host-staged mode the single-GPU multi-process tests use)."""

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
        self.device = torch.device(device)
        self.collectives = 0  # data-path collectives issued (for tests and the benchmark)

    def _gather(self, t):
        torch = self.torch
        out = torch.empty((self.world_size,) + tuple(t.shape), dtype=t.dtype, device=self.device)
        if hasattr(self.dist, "all_gather_into_tensor") and self.device.type == "cuda":
            self.dist.all_gather_into_tensor(out, t)
        else:
            self.dist.all_gather(list(out.unbind(0)), t)
        self.collectives += 1
        return out

    def all_gather_i64(self, x):
        t = self.torch.as_tensor(np.asarray(x, dtype=np.int64), device=self.device)
        return self._gather(t).cpu().numpy()

    def all_gather_f64(self, x):
        return self._gather(x.to(self.device, self.torch.float64).contiguous())

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
        """(status, collisions among the share of the first m, candidates) of walks [walk_begin, +count)."""
        ncm, nc = C.c_int32(), C.c_int32()
        st = N.lib().ez_eizo_session_sample(self._h, k, int(walk_begin), int(count), int(m_local), C.byref(ncm),
                                            C.byref(nc))
        return st, int(ncm.value), int(nc.value)

    def prefetch(self, k: int, walk_begin: int, count: int) -> None:
        """Make iteration k's draws ahead on the session's side stream (a hint)."""
        N.check(N.lib().ez_eizo_session_prefetch(self._h, int(k), int(walk_begin), int(count)))

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


def _raise_worst(statuses) -> None:
    """Raise the mapped error of the worst shard status; every rank holds the same statuses (they
    were all-gathered), so every rank raises the same error and none is left in a collective."""
    worst = int(max(statuses)) if len(statuses) else 0
    if worst:
        msg = N.lib().ez_last_error()
        raise_for_status(worst, (msg.decode() if msg else "") or f"a shard failed with status {worst}")


def inflate_edge_sharded(seg: Segment, domain: HPolytope, params: InflationParams, checker, seed: int = 0,
                         comm: Comm | None = None, shards: int | None = None, rng="counter",
                         session_factory=None) -> InflationReport:
    """EI-ZO with each iteration's sample batch split over the ranks of ``comm``.

    Per iteration two collectives:

    1. one int64 all-gather of ``(status, n_col in the shard's share of the first M, candidates)``
       per shard: every rank gets the global first-M count (the acceptance test,
       inflation.py:294-299), each shard's offset into the global "first N_p colliding by
       index" (inflation.py:300-301), and any shard's failure;
    2. one fp64 all-gather of each shard's bisected rows packed as ``[status | star | pstar |
       dstar]``, sized from the counts of (1), so no size exchange is needed.

    Every rank then runs the identical (deterministic) placement, so no broadcast or status
    exchange follows it.  ``shards`` > 1 with a single-process ``comm`` drives that many shards
    in this process (the equivalence tests use this).  The result equals ``inflate_edge``
    exactly for any number of shards.
    """
    comm = comm or LocalComm()
    if seg.dim != domain.dim:
        from .errors import DimensionMismatch

        raise DimensionMismatch("segment/domain dimension mismatch")
    if domain.slack(seg.v1) >= 0.0 or domain.slack(seg.v2) >= 0.0:
        from .errors import SeedOutsideDomain

        raise SeedOutsideDomain("seed segment must be strictly inside the domain")
    import torch

    n_b = params.n_b if params.n_b is not None else default_bisection_steps(domain, params.delta_max)
    local = shards or 1
    W = comm.world_size * local
    d = seg.dim
    width = 2 * d + 1
    my_shards = [comm.rank * local + j for j in range(local)]
    make = session_factory or (lambda: EizoSession(checker, seg, domain, params, n_b, seed, rng))
    sessions = [make() for _ in my_shards]
    def n_of(k):
        return max(params.n_p, required_batch_size(k, params))

    def prefetch(k, offset):
        # iteration k's draws on each session's side stream, two iterations ahead
        # (the loop's own walks are pipelined one iteration ahead of the host)
        if params.n_it is not None and k > params.n_it:
            return
        for g, S in zip(my_shards, sessions):
            if hasattr(S, "prefetch"):
                lo, hi = shard_range(n_of(k), W, g)
                S.prefetch(k, offset + lo, hi - lo)

    import os
    import time

    prof = {} if os.environ.get("EZ_SHARD_PROFILE") else None

    def tick(name, t0):
        if prof is not None:
            prof[name] = prof.get(name, 0.0) + time.perf_counter() - t0
        return time.perf_counter()

    try:
        k, walk_offset, checks, hyper = 1, 0, 0, 0
        prefetch(1, 0)
        prefetch(2, n_of(1))
        while True:
            m = required_batch_size(k, params)
            n_s = max(params.n_p, m)
            mine = []
            t0 = time.perf_counter()
            for g, S in zip(my_shards, sessions):
                lo, hi = shard_range(n_s, W, g)
                mine.extend(S.sample(k, walk_offset + lo, hi - lo, max(0, min(hi, m) - lo)))
            t0 = tick("sample", t0)
            prefetch(k + 2, walk_offset + n_s + n_of(k + 1))
            t0 = tick("prefetch", t0)
            info = comm.all_gather_i64(mine).reshape(W, 3)  # collective 1
            t0 = tick("collective1", t0)
            _raise_worst(info[:, 0])
            n_col_m = int(info[:, 1].sum())
            walk_offset += n_s
            checks += n_s
            if n_col_m <= m * (1.0 - params.tau) * params.eps:
                terminated = TERMINATED_ACCEPTED
                break
            counts = info[:, 2]
            prefix = np.concatenate([[0], np.cumsum(counts)])
            takes = np.maximum(0, np.minimum(counts, params.n_p - prefix[:-1])).astype(np.int64)
            per_rank = (local + width * takes.reshape(comm.world_size, local).sum(axis=1))
            L = int(per_rank.max())
            parts = []
            t0 = time.perf_counter()
            for g, S in zip(my_shards, sessions):
                st, star, pstar, dstar = S.bisect(k, int(takes[g]))
                head = torch.tensor([float(st)], dtype=torch.float64, device=star.device if star is not None else "cpu")
                if st or star is None:
                    rows = torch.zeros((int(takes[g]), width), dtype=torch.float64, device=head.device)
                else:
                    rows = torch.cat([star, pstar, dstar.reshape(-1, 1)], dim=1)
                parts += [head, rows.reshape(-1).to(head.device)]
            buf = torch.cat([p.to(parts[0].device) for p in parts])
            if buf.numel() < L:
                buf = torch.cat([buf, buf.new_zeros(L - buf.numel())])
            t0 = tick("bisect+pack", t0)
            allbuf = comm.all_gather_f64(buf)  # collective 2
            t0 = tick("collective2", t0)
            heads, rows = [], []
            for r in range(comm.world_size):
                off = 0
                for j in range(local):
                    t = int(takes[r * local + j])
                    heads.append((r, off))
                    rows.append(allbuf[r, off + 1: off + 1 + t * width].reshape(t, width))
                    off += 1 + t * width
            hr = torch.tensor([h[0] for h in heads], device=allbuf.device)
            hc = torch.tensor([h[1] for h in heads], device=allbuf.device)
            _raise_worst(allbuf[hr, hc].cpu().numpy().astype(np.int64))  # one read of every status
            rows = torch.cat(rows)
            C_tot = int(rows.shape[0])
            checks += C_tot * (1 + n_b)
            star, pstar, dstar = rows[:, :d], rows[:, d:2 * d], rows[:, 2 * d]
            t0 = tick("unpack", t0)
            outs = [S.place(k, star, pstar, dstar) for S in sessions]
            t0 = tick("place", t0)
            # placement is deterministic and identical on every rank: no exchange
            _raise_worst([o[0] for o in outs])
            hyper += outs[0][1]
            if params.n_it is not None and k >= params.n_it:
                terminated = TERMINATED_MAX_ITER
                break
            k += 1
        poly = sessions[0].result()
        if prof is not None:
            print("inflate_edge_sharded phases (s):", {k_: round(v, 4) for k_, v in prof.items()}, flush=True)
        checker.calls += checks
        return InflationReport(poly, k, hyper, checks, terminated)
    finally:
        for S in sessions:
            S.close()


# ---------------------------------------------------------------------------
# segment sharding
# ---------------------------------------------------------------------------
def _run_concurrent(fn, items, concurrency):
    from concurrent.futures import ThreadPoolExecutor

    workers = max(1, min(int(concurrency), len(items)))
    if workers == 1:
        return [fn(x) for x in items]
    with ThreadPoolExecutor(max_workers=workers) as ex:
        return list(ex.map(fn, items))


def inflate_segments_sharded(path, domain: HPolytope, params: InflationParams, checker, seed: int = 0,
                             comm: Comm | None = None, rng="counter", inflate_fn=None, concurrency: int = 6,
                             semantics: str = "reference"):
    """Inflate the path's segments round-robin over ranks, then replay the skip rule everywhere.

    A rank runs up to ``concurrency`` of its segments at once (host threads;
    each native inflation takes its own device workspace and stream, so
    several latency-bound regions share the GPU).  Returns ``(Scs,
    local_reports)``; every rank gets the same ``Scs``, whatever the world size
    and concurrency.  ``semantics="reference"``: the corridor equals
    ``corridor.inflate_path``'s (kept sets whose reference seed differs from the
    speculative one are re-inflated, identically on every rank);
    ``"segment"``: segment-keyed seeds, no re-inflation.
    """
    from .corridor import Scs

    if semantics not in ("reference", "segment"):
        raise ValueError("semantics must be 'reference' or 'segment'")
    comm = comm or LocalComm()
    knots = path.knots
    n = knots.shape[0] - 1
    inflate_fn = inflate_fn or inflate_edge
    own = list(shard_segments(n, comm.world_size, comm.rank))

    def one(k, j=None):
        j = k if j is None else j
        rep = inflate_fn(Segment(knots[k], knots[k + 1]), domain, params, checker,
                         seed=child_seed(seed, 0x5E7, j), rng=rng)
        return k, (rep.polytope.A, rep.polytope.b, rep.iterations, rep.hyperplanes_added, rep.collision_checks)

    mine = dict(_run_concurrent(one, own, concurrency))
    allpolys = {}
    for part in comm.all_gather_object(mine):
        allpolys.update(part)
    sets, seeds, coverage = [], [], []
    reinflated = []
    for k in range(n):
        v1, v2 = knots[k], knots[k + 1]
        covered = next((j for j, P in enumerate(sets) if P.contains_segment(v1, v2)), None)
        if covered is None:
            j = len(sets)
            if semantics == "reference" and j != k:
                _, rec = one(k, j)  # the reference's seed for this set (planner.py:121-124)
                reinflated.append(k)
            else:
                rec = allpolys[k]
            sets.append(HPolytope(rec[0], rec[1]))
            seeds.append(Segment(v1, v2))
            covered = len(sets) - 1
        coverage.append(covered)
    scs = Scs(sets, coverage, seeds, path, domain=domain)
    scs.reinflated = reinflated
    return scs, mine


def inflate_paths_sharded(paths, domain: HPolytope, params: InflationParams, checker, seed: int = 0,
                          comm: Comm | None = None, rng="counter", concurrency: int = 6):
    """A stream of paths: rank r inflates paths p = r, r + W, ... with the drop-in ``inflate_path``
    (path p seeded ``child_seed(seed, 0xBA7, p)``), up to ``concurrency`` paths in flight.  No
    collective.  Returns ``{p: Scs}`` for this rank's paths."""
    from .corridor import inflate_path

    comm = comm or LocalComm()
    own = list(shard_segments(len(paths), comm.world_size, comm.rank))

    def one(p):
        return p, inflate_path(paths[p], domain, params, checker, seed=child_seed(seed, 0xBA7, p), rng=rng)

    return dict(_run_concurrent(one, own, concurrency))
