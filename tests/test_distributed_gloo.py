"""Multi-rank driver logic on CPU: torch.distributed (gloo), world_size 2, oracle-backed shards.

The sharded EI-ZO loop (all_reduce of the first-M count, all_gather of
candidate counts and boundary points, identical placement on every rank)
must reproduce the single-process inflation exactly; the segment-sharded
path inflation must agree on every rank.
"""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ref
        from oracle_session import OracleSession
        from paper_2504_10783_b200 import fixtures as fx
        from paper_2504_10783_b200.distributed import TorchComm, inflate_edge_sharded, inflate_segments_sharded
        from paper_2504_10783_b200.eizo import InflationParams, Segment
        from paper_2504_10783_b200.polytope import HPolytope

        comm = TorchComm()
        assert comm.collectives == 0
        world_ = fx.disc_world([[0.0, 2.0], [0.0, -2.0]], radius=0.7)
        ck = ref.OracleChecker(world_)
        seg = Segment(np.array([-1.0, 0.0]), np.array([1.0, 0.0]))
        dom = HPolytope.from_bounds([-5, -5], [5, 5])
        params = InflationParams()
        rep = inflate_edge_sharded(seg, dom, params, ck, seed=2, comm=comm,
                                   session_factory=lambda: OracleSession(ck, seg, dom, params, ref.bisection_steps(dom.A, dom.b, 0.01), 2))
        n_coll = comm.collectives

        def fake_inflate(s, domain, prm, checker, seed=0, rng=None):
            out = ref.inflate_edge(s.v1, s.v2, domain.A, domain.b, ref.OracleChecker(world_), seed=seed, n_it=1)
            from paper_2504_10783_b200.eizo import InflationReport
            return InflationReport(HPolytope(out["A"], out["b"]), out["iterations"], out["hyperplanes_added"],
                                   out["collision_checks"], out["terminated_by"])

        from paper_2504_10783_b200.roadmap import PwlPath

        path = PwlPath(np.array([[-4.0, 0.0], [-2.0, 0.5], [-0.5, 0.0], [1.0, 0.3], [3.0, 0.0]]))
        scs, mine = inflate_segments_sharded(path, dom, params, None, seed=5, comm=comm, inflate_fn=fake_inflate)
        seg_scs, _ = inflate_segments_sharded(path, dom, params, None, seed=5, comm=comm, inflate_fn=fake_inflate,
                                              semantics="segment")
        q.put((rank, rep.polytope.A, rep.polytope.b, rep.iterations, rep.collision_checks, list(scs.coverage),
               [P.A for P in scs.sets], sorted(mine), n_coll, list(seg_scs.coverage), scs.reinflated))
    finally:
        dist.destroy_process_group()


def test_sharded_inflation_and_segments_gloo_world2():
    from oracle import ref
    from paper_2504_10783_b200 import fixtures as fx

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    world_ = fx.disc_world([[0.0, 2.0], [0.0, -2.0]], radius=0.7)
    A0 = np.vstack([np.eye(2), -np.eye(2)])
    b0 = np.array([5.0, 5.0, 5.0, 5.0])
    single = ref.inflate_edge(np.array([-1.0, 0.0]), np.array([1.0, 0.0]), A0, b0, ref.OracleChecker(world_), seed=2)
    for rank, A, b, it, checks, coverage, sets, mine, n_coll, _, _ in res:
        assert np.allclose(A, single["A"], atol=1e-12) and np.allclose(b, single["b"], atol=1e-12)
        assert it == single["iterations"] and checks == single["collision_checks"]
        # two collectives per rejecting iteration, one for the accepting one
        assert n_coll == 2 * it - 1
    # segment sharding with reference semantics == the sequential reference loop (planner.py:103-130)
    from oracle.ref import child_seed
    path = np.array([[-4.0, 0.0], [-2.0, 0.5], [-0.5, 0.0], [1.0, 0.3], [3.0, 0.0]])
    seq_sets, seq_cov = [], []
    for k in range(4):
        v1, v2 = path[k], path[k + 1]
        cov = next((j for j, (A, b) in enumerate(seq_sets) if np.all(A @ v1 <= b + 1e-9) and np.all(A @ v2 <= b + 1e-9)), None)
        if cov is None:
            out = ref.inflate_edge(v1, v2, A0, b0, ref.OracleChecker(world_), seed=child_seed(5, 0x5E7, len(seq_sets)),
                                   n_it=1)
            seq_sets.append((out["A"], out["b"]))
            cov = len(seq_sets) - 1
        seq_cov.append(cov)
    assert res[0][5] == seq_cov
    assert len(res[0][6]) == len(seq_sets) and all(np.array_equal(a, s[0]) for a, s in zip(res[0][6], seq_sets))
    assert res[0][10] == res[1][10]
    # segment sharding: round-robin ownership, identical replayed corridor on both ranks
    assert res[0][7] == [0, 2] and res[1][7] == [1, 3]
    assert res[0][5] == res[1][5] and len(res[0][6]) == len(res[1][6])
    for a0, a1 in zip(res[0][6], res[1][6]):
        assert np.array_equal(a0, a1)


def test_shard_helpers():
    from paper_2504_10783_b200.distributed import shard_range, shard_segments

    for n in (0, 1, 7, 10000, 15008):
        for W in (1, 2, 3, 8):
            parts = [shard_range(n, W, r) for r in range(W)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(W - 1))
    assert shard_segments(10, 4, 1) == [1, 5, 9]
