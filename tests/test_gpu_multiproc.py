"""The native sharded paths across real processes: torch.distributed world size 2 (gloo,
host-staged collectives), both ranks on cuda:0 with their own ``ez_eizo_session``s.

Each rank's kernels only ever wait on its own stream; the ranks meet in gloo collectives on the
host, so two processes on one GPU exercise exactly the code an 8-GPU NCCL run executes, minus
the transport.  Results must equal the single-process drop-in calls bit for bit
(partition invariance, test_cpoly.py:98-118; inflate_path semantics, planner.py:103-130).
"""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _run(rank, q)
    except BaseException:  # report instead of leaving the parent waiting on the queue
        import traceback

        q.put((rank, "error", traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


def _run(rank, q):
    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.distributed import (TorchComm, inflate_edge_sharded, inflate_paths_sharded,
                                                   inflate_segments_sharded)
    from paper_2504_10783_b200.eizo import InflationParams, Segment
    from paper_2504_10783_b200.polytope import HPolytope
    from paper_2504_10783_b200.roadmap import PwlPath

    comm = TorchComm(device="cpu")
    world = fx.franka7_world()
    ck = world.checker()
    v1, v2 = fx.random_free_segment(world, seed=3)
    dom = HPolytope.from_bounds(world.lower, world.upper)
    params = InflationParams(**fx.FRANKA_PARAMS)
    rep = inflate_edge_sharded(Segment(v1, v2), dom, params, ck, seed=7, comm=comm)
    n_coll = comm.collectives
    path = PwlPath(fx.random_free_path(world, 6, seed=5))
    scs, mine = inflate_segments_sharded(path, dom, params, ck, seed=3, comm=comm)
    paths = [PwlPath(fx.random_free_path(world, 3, seed=s)) for s in (5, 6, 7)]
    by_path = inflate_paths_sharded(paths, dom, params, ck, seed=4, comm=comm)
    q.put((rank, rep.polytope.A, rep.polytope.b, rep.iterations, rep.collision_checks, n_coll,
           [(P.A, P.b) for P in scs.sets], list(scs.coverage), sorted(mine),
           {p: [(P.A, P.b) for P in s.sets] for p, s in by_path.items()}))


def test_native_sessions_two_processes_equal_single_gpu():
    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.corridor import inflate_path
    from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge
    from paper_2504_10783_b200.polytope import HPolytope
    from paper_2504_10783_b200.rng import child_seed
    from paper_2504_10783_b200.roadmap import PwlPath

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda r: r[0])
    errors = [r[2] for r in res if isinstance(r[1], str)]
    assert not errors, errors[0]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    world = fx.franka7_world()
    v1, v2 = fx.random_free_segment(world, seed=3)
    dom = HPolytope.from_bounds(world.lower, world.upper)
    params = InflationParams(**fx.FRANKA_PARAMS)
    single = inflate_edge(Segment(v1, v2), dom, params, world.checker(), seed=7)
    path = PwlPath(fx.random_free_path(world, 6, seed=5))
    seq = inflate_path(path, dom, params, world.checker(), seed=3)
    paths = [PwlPath(fx.random_free_path(world, 3, seed=s)) for s in (5, 6, 7)]
    for rank, A, b, it, checks, n_coll, sets, coverage, mine, by_path in res:
        assert np.array_equal(A, single.polytope.A) and np.array_equal(b, single.polytope.b)
        assert (it, checks) == (single.iterations, single.collision_checks)
        assert n_coll == 2 * it - 1
        assert coverage == seq.coverage and len(sets) == len(seq.sets)
        for (a_, b_), P in zip(sets, seq.sets):
            assert np.array_equal(a_, P.A) and np.array_equal(b_, P.b)
        assert mine == list(range(rank, 6, 2))
        assert sorted(by_path) == list(range(rank, 3, 2))
        for p, got in by_path.items():
            want = inflate_path(paths[p], dom, params, world.checker(), seed=child_seed(4, 0xBA7, p))
            assert len(got) == len(want.sets)
            for (a_, b_), P in zip(got, want.sets):
                assert np.array_equal(a_, P.A) and np.array_equal(b_, P.b)


def test_bench_two_ranks_gloo_mode():
    """`bench.py --gpus 2` outside torchrun re-launches itself under torch.distributed.run and
    prints one JSON line from rank 0 with n_gpus 2 (gloo test mode: both ranks on cuda:0)."""
    import json
    import subprocess

    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--dist-backend", "gloo", "--skip-extra", "--skip-eizo", "--skip-cpu"],
                       capture_output=True, text=True, timeout=900, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["value"] > 0 and d["e2e"]["value"] > 0
