"""Config 3 (10-segment 7-DOF path) wall time vs the number of segments in flight on one GPU."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.distributed import inflate_segments_sharded
from paper_2504_10783_b200.eizo import InflationParams
from paper_2504_10783_b200.polytope import HPolytope
from paper_2504_10783_b200.roadmap import PwlPath

world = fx.franka7_world()
path = PwlPath(fx.random_free_path(world, 10, seed=3))
dom = HPolytope.from_bounds(world.lower, world.upper)
params = InflationParams(**fx.FRANKA_PARAMS)
ck = world.checker()
for c in (1, 2, 4, 6, 8, 10):
    inflate_segments_sharded(path, dom, params, ck, seed=11, concurrency=c)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        inflate_segments_sharded(path, dom, params, ck, seed=11, concurrency=c)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(f"concurrency {c}: {1e3 * min(ts):.1f} ms (min of 3)", flush=True)
