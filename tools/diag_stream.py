"""Config 3 stream throughput on one GPU: segments/s over a stream of 10-segment paths vs the
number of paths in flight (inflate_paths_sharded concurrency)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2504_10783_b200 import fixtures as fx  # noqa: E402
from paper_2504_10783_b200.distributed import LocalComm, inflate_paths_sharded  # noqa: E402
from paper_2504_10783_b200.eizo import InflationParams  # noqa: E402
from paper_2504_10783_b200.polytope import HPolytope  # noqa: E402
from paper_2504_10783_b200.roadmap import PwlPath  # noqa: E402

world = fx.franka7_world()
ck = world.checker()
dom = HPolytope.from_bounds(world.lower, world.upper)
params = InflationParams(**fx.FRANKA_PARAMS)
for conc in (4, 8, 12, 16):
    paths = [PwlPath(fx.random_free_path(world, 10, seed=100 + p)) for p in range(conc)]
    inflate_paths_sharded(paths, dom, params, ck, seed=5, comm=LocalComm(), concurrency=conc)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    inflate_paths_sharded(paths, dom, params, ck, seed=5, comm=LocalComm(), concurrency=conc)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{conc} paths in flight: {10 * conc / dt:.0f} segments/s ({dt * 1e3:.1f} ms)", flush=True)
