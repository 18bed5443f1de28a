"""e2e (numpy fp64 host rows -> check_host) per-call time after each bench section: which one slows it?"""
import gc, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np, torch
import bench
from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge
from paper_2504_10783_b200.polytope import HPolytope

w = fx.franka7_world()
ck = w.checker()
nat = ck.native
nat.specialize(1)
n = 1 << 20
pin = torch.empty((n, 7), dtype=torch.float64, pin_memory=True)
pin.copy_(torch.from_numpy(np.random.default_rng(0).uniform(w.lower, w.upper, size=(n, 7))))
Qh = pin.numpy()
res = torch.empty(n, dtype=torch.uint8, pin_memory=True).numpy()


def e2e(tag):
    gc.collect()
    for _ in range(3):
        nat.check_host(Qh, out=res)
    g = []
    for _ in range(3):
        t = time.perf_counter()
        for _ in range(10):
            nat.check_host(Qh, out=res)
        g.append((time.perf_counter() - t) / 10 * 1e3)
    print(f"{tag:28s} ms/call {[round(x, 3) for x in g]}", flush=True)


e2e("start")
bench.bench_config4()
e2e("after config4")
v1, v2 = fx.random_free_segment(w, seed=3)
dom = HPolytope.from_bounds(w.lower, w.upper)
for s in range(5):
    inflate_edge(Segment(v1, v2), dom, InflationParams(**fx.FRANKA_PARAMS), ck, seed=7 + s)
e2e("after eizo")
from paper_2504_10783_b200.distributed import LocalComm, inflate_segments_sharded
from paper_2504_10783_b200.roadmap import PwlPath
path = PwlPath(fx.random_free_path(w, 10, seed=3))
for _ in range(2):
    inflate_segments_sharded(path, dom, InflationParams(**fx.FRANKA_PARAMS), w.checker(), seed=11, comm=LocalComm())
e2e("after config3")
pin2 = torch.empty((n, 7), dtype=torch.float64, pin_memory=True)
pin2.copy_(pin)
Qh = pin2.numpy()
e2e("fresh pinned buffer")
