"""Session (in-segment sharding) overhead: inflate_edge vs inflate_edge_sharded with 1 and 2 local shards."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.distributed import inflate_edge_sharded
from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge
from paper_2504_10783_b200.polytope import HPolytope

for name, w in (("7", fx.franka7_world()), ("14", fx.bimanual14_world())):
    v1, v2 = fx.random_free_segment(w, seed=3)
    dom = HPolytope.from_bounds(w.lower, w.upper)
    p = InflationParams(**fx.FRANKA_PARAMS)
    ck = w.checker()
    inflate_edge(Segment(v1, v2), dom, p, ck, seed=7)
    t0 = time.perf_counter(); r = inflate_edge(Segment(v1, v2), dom, p, ck, seed=7); t1 = time.perf_counter()
    inflate_edge_sharded(Segment(v1, v2), dom, p, ck, seed=7, shards=1)
    for sh in (1, 2):
        t2 = time.perf_counter(); r2 = inflate_edge_sharded(Segment(v1, v2), dom, p, ck, seed=7, shards=sh); t3 = time.perf_counter()
        print(f"{name}-DOF: inflate_edge {1e3*(t1-t0):.1f} ms ({r.iterations} it); sharded x{sh} {1e3*(t3-t2):.1f} ms", flush=True)
