"""Process-phase timings: import, world creation, first and second EI-ZO region (config 4)."""
import sys, time
t0 = time.perf_counter()
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge
from paper_2504_10783_b200.polytope import HPolytope
torch.zeros(1, device="cuda")
t1 = time.perf_counter()
w = fx.bimanual14_world()
ck = w.checker()
_ = ck.native
torch.cuda.synchronize()
t2 = time.perf_counter()
v1, v2 = fx.random_free_segment(w, seed=3)
dom = HPolytope.from_bounds(w.lower, w.upper)
p = InflationParams(**fx.FRANKA_PARAMS)
t3 = time.perf_counter()
r = inflate_edge(Segment(v1, v2), dom, p, ck, seed=7)
t4 = time.perf_counter()
r = inflate_edge(Segment(v1, v2), dom, p, ck, seed=7)
t5 = time.perf_counter()
print(f"import+ctx {t1-t0:.2f}s world {t2-t1:.2f}s segment {t3-t2:.2f}s first {t4-t3:.2f}s second {t5-t4:.2f}s")
