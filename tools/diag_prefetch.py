"""Session prefetch: 14-DOF EI-ZO iterations through EizoSession with and without walking the next iterations ahead."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.distributed import EizoSession
from paper_2504_10783_b200.eizo import InflationParams, Segment, default_bisection_steps, required_batch_size
from paper_2504_10783_b200.polytope import HPolytope
w = fx.bimanual14_world()
v1, v2 = fx.random_free_segment(w, seed=3)
dom = HPolytope.from_bounds(w.lower, w.upper)
p = InflationParams(**fx.FRANKA_PARAMS)
ck = w.checker()
S = EizoSession(ck, Segment(v1, v2), dom, p, default_bisection_steps(dom, p.delta_max), 7)
off = 0
for k in range(1, 6):
    n = max(p.n_p, required_batch_size(k, p))
    t0 = time.perf_counter(); S.prefetch(k, off, n); t1 = time.perf_counter()
    st = S.sample(k, off, n, n); t2 = time.perf_counter()
    print(f"k={k} n={n} prefetch {1e3*(t1-t0):.2f} ms sample {1e3*(t2-t1):.2f} ms", st, flush=True)
    off += n
