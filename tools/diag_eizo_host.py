"""Host-side overhead of inflate_edge: Python wrapper vs the C call vs device time (7-DOF region)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2504_10783_b200 import _native as N
from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge
from paper_2504_10783_b200.polytope import HPolytope

w = fx.franka7_world()
v1, v2 = fx.random_free_segment(w, seed=3)
dom = HPolytope.from_bounds(w.lower, w.upper)
p = InflationParams(**fx.FRANKA_PARAMS)
ck = w.checker()
lib = N.lib()
real = lib.ez_inflate_edge
tc = []


def timed(*a):
    t0 = time.perf_counter()
    r = real(*a)
    tc.append(time.perf_counter() - t0)
    return r


lib.ez_inflate_edge = timed
for _ in range(3):
    inflate_edge(Segment(v1, v2), dom, p, ck, seed=7)
tw, td = [], []
tc.clear()
for _ in range(10):
    t0 = time.perf_counter()
    r = inflate_edge(Segment(v1, v2), dom, p, ck, seed=7)
    tw.append(time.perf_counter() - t0)
    td.append(r.device_ms * 1e-3)
print("wall %.3f  C call %.3f  device %.3f ms" % tuple(1e3 * float(np.median(x)) for x in (tw, tc, td)))
