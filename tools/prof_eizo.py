"""Profiling driver: EI-ZO 7-DOF single-segment region (Franka parameters), repeated."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge
from paper_2504_10783_b200.polytope import HPolytope

w = fx.franka7_world()
v1, v2 = fx.random_free_segment(w, seed=3)
dom = HPolytope.from_bounds(w.lower, w.upper)
p = InflationParams(**fx.FRANKA_PARAMS)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
rng = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else "counter"
ck = w.checker()
if "--jit" in sys.argv:
    print("specialised:", ck.native.specialize(1))
for s in range(reps):
    t0 = time.perf_counter()
    r = inflate_edge(Segment(v1, v2), dom, p, ck, seed=7, rng=rng)
    print(f"region {s}: {1e3*(time.perf_counter()-t0):.2f} ms wall, {r.device_ms:.2f} ms device, it={r.iterations} faces={r.hyperplanes_added} checks={r.collision_checks}")
