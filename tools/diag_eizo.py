"""Diagnose EI-ZO region latency across repeated calls (same / new checker)."""
import gc, sys, time
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
ck = w.checker()
for s in range(4):
    t0 = time.perf_counter()
    r = inflate_edge(Segment(v1, v2), dom, p, ck, seed=7 + s)
    print(f"same checker {s}: {1e3*(time.perf_counter()-t0):.2f} ms wall, {r.device_ms:.2f} ms device it={r.iterations}", flush=True)
keep = []
for s in range(3):
    c = w.checker()
    _ = c.native
    t0 = time.perf_counter()
    r = inflate_edge(Segment(v1, v2), dom, p, c, seed=7 + s)
    keep.append(c)
    print(f"new checker kept {s}: {1e3*(time.perf_counter()-t0):.2f} ms wall, {r.device_ms:.2f} ms device", flush=True)
for s in range(3):
    t0 = time.perf_counter()
    r = inflate_edge(Segment(v1, v2), dom, p, w.checker(), seed=7 + s)
    print(f"new checker dropped {s}: {1e3*(time.perf_counter()-t0):.2f} ms wall, {r.device_ms:.2f} ms device", flush=True)
for rng in ("counter", "philox"):
    for s in range(3):
        t0 = time.perf_counter()
        r = inflate_edge(Segment(v1, v2), dom, p, ck, seed=7 + s, rng=rng)
        print(f"{rng} {s}: {1e3*(time.perf_counter()-t0):.2f} ms wall, {r.device_ms:.2f} ms device it={r.iterations} f={r.hyperplanes_added}", flush=True)
