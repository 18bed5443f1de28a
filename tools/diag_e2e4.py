"""CUPTI trace of the host-buffer check path: copy rates and gaps (is e2e DMA- or host-bound?)."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge
from paper_2504_10783_b200.polytope import HPolytope

w = fx.franka7_world()
nat = w.checker().native
import os
nat.specialize(1 if os.environ.get("SPEC", "1") == "1" else -1)
if "--eizo" in sys.argv:  # what the bench runs before the e2e
    v1, v2 = fx.random_free_segment(w, seed=3)
    dom = HPolytope.from_bounds(w.lower, w.upper)
    for s in range(5):
        inflate_edge(Segment(v1, v2), dom, InflationParams(**fx.FRANKA_PARAMS), w.checker(), seed=7 + s)
n = 1 << 20
pin = torch.empty((n, 7), dtype=torch.float64, pin_memory=True)
pin.copy_(torch.from_numpy(np.random.default_rng(0).uniform(w.lower, w.upper, size=(n, 7))))
res = torch.empty(n, dtype=torch.uint8, pin_memory=True)
for _ in range(5):
    nat.check_host(pin.numpy(), out=res.numpy())
import gc
if os.environ.get("GC") == "collect":
    gc.collect()
elif os.environ.get("GC") == "freeze":
    gc.collect(); gc.freeze()
elif os.environ.get("GC") == "off":
    gc.disable()
ts = []
for _ in range(10):
    t0 = time.perf_counter(); nat.check_host(pin.numpy(), out=res.numpy()); ts.append(time.perf_counter() - t0)
print("ms/call", round(1e3 * float(np.median(ts)), 3))
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    nat.check_host(pin.numpy(), out=res.numpy())
prof.export_chrome_trace("/tmp/t.json")
ev = [e for e in json.load(open("/tmp/t.json"))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
h2d = [e for e in ev if e["cat"] == "gpu_memcpy" and "HtoD" in e["name"]]
print("span us", round(max(e["ts"] + e["dur"] for e in ev) - t0), "H2D copies", len(h2d),
      "sum H2D us", round(sum(e["dur"] for e in h2d)), "mean GB/s",
      round(sum(e["args"].get("bytes", 0) for e in h2d) / max(1, sum(e["dur"] for e in h2d)) / 1e3, 1))
print("first H2D start gaps us", [round(e["ts"] - t0) for e in h2d][:8])
