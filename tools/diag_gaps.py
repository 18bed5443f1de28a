"""GPU busy time vs span of one EI-ZO region (torch.profiler / CUPTI kernel trace)."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge
from paper_2504_10783_b200.polytope import HPolytope

which = sys.argv[1] if len(sys.argv) > 1 else "7"
w = fx.franka7_world() if which == "7" else fx.bimanual14_world()
v1, v2 = fx.random_free_segment(w, seed=3)
dom = HPolytope.from_bounds(w.lower, w.upper)
p = InflationParams(**fx.FRANKA_PARAMS)
ck = w.checker()
if "--jit" in sys.argv:
    print("specialised:", ck.native.specialize(1))
for _ in range(2):
    inflate_edge(Segment(v1, v2), dom, p, ck, seed=7)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r = inflate_edge(Segment(v1, v2), dom, p, ck, seed=7)
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/trace.json")
ev = [e for e in json.load(open("/tmp/trace.json"))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
t0, t1 = ev[0]["ts"], max(e["ts"] + e["dur"] for e in ev)
busy, cur_s, cur_e = 0.0, None, None
for e in ev:
    s, f = e["ts"], e["ts"] + e["dur"]
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, f
    else:
        cur_e = max(cur_e, f)
busy += cur_e - cur_s
by = {}
for e in ev:
    k = e["name"].split("(")[0][:40]
    by[k] = by.get(k, 0.0) + e["dur"]
print(f"region span {t1 - t0:.0f} us, GPU busy {busy:.0f} us ({100 * busy / (t1 - t0):.0f}%), device_ms {r.device_ms:.3f}")
for k, v in sorted(by.items(), key=lambda x: -x[1])[:14]:
    print(f"  {k:40s} {v:9.0f} us")
if "--timeline" in sys.argv:
    for e in ev:
        print(f"  {e['ts'] - t0:9.1f} +{e['dur']:8.1f}  stream {e.get('args', {}).get('stream', '?'):>4}  {e['name'][:50]}")
