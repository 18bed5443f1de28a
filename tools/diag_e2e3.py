"""e2e host path right after a JIT compile (cold vs cached), per-group timing."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2504_10783_b200 import fixtures as fx

w = fx.franka7_world()
n = 1 << 20
Q = np.random.default_rng(0).uniform(w.lower, w.upper, size=(n, 7))
pin = torch.empty((n, 7), dtype=torch.float64, pin_memory=True); pin.copy_(torch.from_numpy(Q))
res = torch.empty(n, dtype=torch.uint8, pin_memory=True)
nat = w.checker().native
t0 = time.perf_counter(); ok = nat.specialize(1); t1 = time.perf_counter()
print("specialize", ok, round((t1 - t0) * 1e3), "ms")
import os
if os.environ.get("SLEEP"):
    time.sleep(float(os.environ["SLEEP"]))
groups = []
for g in range(int(os.environ.get("GROUPS", "10"))):
    t0 = time.perf_counter()
    for _ in range(5):
        nat.check_host(pin.numpy(), out=res.numpy())
    groups.append(round((time.perf_counter() - t0) / 5 * 1e3, 3))
print("ms/call per group", groups)
