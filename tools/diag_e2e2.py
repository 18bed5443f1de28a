"""e2e host path: generic vs specialised kernel, repeated (variance check)."""
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
for mode in ("generic", "jit"):
    nat = w.checker().native
    nat.specialize(1 if mode == "jit" else -1)
    for _ in range(3):
        nat.check_host(pin.numpy(), out=res.numpy())
    ts = []
    for _ in range(10):
        t0 = time.perf_counter(); nat.check_host(pin.numpy(), out=res.numpy()); ts.append(time.perf_counter() - t0)
    print(mode, "ms per 1M: min %.3f median %.3f max %.3f" % (1e3 * min(ts), 1e3 * np.median(ts), 1e3 * max(ts)))
