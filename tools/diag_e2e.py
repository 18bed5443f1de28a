"""Timing breakdown of the host-buffer check path (diagnostic)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200 import _native as N

w = fx.franka7_world(); ck = w.checker(); nat = ck.native
n = 1 << 20
rng = np.random.default_rng(0)
Q = rng.uniform(w.lower, w.upper, size=(n, 7))
pin = torch.empty((n, 7), dtype=torch.float64, pin_memory=True); pin.copy_(torch.from_numpy(Q))
res = torch.empty(n, dtype=torch.uint8, pin_memory=True)
def t(f, reps=5):
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3
print("host pinned  ms", t(lambda: nat.check_host(pin.numpy(), out=res.numpy())))
print("host pageable ms", t(lambda: nat.check_host(Q)))
dq64 = torch.as_tensor(Q, device="cuda"); dq32 = dq64.float()
print("device f64 in ms", t(lambda: nat.check_device(dq64)))
print("device f32 in ms", t(lambda: nat.check_device(dq32)))
print("torch H2D pinned ms", t(lambda: dq64.copy_(pin, non_blocking=True)))
print("device f64 in, fp64 arith ms", t(lambda: nat.check_device(dq64, precision="fp64")))
