"""Latency of the specialised check at bisection-sized batches (fp64 rows, fp32 arithmetic):
how long one dependent round of per-thread checks takes when the GPU is mostly idle."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_10783_b200 import fixtures as fx  # noqa: E402

w = fx.franka7_world()
nat = w.checker().native
nat.specialize(1) if hasattr(nat, "specialize") else None
lo = torch.as_tensor(w.lower, dtype=torch.float64, device="cuda")
hi = torch.as_tensor(w.upper, dtype=torch.float64, device="cuda")
g = torch.Generator(device="cuda")
g.manual_seed(1)
for n in (1024, 4096, 8192, 16384, 29000, 65536, 131072, 262144):
    B = [lo + (hi - lo) * torch.rand((n, 7), generator=g, device="cuda", dtype=torch.float64) for _ in range(4)]
    for i in range(5):
        nat.check_device(B[i % 4])
    torch.cuda.synchronize()
    best = 1e9
    for rep in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(20):
            nat.check_device(B[i % 4])
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 20)
    print(f"n={n:7d}: {best * 1e3:7.1f} us per launch  cta {nat.info()['check_cta']}", flush=True)
