"""fp64-arithmetic check rate (precision='fp64', the generic kernel) on config-2 rows, CUDA events."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_10783_b200 import fixtures as fx  # noqa: E402

w = fx.franka7_world()
nat = w.checker().native
B = [torch.as_tensor(fx.config2_rows(1 << 20, seed=i), device="cuda") for i in range(8)]
for i in range(6):
    nat.check_device(B[i % 8], precision="fp64")
torch.cuda.synchronize()
best = 1e9
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(16):
        nat.check_device(B[i % 8], precision="fp64")
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / 16)
print(f"fp64 arithmetic: {best * 1e3:.1f} us per 2^20 -> {(1 << 20) / (best * 1e-3) / 1e9:.2f}e9 checks/s", flush=True)
