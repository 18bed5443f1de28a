"""Time the specialised fp32 check kernel on 2^20 config-2-style rows (CUDA events, 8 rotating
batches > L2), 7-DOF and 14-DOF; prints checks/s and the CTA size picked."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_10783_b200 import fixtures as fx  # noqa: E402

for name, w in (("franka7", fx.franka7_world()), ("bimanual14", fx.bimanual14_world())):
    nat = w.checker().native
    lo = torch.as_tensor(w.lower, dtype=torch.float32, device="cuda")
    hi = torch.as_tensor(w.upper, dtype=torch.float32, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    B = [lo + (hi - lo) * torch.rand((1 << 20, w.model.dof), generator=g, device="cuda") for _ in range(8)]
    for i in range(6):
        nat.check_device(B[i % 8])
    torch.cuda.synchronize()
    best = 1e9
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(40):
            nat.check_device(B[i % 8])
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 40)
    print(f"{name}: {best * 1e3:.1f} us per 2^20 -> {(1 << 20) / (best * 1e-3) / 1e9:.2f}e9 checks/s  cta {nat.info()['check_cta']} variant {nat.info()['check_variant']}",
          flush=True)
