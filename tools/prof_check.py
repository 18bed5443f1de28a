"""Profiling driver: a few k_check launches on config 2 (1M 7-DOF configs vs 10k voxels)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2504_10783_b200 import fixtures as fx

w = fx.franka7_world()
nat = w.checker().native
if "--generic" in sys.argv:
    nat.specialize(-1)
else:
    print("specialised:", nat.specialize(1))
lo = torch.as_tensor(w.lower, dtype=torch.float32, device="cuda")
hi = torch.as_tensor(w.upper, dtype=torch.float32, device="cuda")
g = torch.Generator(device="cuda"); g.manual_seed(1)
Q = lo + (hi - lo) * torch.rand((1 << 20, 7), generator=g, device="cuda")
prec = "fp64" if "fp64" in sys.argv else "fp32"
for _ in range(4):
    out = nat.check_device(Q, precision=prec)
torch.cuda.synchronize()
print("free fraction", out.float().mean().item(), nat.info())
