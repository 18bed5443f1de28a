"""Profiling driver: a few k_check launches on config 2 (1M 7-DOF configs vs 10k voxels)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2504_10783_b200 import fixtures as fx

w = fx.franka7_world()
nat = w.checker().native
lo = torch.as_tensor(w.lower, dtype=torch.float32, device="cuda")
hi = torch.as_tensor(w.upper, dtype=torch.float32, device="cuda")
g = torch.Generator(device="cuda"); g.manual_seed(1)
Q = lo + (hi - lo) * torch.rand((1 << 20, 7), generator=g, device="cuda")
prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
for _ in range(4):
    out = nat.check_device(Q, precision=prec)
torch.cuda.synchronize()
print("free fraction", out.float().mean().item(), nat.info())
