"""Profiling driver: box robot (scenes/box_arm3d.json) vs the config-2 cloud, 1M configs, generic kernel."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch
from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.scene import World, load_scene

arm = load_scene(ROOT / "scenes" / "box_arm3d.json")
world = World(arm.model, arm.static, fx.franka7_world().vmap, arm.lower, arm.upper)
nat = world.checker().native
lo = torch.as_tensor(world.lower, dtype=torch.float32, device="cuda")
hi = torch.as_tensor(world.upper, dtype=torch.float32, device="cuda")
Q = lo + (hi - lo) * torch.rand((1 << 20, 7), device="cuda")
for _ in range(3):
    out = nat.check_device(Q)
torch.cuda.synchronize()
print("free", float(out.float().mean()))
