"""Time the specialised check kernel on config 2 under several EZ_JIT_* settings (one subprocess each)."""
import json, os, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]

CHILD = r'''
import sys, json, torch
sys.path.insert(0, %r)
from paper_2504_10783_b200 import fixtures as fx
w = fx.%s()
nat = w.checker().native
assert nat.specialize(1)
lo = torch.as_tensor(w.lower, dtype=torch.float32, device="cuda")
hi = torch.as_tensor(w.upper, dtype=torch.float32, device="cuda")
g = torch.Generator(device="cuda"); g.manual_seed(1)
Qs = [lo + (hi - lo) * torch.rand((1 << 20, w.model.dof), generator=g, device="cuda") for _ in range(8)]
ref = nat.check_device(Qs[0]).clone()
for i in range(5): nat.check_device(Qs[i %% 8])
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(40): nat.check_device(Qs[i %% 8])
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 40
print(json.dumps({"ms": ms, "gchecks": 1.048576 / ms, "free": float(ref.float().mean())}))
'''

def run(model, env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", CHILD % (str(ROOT), model)], env=e, capture_output=True, text=True, timeout=300)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-400:]
    return line

if __name__ == "__main__":
    configs = json.loads(sys.argv[1]) if len(sys.argv) > 1 else [{}]
    models = sys.argv[2].split(",") if len(sys.argv) > 2 else ["franka7_world"]
    for m in models:
        for env in configs:
            print(m, env, run(m, env), flush=True)
