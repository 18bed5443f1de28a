"""Specialised (NVRTC) vs generic check kernel: agreement and timing on config 2 (and config 4)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2504_10783_b200 import fixtures as fx

for name, mk in (("franka7", fx.franka7_world), ("bimanual14", fx.bimanual14_world)):
    w = mk()
    gen = w.checker().native
    jit = w.checker().native
    gen.specialize(-1)
    import os
    os.environ["EZ_JIT_DUMP"] = f"gpurun_out/jit_{name}.cu"
    t0 = time.perf_counter()
    ok = jit.specialize(1)
    t1 = time.perf_counter()
    from paper_2504_10783_b200 import _native as N
    print(f"{name}: specialised={ok} compile {1e3 * (t1 - t0):.0f} ms", flush=True)
    if not ok:
        print("  reason:", N.lib().ez_last_error().decode()[:3000])
    lo = torch.as_tensor(w.lower, dtype=torch.float32, device="cuda")
    hi = torch.as_tensor(w.upper, dtype=torch.float32, device="cuda")
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    Q = lo + (hi - lo) * torch.rand((1 << 20, w.model.dof), generator=g, device="cuda")
    a = gen.check_device(Q); b = jit.check_device(Q)
    a64 = gen.check_device(Q.double()); b64 = jit.check_device(Q.double())
    torch.cuda.synchronize()
    print(f"  mismatches f32 rows {int((a != b).sum())}, f64 rows {int((a64 != b64).sum())}, free {a.float().mean():.4f}")
    for lab, nat in (("generic", gen), ("jit", jit)):
        for _ in range(3):
            nat.check_device(Q)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            nat.check_device(Q)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"  {lab}: {ms:.3f} ms per 1M -> {1.048576e9 / ms * 1e-3 / 1e6 * 1e3:.3f} e9 checks/s")
