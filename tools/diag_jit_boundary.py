"""Specialised vs generic fp32 check flags on configurations packed around collision boundaries
(points along segments from free to colliding configurations): mismatch counts per world."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_10783_b200 import fixtures as fx  # noqa: E402

for name, w in (("franka7", fx.franka7_world()), ("bimanual14", fx.bimanual14_world())):
    gen, jit = w.checker(specialize=False).native, w.checker(specialize=False).native
    assert jit.specialize(1)
    d = w.model.dof
    lo = torch.as_tensor(w.lower, dtype=torch.float64, device="cuda")
    hi = torch.as_tensor(w.upper, dtype=torch.float64, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    Q = lo + (hi - lo) * torch.rand((1 << 18, d), generator=g, device="cuda", dtype=torch.float64)
    f = gen.check_device(Q).bool()
    a, b = Q[f][: 1 << 15], Q[~f][: 1 << 15]
    n = min(len(a), len(b))
    t = torch.linspace(0, 1, 129, device="cuda", dtype=torch.float64)[:, None, None]
    P = (a[:n][None] + t * (b[:n] - a[:n])[None]).reshape(-1, d)
    # bisect each pair 24 times on the generic check, keeping every visited point
    lo_, hi_ = a[:n].clone(), b[:n].clone()
    pts = [P]
    for _ in range(24):
        m = 0.5 * (lo_ + hi_)
        fm = gen.check_device(m).bool()
        lo_ = torch.where(fm[:, None], m, lo_)
        hi_ = torch.where(fm[:, None], hi_, m)
        pts.append(m)
    P = torch.cat(pts)
    tot = 0
    for prec_rows in (P, P.float()):
        fg, fj = gen.check_device(prec_rows), jit.check_device(prec_rows)
        mism = (fg != fj).nonzero().flatten()
        tot += len(mism)
        print(f"{name} rows {prec_rows.dtype}: {len(prec_rows)} points, {len(mism)} mismatches", flush=True)
        if len(mism):
            torch.save(prec_rows[mism[:64]].cpu(), f"gpurun_out/jit_mismatch_{name}_{str(prec_rows.dtype)[6:]}.pt")
