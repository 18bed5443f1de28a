"""How far from contact can the fp32 check disagree with the reference's fp64 arithmetic?  Points
packed around collision boundaries (bisection on the fp32 check between free and colliding
configurations, every visited point kept), fp32 flags vs the oracle's fp64 flags: the largest
|fp64 clearance| of a disagreement bounds the fp32 contact band actually needed."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import ref  # noqa: E402
from paper_2504_10783_b200 import fixtures as fx  # noqa: E402

for name, w in (("franka7", fx.franka7_world()), ("bimanual14", fx.bimanual14_world())):
    nat = w.checker().native
    d = w.model.dof
    lo = torch.as_tensor(w.lower, dtype=torch.float64, device="cuda")
    hi = torch.as_tensor(w.upper, dtype=torch.float64, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    Q = lo + (hi - lo) * torch.rand((1 << 15, d), generator=g, device="cuda", dtype=torch.float64)
    f = nat.check_device(Q).bool()
    a, b = Q[f][:1500], Q[~f][:1500]
    n = min(len(a), len(b))
    a, b = a[:n], b[:n]
    pts = []
    for it in range(30):
        m = 0.5 * (a + b)
        fm = nat.check_device(m).bool()
        a = torch.where(fm[:, None], m, a)
        b = torch.where(fm[:, None], b, m)
        if it >= 12:
            pts.append(m)
    P = torch.cat(pts)
    f32 = nat.check_device(P).cpu().numpy().astype(bool)
    Pn = P.cpu().numpy()
    oc = ref.OracleChecker(w, workers=8)
    clr = oc.clearance(Pn)
    f64 = clr > 0
    mism = f32 != f64
    c = np.abs(clr[mism])
    print(f"{name}: {len(Pn)} boundary points (|clearance| median {np.median(np.abs(clr)):.2e}); "
          f"{int(mism.sum())} fp32/fp64 disagreements, |clearance| max {c.max() if len(c) else 0:.2e}, "
          f"99% {np.quantile(c, 0.99) if len(c) else 0:.2e}", flush=True)
