"""fp32 flags of the 2^20 config-2 golden rows against the reference's: how many differ (all inside
the 1e-5 contact band by the parity test) and how close to contact they are (oracle fp64 clearance)."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import ref  # noqa: E402
from paper_2504_10783_b200 import fixtures as fx  # noqa: E402

g = np.load(ROOT / "tests/golden/config2_1m.npz")
n = int(g["n"])
free_ref = np.unpackbits(g["free_bits"])[:n].astype(bool)
w = fx.franka7_world()
nat = w.checker().native
Q = fx.config2_rows()
free = nat.check_device(torch.as_tensor(Q, device="cuda")).cpu().numpy().astype(bool)
mism = np.nonzero(free != free_ref)[0]
clr = ref.OracleChecker(w).clearance(Q[mism].astype(np.float64)) if len(mism) else np.zeros(0)
print(f"{len(mism)} mismatches of {n} ({len(g['band'])} rows in the 1e-5 band); "
      f"max |clearance| of a mismatch {np.abs(clr).max() if len(clr) else 0:.3e}", flush=True)
