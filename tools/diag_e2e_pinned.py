"""Pinned fp32 check_batch: Python wall per call vs the C call (EZ_HOST_PROFILE) vs the PCIe floor."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_10783_b200 import fixtures as fx  # noqa: E402

ck = fx.franka7_world().checker()
pins = []
for i in range(2):
    t = torch.empty((1 << 20, 7), dtype=torch.float32, pin_memory=True)
    t.numpy()[:] = fx.config2_rows(1 << 20, seed=i)
    pins.append(t.numpy())
for i in range(30):
    ck.check_batch(pins[i % 2])
ts = []
for i in range(20):
    t0 = time.perf_counter()
    ck.check_batch(pins[i % 2])
    ts.append(time.perf_counter() - t0)
print(f"pinned fp32 check_batch: median {np.median(ts) * 1e3:.3f} ms per 2^20 rows "
      f"({(1 << 20) / np.median(ts) / 1e9:.2f}e9/s); PCIe floor 29.36 MB / 54.9 GB/s = 0.535 ms", flush=True)
