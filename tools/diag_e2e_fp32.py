"""e2e through CollisionChecker.check_batch on host rows: pageable/pinned fp32 and fp64, per chunk size."""
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_10783_b200 import fixtures as fx  # noqa: E402

ck = fx.franka7_world().checker()
rows = [fx.config2_rows(1 << 20, seed=i) for i in range(4)]


def rate(batches, steps=10):
    t_w = time.perf_counter()
    i = 0
    while time.perf_counter() - t_w < 1.0:
        ck.check_batch(batches[i % len(batches)])
        i += 1
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        for i in range(steps):
            ck.check_batch(batches[i % len(batches)])
        ts.append(time.perf_counter() - t0)
    return (1 << 20) * steps / np.median(ts)


pin32 = []
for r in rows[:2]:
    t = torch.empty(r.shape, dtype=torch.float32, pin_memory=True)
    t.numpy()[:] = r
    pin32.append(t.numpy())
print(os.environ.get("EZ_HOST_CHUNK", "default"), f"pageable fp32 {rate(rows) / 1e9:.3f}e9/s  pinned fp32 {rate(pin32) / 1e9:.3f}e9/s "
      f" pageable fp64 {rate([r.astype(np.float64) for r in rows[:2]]) / 1e9:.3f}e9/s", flush=True)
