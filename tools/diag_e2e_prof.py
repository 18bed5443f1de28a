"""Host-side costs of the pageable check_batch path: numpy copy rate and EZ_HOST_PROFILE call times."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_10783_b200 import fixtures as fx
ck = fx.franka7_world().checker()
rows = [fx.config2_rows(1 << 20, seed=i) for i in range(2)]
for i in range(30):
    ck.check_batch(rows[i % 2])
t = time.perf_counter(); x = rows[0].copy(); print("numpy copy 28MB ms", (time.perf_counter() - t) * 1e3)
