"""Pageable fp32 check_batch calls with EZ_HOST_PROFILE=2: per-call time split into host copies, API calls and stage waits."""
import sys, time
from pathlib import Path
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2504_10783_b200 import fixtures as fx
ck = fx.franka7_world().checker()
rows = [fx.config2_rows(1 << 20, seed=i) for i in range(2)]
for i in range(20):
    ck.check_batch(rows[i % 2])
import os
t=time.perf_counter()
for i in range(5):
    ck.check_batch(rows[i % 2])
print("per call ms", (time.perf_counter()-t)/5*1e3, flush=True)
