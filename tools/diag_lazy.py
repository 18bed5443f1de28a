"""First-call latency of the hit-and-run paths (CUDA lazy module loading)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2504_10783_b200.polytope import HPolytope, hit_and_run_sample

torch.zeros(1, device="cuda")
rng = np.random.default_rng(0)
for F in (200, 200, 20, 20, 120):
    A = rng.normal(size=(F, 14)); A /= np.linalg.norm(A, axis=1, keepdims=True)
    p = HPolytope(A, np.full(F, 0.5))
    t0 = time.perf_counter()
    hit_and_run_sample(p, np.zeros((1, 14)), 1000, 10, seed=1)
    print(f"F={F}: {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
