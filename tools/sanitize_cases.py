"""Small invocations of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): fused check (generic, specialised, fp64, host pipeline), hit-and-run (DMMA
and lane walks), EI-ZO (planar and one 7-DOF iteration: compaction, bisection, cluster/DSMEM
placement, draws), sharded session, voxelise + prune, collision-map build, k-NN adjacency."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_10783_b200 import fixtures as fx  # noqa: E402
from paper_2504_10783_b200.distributed import inflate_edge_sharded  # noqa: E402
from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge  # noqa: E402
from paper_2504_10783_b200.polytope import HPolytope, hit_and_run_sample  # noqa: E402
from paper_2504_10783_b200.roadmap import Grid, build_drm, collision_set  # noqa: E402
from paper_2504_10783_b200.scene import voxelize_point_cloud  # noqa: E402

w7 = fx.franka7_world()
Q = fx.config2_rows(4096)
gen = w7.checker(specialize=False)
jit = w7.checker(specialize=True)
f64 = w7.checker(precision="fp64", specialize=False)
a = gen.check_batch(torch.as_tensor(Q, device="cuda")).cpu().numpy()
b = jit.check_batch(torch.as_tensor(Q, device="cuda")).cpu().numpy()
c = f64.check_batch(Q)
d = jit.check_batch(Q)  # host pipeline
assert (a == b).all() and (b == d).all()
print("check ok", a.mean(), c.mean())
box = HPolytope.from_bounds(w7.lower, w7.upper)
X = hit_and_run_sample(box, fx.HOME7[None, :], 512, 8, seed=3).points
X2 = hit_and_run_sample(box, fx.HOME7[None, :], 512, 8, seed=3, rng="philox").points
print("hnr ok", X.shape, X2.shape)
arm = fx.arm3_world()
rep = inflate_edge(Segment(*fx.ARM3_SEGMENT), HPolytope.from_bounds(arm.lower, arm.upper), InflationParams(),
                   arm.checker(), seed=0)
print("eizo arm3 ok", rep.iterations, rep.hyperplanes_added)
v1, v2 = fx.random_free_segment(w7, seed=3)
p1 = InflationParams(**{**fx.FRANKA_PARAMS, "n_it": 1, "n_p": 2000})
rep = inflate_edge(Segment(v1, v2), box, p1, jit, seed=7)
print("eizo 7-DOF ok", rep.iterations, rep.hyperplanes_added)
rep = inflate_edge_sharded(Segment(*fx.ARM3_SEGMENT), HPolytope.from_bounds(arm.lower, arm.upper), InflationParams(),
                           arm.checker(), seed=0, shards=2)
print("sharded ok", rep.iterations)
grid = Grid(np.array([-0.75, -1.02, -0.36]), 0.06, (25, 34, 26))
base = fx.franka7_world(False)
drm = build_drm(base.model, base.checker(), base.lower, base.upper, 300, 10, 10.0, 10.0, grid, seed=0)
pts = np.random.default_rng(0).normal(size=(5000, 3)) * 0.2 + np.array([0.5, 0.0, 0.5])
cs = collision_set(drm, voxelize_point_cloud(pts, grid.side, grid.origin))
print("drm ok", drm.adj_ids.shape, len(cs))
torch.cuda.synchronize()
print("all cases done")
