"""Breakdown of the DRM online phase: points -> voxelize_point_cloud -> collision_set (config 5)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import bench
from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.roadmap import DeviceRoadmap, Drm, Grid, collision_set, sample_free_nodes
from paper_2504_10783_b200.scene import voxelize_point_cloud

grid = Grid(np.array([-0.75, -1.02, -0.36]), 0.06, (25, 34, 26))
base = fx.franka7_world(False)
nodes = sample_free_nodes(base, 100_000, seed=0)
rm = DeviceRoadmap.build(base, nodes, grid)
off, ids = rm.export()
drm = Drm(nodes, np.zeros(100_001, np.int64), np.zeros(0, np.int32), off, ids, np.zeros((100_000, 7)), grid)
pts = bench.clustered_cloud(100_000, 3, seed=3)
for _ in range(3):
    cs = collision_set(drm, voxelize_point_cloud(pts, 0.06, grid.origin))
T = {"h2d": [], "vox": [], "cs": [], "all": []}
for _ in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d = torch.as_tensor(pts, device="cuda"); torch.cuda.synchronize()
    t1 = time.perf_counter()
    vm = voxelize_point_cloud(pts, 0.06, grid.origin)
    t2 = time.perf_counter()
    cs = collision_set(drm, vm)
    t3 = time.perf_counter()
    T["h2d"].append(t1 - t0); T["vox"].append(t2 - t1); T["cs"].append(t3 - t2); T["all"].append(t3 - t1)
print({k: round(1e3 * float(np.median(v)), 3) for k, v in T.items()}, "ms; voxels", vm.n_occupied, "blocked", len(cs.ids))

# finer split of collision_set
import paper_2504_10783_b200.roadmap as R
vm = voxelize_point_cloud(pts, 0.06, grid.origin)
dm = drm.device_map()
tt = {"allclose": [], "blocked_bits": [], "cpu": [], "unpack": []}
for _ in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    same = bool(np.allclose(vm.origin, drm.grid.origin) and np.isclose(vm.side, drm.grid.side))
    t1 = time.perf_counter()
    bits, _ = dm.blocked_bits(vm, same, count=False)
    t2 = time.perf_counter()
    words = bits.cpu().numpy().view(np.uint32)
    t3 = time.perf_counter()
    flags = np.unpackbits(words.view(np.uint8), bitorder="little")[: drm.n_nodes]
    ids_ = np.flatnonzero(flags).astype(np.int64)
    t4 = time.perf_counter()
    for k, a, b in (("allclose", t0, t1), ("blocked_bits", t1, t2), ("cpu", t2, t3), ("unpack", t3, t4)):
        tt[k].append(b - a)
print({k: round(1e3 * float(np.median(v)), 3) for k, v in tt.items()}, "ms")
