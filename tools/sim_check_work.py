"""CPU model of the specialised check kernel's work on config-2 rows: phase-A decisions, and for
phase-B survivors the position of the deciding test, voxel tests in/out of the distance grid and
in the quantised-distance ambiguity band (list walks).  Test order is read from a dumped kernel
source (tools/dump_jit.py)."""
import re
import sys
from pathlib import Path

import numpy as np
from scipy.spatial import cKDTree

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import ref  # noqa: E402
from paper_2504_10783_b200 import fixtures as fx  # noqa: E402

src = Path(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/jit_franka7.cu").read_text()
a_part, b_part = src.split("bool b(const Q* row", 1)
hot = [(int(x), int(y)) for x, y in re.findall(r"if \(sq3\(c(\d+)_0 - c(\d+)_0", a_part)]
vox_order = [int(x) for x in re.findall(r"voxel_decide<float>\(M\.vox, w\d, e\d, c(\d+)_0", b_part)]
world = fx.franka7_world()
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
Q = fx.config2_rows(n).astype(np.float64)
_, tr = ref.geometry_poses(world.model, Q)
C = np.stack(tr, axis=1)  # (n, S, 3)
S = C.shape[1]
R = 0.055 + world.vmap.sphere_radius
pairs = np.array(world.model.self_pairs)
pair_hit = np.linalg.norm(C[:, pairs[:, 0]] - C[:, pairs[:, 1]], axis=2) <= 0.11
hot_idx = [int(np.flatnonzero((pairs[:, 0] == min(p)) & (pairs[:, 1] == max(p)))[0]) for p in hot]
a_hit = pair_hit[:, hot_idx].any(axis=1)
tree = cKDTree(world.vmap.centers())
d, _ = tree.query(C.reshape(-1, 3), k=1)
d = d.reshape(n, S)
vox_hit = d <= R
# grid extent: lattice box of the cloud padded by 6 voxels (list radius), cells h = 0.01
idx = world.vmap.index_array()
lo = world.vmap.origin + (idx.min(0) - 6) * world.vmap.side
hi = world.vmap.origin + (idx.max(0) + 7) * world.vmap.side
in_grid = np.all((C >= lo) & (C < hi), axis=2)
h = 0.01
e = np.linalg.norm((C - lo) / h - np.floor((C - lo) / h) - 0.5, axis=2) * h
dq = 0.081 / 255
dc_lo, dc_hi = d - e, d + e  # the cell-centre distance is within e of d
amb = in_grid & ~((dc_lo - e > R) | (dc_hi + dq + e <= R))
surv = ~a_hit
print(f"rows {n}: colliding {(~ref.OracleChecker(world).check_batch(Q[:20000])).mean():.3f} (20k sample); "
      f"phase A decides {a_hit.mean():.3f}; survivors {surv.mean():.3f}")
# phase B sequence for survivors: voxel tests in vox_order, then the remaining pairs (any order)
first = np.full(n, -1)
vh = vox_hit[:, vox_order]
anyv = vh.any(axis=1)
first[anyv] = np.argmax(vh[anyv], axis=1)
rest_pairs = np.setdiff1d(np.arange(pairs.shape[0]), hot_idx)
pb = pair_hit[:, rest_pairs].any(axis=1)
s = surv
print(f"survivors: voxel hit {anyv[s].mean():.3f}, pair hit after voxels {(pb & ~anyv)[s].mean():.3f}, "
      f"free {(~anyv & ~pb)[s].mean():.3f}")
tests = np.where(first >= 0, first + 1, len(vox_order))
print(f"voxel tests per survivor: mean {tests[s].mean():.1f}; in grid {np.mean([in_grid[i, vox_order[:t]].sum() for i, t in zip(np.flatnonzero(s)[:5000], tests[s][:5000])]):.1f}; "
      f"ambiguous (list walk) {np.mean([amb[i, vox_order[:t]].sum() for i, t in zip(np.flatnonzero(s)[:5000], tests[s][:5000])]):.2f}")
warp = np.flatnonzero(s)[: (s.sum() // 32) * 32].reshape(-1, 32)
tw = tests[warp]
print(f"warp-level: lanes active per voxel test {np.mean(tw.sum(axis=1) / (tw.max(axis=1) * 32)):.2f} of 32 "
      f"(max tests per warp {tw.max(axis=1).mean():.1f})")
print("in-grid fraction of all spheres", in_grid.mean(), "per sphere", np.round(in_grid.mean(0), 2))
print("voxel hit rate per sphere in order", [round(float(vox_hit[s][:, k].mean()), 3) for k in vox_order])
