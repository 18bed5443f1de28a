"""Run the config-4 (14-DOF) and the bench 7-DOF EI-ZO regions once and save their polytopes
(gpurun_out/region{14,7}.npz) for the off-line face-redundancy analysis (tools/redundancy.py)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_10783_b200 import fixtures as fx  # noqa: E402
from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge  # noqa: E402
from paper_2504_10783_b200.polytope import HPolytope  # noqa: E402

out = Path(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out")
out.mkdir(exist_ok=True)
for tag, world in (("7", fx.franka7_world()), ("14", fx.bimanual14_world())):
    v1, v2 = fx.random_free_segment(world, seed=3)
    dom = HPolytope.from_bounds(world.lower, world.upper)
    ck = world.checker()
    ck.native.specialize(1)
    p = InflationParams(**fx.FRANKA_PARAMS)
    inflate_edge(Segment(v1, v2), dom, p, ck, seed=6)
    t0 = time.perf_counter()
    rep = inflate_edge(Segment(v1, v2), dom, p, ck, seed=7)
    wall = (time.perf_counter() - t0) * 1e3
    np.savez(out / f"region{tag}.npz", A=rep.polytope.A, b=rep.polytope.b, v1=v1, v2=v2, it=rep.iterations,
             checks=rep.collision_checks, device_ms=rep.device_ms, wall_ms=wall)
    print(f"region{tag}: it={rep.iterations} faces={rep.hyperplanes_added} checks={rep.collision_checks} "
          f"device {rep.device_ms:.2f} ms wall {wall:.2f} ms")
