#!/usr/bin/env python
"""Benchmark of the EI-ZO hot path (BASELINE.json): collision checks/s, 7-DOF vs 10k voxel spheres.

One step = one pass of the fused FK + collision kernel over a batch of 2^20
7-DOF configurations (config 2 of BASELINE.json) per GPU.  Weak scaling: each
rank checks its own batches (no data-path collective); the whole-job value is
all configurations / the max-over-ranks device time.  Inputs are 8 resident
batches (224 MB > the 126 MB L2) used in rotation, so no step reads its
configurations from L2.  Batch 0 of rank 0 is ``fixtures.config2_rows()``, the
rows whose reference flags tests/golden/config2_1m.npz holds.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

``--gpus N`` outside torchrun re-launches itself under torch.distributed.run
with N ranks (one per GPU, NCCL).

Extra keys: ``roofline`` (FP32-FMA bound; measured FMA peak), ``cpu_baseline``
(the oracle port on this host, bounded sample), ``e2e`` (the drop-in numpy
call ``CollisionChecker.check_batch`` on pageable fp32 rows, copies inside the
timed region; pinned and fp64 variants beside it), ``eizo`` (7-DOF region
latency, its roofline and CPU baseline), ``config1``/``config3``/``config4``/
``drm``/``boxes``, ``clocks``.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "collision checks/sec (7-DOF, 10k obstacle spheres); EI-ZO ms per segment region"
UNIT = "checks/s"
BATCH = 1 << 20          # configurations per step per GPU (config 2: 1M configs)
N_BATCHES = 8            # rotating resident batches: 8 x 28 MB > L2
FLOP_PER_CHECK = 3416    # FK + spheres + 232 pairs + 33 obstacle tests


def _rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


_BACKEND = {"name": "nccl"}


def _max_over_ranks(x: float, world_size: int) -> float:
    """Max of a host scalar over ranks (NCCL: on the device; gloo test mode: on the host)."""
    if world_size == 1:
        return float(x)
    import torch
    import torch.distributed as dist

    dev = "cuda" if _BACKEND["name"] == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _barrier(world_size: int) -> None:
    if world_size > 1:
        import torch.distributed as dist

        dist.barrier()


def _comm(world_size: int):
    from paper_2504_10783_b200.distributed import LocalComm, TorchComm

    if world_size == 1:
        return LocalComm()
    return TorchComm() if _BACKEND["name"] == "nccl" else TorchComm(device="cpu")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons, sampled every 100 ms over a window of untimed steps
    that brackets the (millisecond-long) timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._p = None
        self._t = None

    def __enter__(self):
        try:
            self._p = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self._p = None
        return self

    def wait_first(self, timeout: float = 15.0) -> None:
        """Block until nvidia-smi has produced a sample (its start-up can take a second)."""
        t_end = time.perf_counter() + timeout
        while self._p is not None and not self.samples and time.perf_counter() < t_end:
            time.sleep(0.01)

    def _read(self):
        for line in self._p.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def __exit__(self, *exc):
        if self._p is not None:
            time.sleep(0.25)
            self._p.terminate()
            try:
                self._p.wait(timeout=2)
            except Exception:
                self._p.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [s[0] for s in self.samples]
        mx = max(s[1] for s in self.samples)
        bits = 0
        for s in self.samples:
            bits |= s[2]
        names = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
                 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
                 0x100: "display_clock_setting"}
        reasons = [n for b, n in names.items() if bits & b]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": reasons, "samples": len(sm),
                "window": "0.4 s of untimed steps, the timed region, 0.4 s of untimed steps"}


def _measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            pass
    return {}


def cpu_model() -> str:
    """The host CPU's model name (/proc/cpuinfo), for the CPU-baseline lines."""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_oracle_rate(world, n: int, workers: int) -> dict:
    """The oracle port (numpy + cKDTree, oracle/ref.py) on a bounded sample of the same workload."""
    from oracle import ref

    rng = np.random.default_rng(1)
    Q = rng.uniform(world.lower, world.upper, size=(n, len(world.lower))).astype(np.float32).astype(np.float64)
    ck = ref.OracleChecker(world, workers=workers)
    ck.check_batch(Q[:256])
    t0 = time.perf_counter()
    ck.check_batch(Q)  # cKDTree queries use `workers` threads; numpy FK / pairs are single threaded
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": UNIT, "cores": workers, "kind": "port",
            "sample": f"{n} uniform 7-DOF configs, oracle/ref.py (numpy+cKDTree restatement of world.py:483-565)",
            "cpu": cpu_model(), "host_cpus": os.cpu_count()}


def clustered_cloud(n_points: int, n_blobs: int, seed: int = 0) -> np.ndarray:
    """Synthetic perception: Gaussian blobs in front of the arm."""
    rng = np.random.default_rng(seed)
    per = n_points // n_blobs
    pts = []
    for _ in range(n_blobs):
        c = rng.uniform([0.3, -0.6, 0.0], [0.9, 0.6, 1.0])
        r = rng.uniform(0.03, 0.10)
        pts.append(c + rng.normal(size=(per, 3)) * r / 2)
    return np.concatenate(pts)


def bench_config1(cpu: bool = True) -> dict:
    """Config 1: EI-ZO of the 3-DOF planar arm's segment with the reference's default parameters,
    on the GPU and (CPU baseline) through the oracle port, the reference's own CPU-runnable case."""
    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge
    from paper_2504_10783_b200.polytope import HPolytope

    world = fx.arm3_world()
    v1, v2 = fx.ARM3_SEGMENT
    dom = HPolytope.from_bounds(world.lower, world.upper)
    ck = world.checker()
    inflate_edge(Segment(v1, v2), dom, InflationParams(), ck, seed=0)
    walls = []
    for _ in range(5):
        t0 = time.perf_counter()
        rep = inflate_edge(Segment(v1, v2), dom, InflationParams(), ck, seed=0)
        walls.append((time.perf_counter() - t0) * 1e3)
    out = {"ms_per_region_wall": float(np.median(walls)), "device_ms": rep.device_ms, "iterations": rep.iterations,
           "faces": rep.hyperplanes_added, "collision_checks": rep.collision_checks,
           "workload": "3-link planar arm among 3 discs + table, ARM3 segment, default InflationParams, seed 0"}
    if cpu:
        from oracle import ref
        t0 = time.perf_counter()
        r = ref.inflate_edge(v1, v2, dom.A, dom.b, ref.OracleChecker(world, workers=1), seed=0)
        out["cpu_oracle_ms"] = (time.perf_counter() - t0) * 1e3
        out["cpu_iterations"] = r["iterations"]
        out["cpu_collision_checks"] = r["collision_checks"]
    return out


def bench_boxes(checks_n: int = 1 << 20) -> dict:
    """Robot boxes: a Franka-like chain of 8 oriented boxes + a tool sphere
    (scenes/box_arm3d.json) against the config-2 cloud; generic kernel (box SAT, box vs voxel
    lattice through the occupancy bitmap)."""
    import torch

    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.scene import World, load_scene

    arm = load_scene(ROOT / "scenes" / "box_arm3d.json")
    cloud = fx.franka7_world().vmap
    world = World(arm.model, arm.static, cloud, arm.lower, arm.upper)
    nat = world.checker().native
    lo = torch.as_tensor(world.lower, dtype=torch.float32, device="cuda")
    hi = torch.as_tensor(world.upper, dtype=torch.float32, device="cuda")
    Q = lo + (hi - lo) * torch.rand((checks_n, world.model.dof), device="cuda")
    for _ in range(3):
        out = nat.check_device(Q)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        nat.check_device(Q)
    e1.record()
    torch.cuda.synchronize()
    return {"checks_per_s": 5 * checks_n / (e0.elapsed_time(e1) * 1e-3), "free_fraction": float(out.float().mean()),
            "workload": "8 robot boxes + 1 sphere, 20 self pairs (box-box SAT, sphere-box), 1 static box, 10k voxels"}


def bench_config4(checks_n: int = 1 << 20, cpu: bool = True, fp64_peak: float = 0.0) -> dict:
    """Config 4: 14-DOF bimanual (66 spheres, 1,248 pairs): checks/s and one EI-ZO region."""
    import torch

    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge
    from paper_2504_10783_b200.polytope import HPolytope

    world = fx.bimanual14_world()
    t_jit = time.perf_counter()
    ck = world.checker()  # "auto" specialisation at creation; also used by the EI-ZO loop below
    nat = ck.native
    jit_ms = (time.perf_counter() - t_jit) * 1e3
    specialised = nat.specialize(0)
    lo = torch.as_tensor(world.lower, dtype=torch.float32, device="cuda")
    hi = torch.as_tensor(world.upper, dtype=torch.float32, device="cuda")
    Q = lo + (hi - lo) * torch.rand((checks_n, 14), device="cuda")
    for _ in range(3):
        nat.check_device(Q)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        nat.check_device(Q)
    e1.record()
    torch.cuda.synchronize()
    rate = 5 * checks_n / (e0.elapsed_time(e1) * 1e-3)
    v1, v2 = fx.random_free_segment(world, seed=3)
    dom = HPolytope.from_bounds(world.lower, world.upper)
    params = InflationParams(**fx.FRANKA_PARAMS)
    rep = inflate_edge(Segment(v1, v2), dom, params, ck, seed=7)
    t0 = time.perf_counter()
    rep = inflate_edge(Segment(v1, v2), dom, params, ck, seed=7)
    wall = (time.perf_counter() - t0) * 1e3
    flop, walk_gemm = region_flop(rep, params, 14, dom.n_faces, 13104)
    out = {"checks_per_s": rate, "flop_per_check": 13104, "specialised_kernel": specialised, "jit_compile_ms": jit_ms,
           "cta": nat.info()["check_cta"],
           "eizo_ms_wall": wall, "eizo_device_ms": rep.device_ms, "iterations": rep.iterations,
           "faces": rep.hyperplanes_added, "collision_checks": rep.collision_checks,
           "terminated_by": rep.terminated_by,
           "eizo_roofline": {"bound": "FP64 tensor (DMMA) in the walk", "flop_per_region": flop,
                             "walk_gemm_flop": walk_gemm,
                             "achieved_tflops": flop / (rep.device_ms * 1e-3) / 1e12,
                             "peak_tflops": fp64_peak,
                             "walk_dmma_bound_ms": walk_gemm / (fp64_peak * 1e12) * 1e3 if fp64_peak else None,
                             "frac_of_dmma_bound": (walk_gemm / (fp64_peak * 1e12)) / (rep.device_ms * 1e-3)
                             if fp64_peak else None,
                             "note": "93% of the region is the walk over up to 1,860 faces; an LP analysis "
                                     "(tools/redundancy.py) finds <3% of the faces redundant"},
           "workload": "14-DOF bimanual sphere model vs 10k voxels; EI-ZO single segment, Franka (eps, delta)"}
    if cpu:
        from oracle import ref

        oc = ref.OracleChecker(world, workers=os.cpu_count() or 1)
        rows = np.random.default_rng(2).uniform(world.lower, world.upper, size=(4000, 14))
        t0 = time.perf_counter()
        oc.check_batch(rows)
        t_chk = (time.perf_counter() - t0) / rows.shape[0]
        out["cpu_baseline"] = {"kind": "port", "cores": os.cpu_count(), "cpu": cpu_model(),
                               "checks_per_s": 1.0 / t_chk,
                               "sample": "4,000 uniform 14-DOF configs through oracle/ref.py",
                               "region_checks_alone_s": rep.collision_checks * t_chk,
                               "note": "the full region (187 iterations, walks over up to 1,860 faces) is "
                                       "not affordable on the CPU; its checks alone take region_checks_alone_s"}
    return out


def bench_drm(n_nodes: int = 100_000, reps: int = 10, cpu: bool = True) -> dict:
    """Config 5: point cloud -> active voxels -> blocked nodes on a 25x34x26 grid, 100k-node roadmap."""
    import torch

    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.roadmap import DeviceRoadmap, Drm, Grid, collision_set, sample_free_nodes
    from paper_2504_10783_b200.scene import voxelize_point_cloud

    grid = Grid(np.array([-0.75, -1.02, -0.36]), 0.06, (25, 34, 26))
    base = fx.franka7_world(False)
    sample_free_nodes(base, n_nodes, seed=0)  # warm-up: compiles the specialised check kernel once
    t0 = time.perf_counter()
    nodes = sample_free_nodes(base, n_nodes, seed=0)
    t_nodes = time.perf_counter() - t0
    builds = []
    for _ in range(3):  # first build maps the pool and loads the kernels; report it and the median
        t0 = time.perf_counter()
        rm = DeviceRoadmap.build(base, nodes, grid)
        torch.cuda.synchronize()
        builds.append(time.perf_counter() - t0)
    t_map = float(np.median(builds))
    off, ids = rm.export()
    drm = Drm(nodes, np.zeros(n_nodes + 1, np.int64), np.zeros(0, np.int32), off, ids, np.zeros((n_nodes, 7)), grid)
    out = {"grid": "25x34x26 side 0.06", "n_nodes": n_nodes, "cmap_nnz": int(ids.shape[0]),
           "node_sampling_s": t_nodes, "cmap_build_s": t_map, "cmap_first_build_s": builds[0], "clouds": []}
    # 10^5-point clouds at the paper's ~360 active voxels, and the survey's
    # stress case: 10^6 points, ~2k active voxels
    for n_pts, blobs in ((100_000, 3), (100_000, 8), (1_000_000, 30)):
        pts = clustered_cloud(n_pts, blobs, seed=blobs)
        vm = voxelize_point_cloud(pts, grid.side, grid.origin)
        cs = collision_set(drm, vm)
        times = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            vm = voxelize_point_cloud(pts, grid.side, grid.origin)
            cs = collision_set(drm, vm)
            times.append((time.perf_counter() - t0) * 1e3)
        rec = {"points": pts.shape[0], "blobs": blobs, "active_voxels": vm.n_occupied, "blocked": len(cs),
               "voxelize_plus_prune_ms": float(np.median(times))}
        if cpu:
            from oracle import ref

            t0 = time.perf_counter()
            idx = ref.voxelize(pts, grid.side, grid.origin)
            blocked = ref.collision_set(off, ids, grid.origin, grid.side, grid.extents, idx, grid.origin, grid.side)
            rec["cpu_port_ms"] = (time.perf_counter() - t0) * 1e3
            rec["cpu_matches"] = bool(np.array_equal(blocked, cs.ids))
        out["clouds"].append(rec)
    # the whole drop-in build_drm (drm.py:207-255): reference draws, fp64 checks, poses, k-NN
    # adjacency (k = 10, d_cs = 1.5, d_ts = 0.5) and the collision map, 100k nodes
    from paper_2504_10783_b200.roadmap import build_drm

    base64 = base.checker(precision="fp64")
    build_drm(base.model, base64, base.lower, base.upper, 2000, 10, 1.5, 0.5, grid, seed=1)  # warm-up
    t0 = time.perf_counter()
    full = build_drm(base.model, base64, base.lower, base.upper, n_nodes, 10, 1.5, 0.5, grid, seed=1)
    torch.cuda.synchronize()
    out["build_drm"] = {"seconds": time.perf_counter() - t0, "n_nodes": n_nodes, "k": 10, "d_cs": 1.5, "d_ts": 0.5,
                        "adj_nnz": int(full.adj_ids.shape[0]), "cmap_nnz": int(full.cmap_ids.shape[0]),
                        "reference_estimate": "SURVEY 8(d): ~15 min on the CPU for a 100k-node build"}
    return out


CONFIG2 = {"workload": "config 2: Franka-like 7-DOF (33 spheres r=0.055, 232 self pairs) vs 10k voxel "
                       "spheres (side 0.02), uniform fp32 configs in the joint limits (default_rng)",
           "configs_per_step_per_gpu": BATCH, "l2": "8 rotating resident batches (224 MB > L2)"}


def run_reference(args):
    """The reference arm: the reference's CPU algorithm for config 2 on this host's cores.  The
    reference package cannot travel to the GPU box (/root/reference is absent there), so this is
    its restatement oracle/ref.py (kind "port": numpy FK and pairs, the reference's own
    scipy.spatial.cKDTree for the voxel query, all host threads), pinned to the reference's flags
    by tests/test_oracle_goldens.py; the reference package itself measured 3.8e3 checks/s
    (SURVEY.md §6).  Each step checks a bounded sample of the config-2 rows."""
    rank, world_size, _ = _rank()
    if rank != 0:
        return
    from paper_2504_10783_b200 import fixtures as fx

    world = fx.franka7_world()
    cores = os.cpu_count() or 1
    n = 20_000
    vals = []
    for _ in range(args.warmup):
        cpu_oracle_rate(world, 2_000, cores)
    t_steps = []
    for _ in range(args.steps):
        r = cpu_oracle_rate(world, n, cores)
        vals.append(r["value"])
        t_steps.append(n / r["value"])
    value = float(np.median(vals))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(t_steps)), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(CONFIG2),
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{n} config-2 rows per step (bounded sample of the {BATCH}-row step), "
                                       f"oracle/ref.py (restatement of world.py:483-565) with {cores} threads",
                             "cpu": cpu_model(), "host_cpus": os.cpu_count(),
                             "note": "the reference package itself: 3.8e3 checks/s (SURVEY.md §6); the port is "
                                     "~16x faster, so ratios against it are conservative"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def region_flop(rep, params, d: int, f0: int, flop_per_check: float, n_b: int = 11):
    """SURVEY.md §8(d) algorithmic FLOP of one EI-ZO region from its report:
    sum_k N_k N_ms (4 F_k d + 2 F_k + 6 d) + checks * F_check + C N_f 2 d, with N_k = max(N_p, M_k)
    (inflation.py:156-161, 288-290), F_k = F_0 + faces placed before iteration k, and the
    candidates C from the reference's own count (collision_checks = sum N_k + C (1 + N_b)).
    Returns (total, walk GEMM part sum_k N_k N_ms 4 F_k d)."""
    from paper_2504_10783_b200.eizo import required_batch_size

    walks, walk_total, walk_gemm, faces, placed = 0, 0.0, 0.0, f0, 0
    for k in range(1, rep.iterations + 1):
        n_k = max(params.n_p, required_batch_size(k, params))
        walks += n_k
        walk_gemm += n_k * params.n_ms * 4.0 * faces * d
        walk_total += n_k * params.n_ms * (4.0 * faces * d + 2.0 * faces + 6.0 * d)
        step = min(params.n_f, rep.hyperplanes_added - placed)
        placed += step
        faces += step
    cands = max(0, rep.collision_checks - walks) / (1 + n_b)
    total = walk_total + rep.collision_checks * flop_per_check + cands * params.n_f * 2.0 * d
    return total, walk_gemm


def _peak(fn_name: str, device: int) -> float:
    from paper_2504_10783_b200 import _native as N

    tf, ms = N.C.c_double(0.0), N.C.c_double(0.0)
    N.check(getattr(N.lib(), fn_name)(device, N.C.byref(tf), N.C.byref(ms)))
    return float(tf.value)


def bench_eizo7(world, ck, cpu: bool, fp64_peak: float) -> dict:
    """7-DOF single-segment region (Franka parameters): latency, roofline, CPU baseline."""
    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge
    from paper_2504_10783_b200.polytope import HPolytope

    v1, v2 = fx.random_free_segment(world, seed=3)
    dom = HPolytope.from_bounds(world.lower, world.upper)
    params = InflationParams(**fx.FRANKA_PARAMS)
    inflate_edge(Segment(v1, v2), dom, params, ck, seed=6)  # warm-up (module load, workspace)
    times, reps = [], []
    for s_ in range(5):
        t_r = time.perf_counter()
        rep = inflate_edge(Segment(v1, v2), dom, params, ck, seed=7 + (s_ % 4))
        times.append((time.perf_counter() - t_r) * 1e3)
        reps.append(rep)
    seed7 = reps[0]
    flop, walk_flop = region_flop(seed7, params, 7, dom.n_faces, FLOP_PER_CHECK)
    out = {"ms_per_region_wall": float(np.median(times)),
           "device_ms": float(np.median([r.device_ms for r in reps])),
           "seed7": {"iterations": seed7.iterations, "faces": seed7.hyperplanes_added,
                     "collision_checks": seed7.collision_checks, "device_ms": seed7.device_ms,
                     "matches_reference_counters": [seed7.iterations, seed7.hyperplanes_added,
                                                    seed7.collision_checks] == [6, 50, 295128]},
           "iterations": [r.iterations for r in reps], "faces": [r.hyperplanes_added for r in reps],
           "collision_checks": [r.collision_checks for r in reps],
           "segment": "7-DOF Franka-like + 10k voxels, length 0.6, free with margin 0.02 (default_rng(3))",
           "params": "delta=eps=0.005, N_p=1e4, N_f=10, N_ms=60, delta_max=0.01, N_b=11",
           "target_ms": 5.0,
           "roofline": {"bound": "critical path (latency); FP64 tensor (walk)",
                        "flop_per_region": flop, "walk_gemm_flop": walk_flop,
                        "achieved": flop / (seed7.device_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                        "peak": fp64_peak, "frac": flop / (seed7.device_ms * 1e-3) / 1e12 / fp64_peak,
                        "peak_source": "ez_fp64_tc_peak (DMMA m8n8k4) measured in this run",
                        "note": "SURVEY 8(d) per-region FLOP / device time; the region is a chain of "
                                "~6 dependent iterations of 5 kernels, see profiles/r01_eizo7_region_trace.txt"}}
    if cpu:
        from oracle import ref

        t0 = time.perf_counter()
        r1 = ref.inflate_edge(v1, v2, dom.A, dom.b, ref.OracleChecker(world, workers=os.cpu_count() or 1),
                              seed=7, n_it=1, **{k: v for k, v in fx.FRANKA_PARAMS.items()})
        t1 = time.perf_counter() - t0
        out["cpu_baseline"] = {
            "kind": "port", "cores": os.cpu_count(), "cpu": cpu_model(),
            "sample": "iteration 1 of the same region (oracle/ref.py inflate_edge, n_it=1, seed 7): "
                      f"{r1['collision_checks']} checks, {r1['hyperplanes_added']} faces",
            "first_iteration_s": t1,
            "reference_full_region_s": 93.7,
            "reference_full_region_note": "the reference package's own inflate_edge on this segment/seed, "
                                          "measured in the build container (tests/golden/region7.npz ref_seconds)"}
    return out


def bench_config3(world, ck, comm, world_size: int, rank: int) -> dict:
    """Config 3: 10-segment 7-DOF paths.  Latency of one path (sequential drop-in inflate_path and
    segment-sharded speculation, both with the reference's seeding) and segments/s over a stream
    of paths sharded across ranks (weak scaling: 8 paths per rank, all in flight at once)."""
    import torch

    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.corridor import inflate_path
    from paper_2504_10783_b200.distributed import inflate_paths_sharded, inflate_segments_sharded
    from paper_2504_10783_b200.eizo import InflationParams
    from paper_2504_10783_b200.polytope import HPolytope
    from paper_2504_10783_b200.roadmap import PwlPath

    path = PwlPath(fx.random_free_path(world, 10, seed=3))
    dom = HPolytope.from_bounds(world.lower, world.upper)
    params = InflationParams(**fx.FRANKA_PARAMS)

    def max_over_ranks(x):
        return _max_over_ranks(x, world_size)

    def barrier():
        _barrier(world_size)
        torch.cuda.synchronize()

    out = {"segments": 10, "path": "10 chained 0.6-long segments, free with margin 0.02 (default_rng(3))"}
    seq = inflate_path(path, dom, params, ck, seed=11)  # warm-up
    t0 = time.perf_counter()
    seq = inflate_path(path, dom, params, ck, seed=11)
    out["sequential_drop_in_ms"] = (time.perf_counter() - t0) * 1e3
    out["sets_kept"] = len(seq.sets)
    inflate_segments_sharded(path, dom, params, ck, seed=11, comm=comm)  # warm-up
    barrier()
    t0 = time.perf_counter()
    scs, mine = inflate_segments_sharded(path, dom, params, ck, seed=11, comm=comm)
    torch.cuda.synchronize()
    out["sharded_speculative_ms_max_over_ranks"] = max_over_ranks((time.perf_counter() - t0) * 1e3)
    out["sharded_equals_sequential"] = (scs.coverage == seq.coverage and all(
        np.array_equal(a.A, b.A) for a, b in zip(scs.sets, seq.sets)))
    out["sharded_reinflated"] = scs.reinflated
    out["path_latency_ms"] = min(out["sequential_drop_in_ms"], out["sharded_speculative_ms_max_over_ranks"])
    # throughput: a stream of paths, 8 per rank in flight (8 gives 2.8k segments/s on one GPU,
    # 4 gives 2.2k: tools/diag_stream.py), each through inflate_path (reference semantics)
    per_rank = 8
    paths = [PwlPath(fx.random_free_path(world, 10, seed=100 + p)) for p in range(per_rank * world_size)]
    inflate_paths_sharded(paths, dom, params, ck, seed=5, comm=comm, concurrency=per_rank)  # warm-up (workspaces)
    barrier()
    t0 = time.perf_counter()
    got = inflate_paths_sharded(paths, dom, params, ck, seed=5, comm=comm, concurrency=per_rank)
    torch.cuda.synchronize()
    dt = max_over_ranks(time.perf_counter() - t0)
    out["stream"] = {"paths": len(paths), "paths_per_rank": per_rank, "segments": 10 * len(paths),
                     "inflations_on_rank0": sum(len(s.sets) for s in got.values()) if rank == 0 else None,
                     "seconds_max_over_ranks": dt, "segments_per_s": 10 * len(paths) / dt,
                     "scaling": "weak (8 paths per rank in flight, no collective)"}
    return out


def bench_e2e(ck, host_batches, world_size: int, steps: int) -> dict:
    """End to end through the drop-in call: ``CollisionChecker.check_batch(numpy)`` -> one
    ``ez_check_batch_host`` per step; the H2D copy of the step's rows and the D2H read of its
    flags are inside the timed region.  Pageable fp32 (the headline), pinned fp32, pinned fp64."""
    import torch
    import torch.distributed as dist

    def timed(batches, label):
        gc.collect()
        t_w, n_w = time.perf_counter(), 0
        while n_w < 3 or time.perf_counter() - t_w < 1.0:  # copies run slower in a buffer's first second
            ck.check_batch(batches[n_w % len(batches)])
            n_w += 1
        _barrier(world_size)
        groups = []
        for _ in range(3):
            t_e = time.perf_counter()
            for i in range(steps):
                ck.check_batch(batches[i % len(batches)])
            groups.append(time.perf_counter() - t_e)
        return BATCH * steps * world_size / _max_over_ranks(float(np.median(groups)), world_size)

    pageable = host_batches
    pinned32 = []
    for hb in host_batches[:2]:
        t = torch.empty(hb.shape, dtype=torch.float32, pin_memory=True)
        t.numpy()[:] = hb
        pinned32.append(t.numpy())
    pinned64 = []
    for hb in host_batches[:2]:
        t = torch.empty(hb.shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[:] = hb
        pinned64.append(t.numpy())
    e_steps = max(3, min(steps, 10))
    return {"pageable_fp32": timed(pageable, "pageable"), "pinned_fp32": timed(pinned32, "pinned"),
            "pinned_fp64": timed(pinned64, "pinned64"), "steps": e_steps,
            "h2d_bytes_per_step": BATCH * 7 * 4, "d2h_bytes_per_step": BATCH}


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world_size, local_rank = _rank()
    if world_size != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world_size}")
    # one GPU per rank; the gloo test mode (--dist-backend gloo) may put several ranks on one GPU
    gpu = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    _BACKEND["name"] = args.dist_backend
    if world_size > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    from paper_2504_10783_b200 import _native as N
    from paper_2504_10783_b200 import fixtures as fx
    world = fx.franka7_world()
    t_jit = time.perf_counter()
    ck = world.checker()  # "auto": the model-specialised kernel is compiled with the device world
    nat = ck.native
    jit_ms = (time.perf_counter() - t_jit) * 1e3
    specialised = nat.specialize(0)
    # config 2 rows: U(joint limits) from default_rng, fp32; rank 0 batch 0 = the golden rows
    host_batches = [fx.config2_rows(BATCH, seed=rank * N_BATCHES + i) for i in range(N_BATCHES)]
    batches = [torch.as_tensor(h, device=dev) for h in host_batches]
    out = torch.empty(BATCH, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream

    def step(i, precision=0):
        N.check(N.lib().ez_check_batch(nat.handle, batches[i % N_BATCHES].data_ptr(), 0, BATCH, 7, out.data_ptr(),
                                       precision, sh))

    gc.collect()
    for i in range(max(3, args.warmup)):
        step(i)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    _barrier(world_size)
    torch.cuda.synchronize()

    def busy(seconds: float) -> None:
        # untimed steps around the timed region, so the 100 ms clock samples
        # see the GPU under this load (the timed region itself is milliseconds)
        t_end = time.perf_counter() + seconds
        i = 0
        while time.perf_counter() < t_end:
            step(i)
            i += 1
            if i % 64 == 0:
                torch.cuda.synchronize()
        torch.cuda.synchronize()

    with ClockSampler(gpu) as clk:
        clk.wait_first()
        busy(0.4)
        _barrier(world_size)
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            step(i)
            ev[i][1].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
        _barrier(world_size)
        busy(0.4)
    _barrier(world_size)
    total_ms = t0.elapsed_time(t1)
    launch_ms = [a.elapsed_time(b) for a, b in ev]
    max_ms = _max_over_ranks(total_ms, world_size)
    checks = BATCH * args.steps * world_size
    value = checks / (max_ms * 1e-3)
    step(0)
    free_frac = float(out.float().mean().item())
    # the reference's own arithmetic (fp64 kinematics and distances) on the same rows
    e64a, e64b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step(0, 1)
    e64a.record(stream)
    for i in range(4):
        step(i, 1)
    e64b.record(stream)
    torch.cuda.synchronize()
    fp64_rate = 4 * BATCH / (e64a.elapsed_time(e64b) * 1e-3)

    e2e = bench_e2e(ck, host_batches, world_size, max(3, min(args.steps, 10)))
    comm = _comm(world_size)
    fp64_peak = _peak("ez_fp64_tc_peak", gpu)
    eizo = None if args.skip_eizo else bench_eizo7(world, ck, cpu=(world_size == 1 and not args.skip_cpu),
                                                   fp64_peak=fp64_peak)
    config3 = None if args.skip_eizo else bench_config3(world, ck, comm, world_size, rank)
    config4_sharded = None
    if world_size > 1 and not args.skip_extra:
        config4_sharded = bench_config4_sharded(comm, world_size)

    if rank != 0:
        if world_size > 1:
            dist.destroy_process_group()
        return

    peak_tf = _peak("ez_fp32_peak", gpu)
    avg_launch_ms = float(np.mean(launch_ms))
    achieved_tf = FLOP_PER_CHECK * BATCH / (avg_launch_ms * 1e-3) / 1e12
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get("check_bytes_per_launch")
        except Exception:
            traffic = None
    cpu = None
    if world_size == 1 and not args.skip_cpu:
        cpu = cpu_oracle_rate(world, args.cpu_sample, 1)
    peaks = _measured_peaks()
    extra = {}
    if world_size == 1 and not args.skip_extra:
        extra["config1"] = bench_config1(cpu=not args.skip_cpu)
        extra["config4"] = bench_config4(cpu=not args.skip_cpu, fp64_peak=fp64_peak)
        extra["boxes"] = bench_boxes()
        extra["drm"] = bench_drm(cpu=not args.skip_cpu)
    if config4_sharded is not None:
        extra["config4_in_segment_sharded"] = config4_sharded
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world_size, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": dict(CONFIG2),
        "workload_detail": {"free_fraction": free_frac, "precision": "fp32 (flags exact outside a 1e-5 contact band)",
                            "parity": "batch 0 = tests/golden/config2_1m.npz rows (reference flags, "
                                      "tests/test_gpu_pinned.py::test_config2_full_size_through_the_bench_launch)"},
        "roofline": {"bound": "fp32", "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": achieved_tf / peak_tf, "traffic": traffic,
                     "kernel": ("ez_check_jit_f (k_check specialised for the model at run time, NVRTC sm_100a)"
                                if specialised else "k_check<float,float>"),
                     "jit_compile_ms": jit_ms, "cta": nat.info()["check_cta"], "flop_per_check": FLOP_PER_CHECK,
                     "avg_launch_ms": avg_launch_ms,
                     "frac_note": "of measured: the FP32 FMA peak of this GPU, measured in this run; FLOP are "
                                  "SURVEY 8(d)'s per-check model (every test), early exit skips part of them",
                     "peak_source": "ez_fp32_peak FMA microbenchmark measured in this run "
                                    "(MEASURED_PEAKS.json has HBM %.0f GB/s and bf16 only)" % peaks.get("hbm_gbs", 0),
                     # the same launch on the HBM roofline (28 B in + 1 B out per check)
                     "hbm": {"achieved": 29.0 * BATCH / (avg_launch_ms * 1e-3) / 1e9, "peak": peaks.get("hbm_gbs"),
                             "unit": "GB/s",
                             "frac": (29.0 * BATCH / (avg_launch_ms * 1e-3) / 1e9 / peaks["hbm_gbs"])
                             if peaks.get("hbm_gbs") else None,
                             "frac_note": "of measured (MEASURED_PEAKS.json hbm_gbs): not the bound"}},
        "e2e": {"value": e2e["pinned_fp32"], "unit": UNIT, "h2d_bytes_per_step": e2e["h2d_bytes_per_step"],
                "d2h_bytes_per_step": e2e["d2h_bytes_per_step"],
                "api": "CollisionChecker.check_batch(numpy fp32 rows in pinned host memory) -> ez_check_batch_host",
                "pageable_fp32": e2e["pageable_fp32"], "pinned_fp64": e2e["pinned_fp64"]},
        "fp64_arithmetic": {"checks_per_s": fp64_rate, "note": "precision='fp64' (the reference's arithmetic, "
                                                                 "flags bit-exact except |c| < 1e-12), same rows"},
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "eizo": eizo,
        "config3": config3,
        **extra,
    }
    print(json.dumps(line), flush=True)
    if world_size > 1:
        dist.destroy_process_group()


def bench_config4_sharded(comm, world_size: int) -> dict:
    """Config 4 region with each iteration's samples split over the ranks (2 collectives/iteration)."""
    import torch

    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.distributed import inflate_edge_sharded
    from paper_2504_10783_b200.eizo import InflationParams, Segment
    from paper_2504_10783_b200.polytope import HPolytope

    world = fx.bimanual14_world()
    ck = world.checker()
    v1, v2 = fx.random_free_segment(world, seed=3)
    dom = HPolytope.from_bounds(world.lower, world.upper)
    params = InflationParams(**fx.FRANKA_PARAMS)
    _barrier(world_size)
    t0 = time.perf_counter()
    rep = inflate_edge_sharded(Segment(v1, v2), dom, params, ck, seed=7, comm=comm)
    torch.cuda.synchronize()
    dt = _max_over_ranks(time.perf_counter() - t0, world_size)
    return {"ms_wall_max_over_ranks": dt * 1e3, "iterations": rep.iterations,
            "faces": rep.hyperplanes_added, "collision_checks": rep.collision_checks,
            "collectives": comm.collectives, "ranks": world_size}


def _relaunch_under_torchrun(args) -> None:
    """``--gpus N`` (N > 1) outside torchrun: re-exec under torch.distributed.run, one rank per GPU."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--skip-eizo", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-extra", action="store_true", help="skip the config-4 and config-5 (DRM) sections")
    ap.add_argument("--cpu-sample", type=int, default=30_000)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: host-staged collectives, ranks may share a GPU (tests of the multi-rank path)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _relaunch_under_torchrun(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
