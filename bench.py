#!/usr/bin/env python
"""Benchmark of the EI-ZO hot path (BASELINE.json): collision checks/s, 7-DOF vs 10k voxel spheres.

One step = one pass of the fused FK + collision kernel over a batch of 1M
7-DOF configurations (config 2 of BASELINE.json) per GPU.  Weak scaling:
under torchrun every rank checks its own 1M-config batches (no data-path
collective); the whole-job value is all configurations / max-over-ranks
device time.  Inputs are 8 resident batches (224 MB > the 126 MB L2) used in
rotation, so no step reads its configurations from L2.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Extra keys: ``roofline`` (FP32-FMA bound; measured FMA peak), ``cpu_baseline``
(the oracle port on this host, bounded sample), ``e2e`` (public numpy API
with pinned host buffers, copies inside the timed region), ``eizo`` (7-DOF
single-segment region latency), ``clocks``.
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


def bench_config4(checks_n: int = 1 << 20) -> dict:
    """Config 4: 14-DOF bimanual (66 spheres, 1,248 pairs): checks/s and one EI-ZO region."""
    import torch

    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge
    from paper_2504_10783_b200.polytope import HPolytope

    world = fx.bimanual14_world()
    ck = world.checker()
    lo = torch.as_tensor(world.lower, dtype=torch.float32, device="cuda")
    hi = torch.as_tensor(world.upper, dtype=torch.float32, device="cuda")
    Q = lo + (hi - lo) * torch.rand((checks_n, 14), device="cuda")
    nat = ck.native
    t_jit = time.perf_counter()
    specialised = nat.specialize(1)  # model-specialised kernel, also used by the EI-ZO loop below
    jit_ms = (time.perf_counter() - t_jit) * 1e3
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
    return {"checks_per_s": rate, "flop_per_check": 13104, "specialised_kernel": specialised, "jit_compile_ms": jit_ms,
            "cta": nat.info()["check_cta"],
            "eizo_ms_wall": wall, "eizo_device_ms": rep.device_ms, "iterations": rep.iterations,
            "faces": rep.hyperplanes_added, "collision_checks": rep.collision_checks,
            "terminated_by": rep.terminated_by,
            "workload": "14-DOF bimanual sphere model vs 10k voxels; EI-ZO single segment, Franka (eps, delta)"}


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
    return out


def run_reference(args):
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
            "config": {"workload": "config 2: Franka-like 7-DOF (33 spheres, 232 self pairs) vs 10k voxel spheres",
                       "sample_per_step": n},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{n} configs per step, oracle/ref.py with {cores} threads",
                             "cpu": cpu_model(), "host_cpus": os.cpu_count()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world_size, local_rank = _rank()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world_size > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_2504_10783_b200 import _native as N
    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge
    from paper_2504_10783_b200.polytope import HPolytope

    world = fx.franka7_world()
    ck = world.checker()
    nat = ck.native
    lo = torch.as_tensor(world.lower, dtype=torch.float32, device=dev)
    hi = torch.as_tensor(world.upper, dtype=torch.float32, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    batches = [lo + (hi - lo) * torch.rand((BATCH, 7), generator=gen, device=dev) for _ in range(N_BATCHES)]
    out = torch.empty(BATCH, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream

    def step(i):
        N.check(N.lib().ez_check_batch(nat.handle, batches[i % N_BATCHES].data_ptr(), 0, BATCH, 7, out.data_ptr(),
                                       0, sh))

    # model-specialised check kernel (NVRTC, ez_world_specialize); compiled
    # before the warm-up, outside every timed region
    t_jit = time.perf_counter()
    specialised = nat.specialize(1)
    jit_ms = (time.perf_counter() - t_jit) * 1e3

    gc.collect()
    for i in range(max(3, args.warmup)):
        step(i)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world_size > 1:
        dist.barrier()
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

    with ClockSampler(local_rank) as clk:
        clk.wait_first()
        busy(0.4)
        if world_size > 1:
            dist.barrier()
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
        if world_size > 1:
            dist.barrier()
        busy(0.4)
    if world_size > 1:
        dist.barrier()
    total_ms = t0.elapsed_time(t1)
    launch_ms = [a.elapsed_time(b) for a, b in ev]
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world_size > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    checks = BATCH * args.steps * world_size
    value = checks / (max_ms * 1e-3)
    free_frac = float(out.float().mean().item())

    # EI-ZO single-segment 7-DOF region (Franka parameters), latency per region
    eizo = None
    if not args.skip_eizo:
        v1, v2 = fx.random_free_segment(world, seed=3)
        dom = HPolytope.from_bounds(world.lower, world.upper)
        params = InflationParams(**fx.FRANKA_PARAMS)
        times, reps = [], []
        eck = ck  # the specialised checker: EI-ZO's checks run the per-model kernel
        inflate_edge(Segment(v1, v2), dom, params, eck, seed=6)  # warm-up (module load, workspace)
        for s in range(4):
            t_r = time.perf_counter()
            rep = inflate_edge(Segment(v1, v2), dom, params, eck, seed=7 + s)
            times.append((time.perf_counter() - t_r) * 1e3)
            reps.append(rep)
        eizo = {"ms_per_region_wall": float(np.median(times)),
                "device_ms": float(np.median([r.device_ms for r in reps])),
                "iterations": [r.iterations for r in reps], "faces": [r.hyperplanes_added for r in reps],
                "collision_checks": [r.collision_checks for r in reps],
                "segment": "7-DOF Franka-like + 10k voxels, length 0.6, free with margin 0.02 (default_rng(3))",
                "params": "delta=eps=0.005, N_p=1e4, N_f=10, N_ms=60, delta_max=0.01, N_b=11"}

    # config 3: a 10-segment 7-DOF path, segments sharded round-robin over the ranks
    config3 = None
    if not args.skip_eizo:
        from paper_2504_10783_b200.distributed import LocalComm, TorchComm, inflate_segments_sharded
        from paper_2504_10783_b200.roadmap import PwlPath

        knots = fx.random_free_path(world, 10, seed=3)
        path = PwlPath(knots)
        dom = HPolytope.from_bounds(world.lower, world.upper)
        params = InflationParams(**fx.FRANKA_PARAMS)
        comm = TorchComm() if world_size > 1 else LocalComm()
        eck = ck  # the specialised checker: EI-ZO's checks run the per-model kernel
        inflate_segments_sharded(path, dom, params, eck, seed=11, comm=comm)  # warm-up
        if world_size > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t_p = time.perf_counter()
        scs, mine = inflate_segments_sharded(path, dom, params, eck, seed=11, comm=comm)
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t_p], dtype=torch.float64, device=dev)
        if world_size > 1:
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        config3 = {"segments": 10, "path_ms_wall_max_over_ranks": float(dt.item()) * 1e3,
                   "segments_per_s": 10 / float(dt.item()), "sets_kept": len(scs.sets),
                   "segments_on_rank0": sorted(mine), "scaling": "strong (fixed 10-segment path)",
                   "note": "segment-keyed seeds child_seed(seed, 0x5E7, k); skip rule replayed on every rank"}

    # e2e through the public numpy API: pinned fp64 host buffers, H2D + D2H inside the timed region
    pin = torch.empty((BATCH, 7), dtype=torch.float64, pin_memory=True)
    pin.copy_(batches[0].double().cpu())
    Qh = pin.numpy()
    res_pin = torch.empty(BATCH, dtype=torch.uint8, pin_memory=True).numpy()
    # measured last, away from the nvidia-smi clock sampler and seconds after
    # the CUDA context came up (host-driven copies ran slower in the first
    # second of a process, tools/diag_e2e3.py); the median of three groups
    e2e_steps = max(3, min(args.steps, 10))
    # collect the garbage of the sections above first: a collection inside the
    # timed calls would run their checkers' destructors (cudaFree, unpinning)
    # there (measured: 1.2 -> 1.7 ms per call)
    gc.collect()
    # warm-up by time, not count: copies from a freshly pinned buffer ran ~25%
    # slower for about a second (tools/diag_e2e5.py)
    t_w, n_w = time.perf_counter(), 0
    while n_w < 3 or time.perf_counter() - t_w < 1.5:
        nat.check_host(Qh, out=res_pin)
        n_w += 1
    if world_size > 1:
        dist.barrier()
    groups = []
    for _ in range(3):
        t_e = time.perf_counter()
        for _ in range(e2e_steps):
            nat.check_host(Qh, out=res_pin)
        groups.append(time.perf_counter() - t_e)
    e2e_s = float(np.median(groups))
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world_size > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = BATCH * e2e_steps * world_size / float(te.item())

    if rank != 0:
        if world_size > 1:
            dist.destroy_process_group()
        return

    peak_tf = N.C.c_double(0.0)
    peak_ms = N.C.c_double(0.0)
    N.check(N.lib().ez_fp32_peak(local_rank, N.C.byref(peak_tf), N.C.byref(peak_ms)))
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
        extra["config4"] = bench_config4()
        extra["boxes"] = bench_boxes()
        extra["drm"] = bench_drm(cpu=not args.skip_cpu)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world_size, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "config 2: Franka-like 7-DOF (33 spheres r=0.055, 232 self pairs) vs 10k voxel "
                               "spheres (side 0.02), uniform configs in the joint limits",
                   "configs_per_step_per_gpu": BATCH, "l2": "8 rotating resident batches (224 MB > L2)",
                   "free_fraction": free_frac, "precision": "fp32 (flags exact outside a 1e-5 contact band)"},
        "roofline": {"bound": "fp32", "achieved": achieved_tf, "peak": peak_tf.value, "unit": "TFLOP/s",
                     "frac": achieved_tf / peak_tf.value, "traffic": traffic,
                     "kernel": ("ez_check_jit_f (k_check specialised for the model at run time, NVRTC sm_100a)"
                                if specialised else "k_check<float,float>"),
                     "jit_compile_ms": jit_ms, "cta": nat.info()["check_cta"], "flop_per_check": FLOP_PER_CHECK,
                     "avg_launch_ms": avg_launch_ms,
                     "frac_note": "of measured: the FP32 FMA peak of this GPU, measured in this run",
                     "peak_source": "ez_fp32_peak FMA microbenchmark measured in this run "
                                    "(MEASURED_PEAKS.json has HBM %.0f GB/s and bf16 only)" % peaks.get("hbm_gbs", 0),
                     # the same launch on the HBM roofline (28 B in + 1 B out per check)
                     "hbm": {"achieved": 29.0 * BATCH / (avg_launch_ms * 1e-3) / 1e9, "peak": peaks.get("hbm_gbs"),
                             "unit": "GB/s",
                             "frac": (29.0 * BATCH / (avg_launch_ms * 1e-3) / 1e9 / peaks["hbm_gbs"])
                             if peaks.get("hbm_gbs") else None,
                             "frac_note": "of measured (MEASURED_PEAKS.json hbm_gbs): not the bound"}},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": BATCH * 7 * 8, "d2h_bytes_per_step": BATCH,
                "api": "CollisionChecker.check_batch(numpy fp64, pinned) -> ez_check_batch_host"},
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
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
