"""Benchmark: radio-map SBR ray-bounces/s on the config-2 street canyon (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

Workload (BASELINE.json configs[1], the largest single-GPU radio-map config):
procedural street canyon (11,600 triangles), 1e7 Fibonacci rays per GPU,
{R, S} depth 5, concrete with S = 0.3, 200 x 200 cells of 1 m at z = 1.5,
Tx (0, 5, 20).  A step = one full map: the bounce megakernel over the rank's
shard of global sample ids, the direct term (rank 0), and (N > 1) an NCCL
all-reduce of the float64 grid + counters.  Weak scaling: each rank traces
its own 1e7 samples of an N*1e7-sample lattice.

value      : total ray-bounces of all ranks / max-over-ranks device time
e2e        : same metric through the public API compute_radio_map_sbr with
             host output (params H2D, grid + counters D2H every step)
roofline   : dominant kernel of the wavefront (k_map_trace / k_map_shade, timed
             with CUDA events inside libsbr on the launching stream), 176
             algorithmic bytes per ray-bounce / its summed
             launch time, vs measured HBM GB/s
cir        : config 3 (city, 1 Tx x 1024 Rx, N_S = 1e6, depth 5): ms per
             compute_paths solve (the CIR half of the BASELINE metric)
config4    : city radio map, 1e9 rays strong-scaled over the N GPUs (the
             multi-GPU radio-map config of BASELINE.json), rb/s
cpu_baseline: the CPU oracle port (oracle/, scalar C restatement of the
             reference loop) on this host's cores over a bounded subsample
--impl reference: that CPU port alone, on all host threads, same metric.
"""

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "radio-map SBR ray-bounces/sec"
UNIT = "ray-bounces/s"
SAMPLES_PER_GPU = 10_000_000
CIR_SAMPLES = 1_000_000
CIR_CPU_SAMPLES = 2_000
C4_SAMPLES = 1_000_000_000
BYTES_PER_RB = 176  # 64 B ray state in + 64 B out + 48 B hit triangle
TX = (0.0, 5.0, 20.0)


def workload(n_total):
    from paper_2504_21719_b200 import scenes
    from paper_2504_21719_b200.radiomap import MeasurementGrid, RadioMapConfig
    from paper_2504_21719_b200.sampling import Interaction
    meshes = scenes.street_canyon()
    mats = scenes.uniform_materials(meshes, scenes.concrete(scattering=0.3))
    grid = MeasurementGrid((0.0, 0.0, 1.5), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (200, 200))
    cfg = RadioMapConfig(num_samples=n_total, max_depth=5, seed=0,
                         enabled=frozenset({Interaction.REFLECTION, Interaction.SCATTERING}))
    return meshes, mats, grid, cfg


def config_dict(n_gpus, ntri):
    return {
        "workload": "config2: procedural street canyon radio map, 1e7 rays per GPU, "
                    "{R,S} depth 5, 200x200 cells of 1 m, Tx (0,5,20)",
        "scene_triangles": ntri,
        "samples_per_gpu": SAMPLES_PER_GPU,
        "max_depth": 5,
        "grid_cells": 40000,
        "l2": "flushed between timed steps (256 MiB write, outside the per-step events)",
        "parallelism": f"dp{n_gpus}: chunk-cyclic global sample-id shards (2^19-id RNG chunks "
                       "dealt round-robin), NCCL all-reduce of the grid",
    }


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[3:7]):
                if flag.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def profiled_traffic(kernel):
    """Mean dram bytes per launch of `kernel` from the committed ncu capture
    (profiles/traffic_<kernel>.json, tools/ncu_summary.py traffic), if any."""
    path = os.path.join(ROOT, "profiles", f"traffic_{kernel}.json")
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------
# CPU: the oracle port (bench cpu_baseline leg and --impl reference)

def cpu_port_rate(threads, target_samples):
    """Run the oracle over `target_samples` rays spread across the 1e7 lattice."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    meshes, mats, grid, cfg = workload(SAMPLES_PER_GPU)
    sc = oracle.OracleScene(meshes, mats)
    sc.bind_frequency(cfg.frequency)
    pieces = 400
    per = max(1, target_samples // pieces)
    stride = SAMPLES_PER_GPU // pieces
    ranges = [(i * stride, i * stride + per) for i in range(pieces)]

    def run(rg):
        _, d = sc.radiomap(np.array(TX), grid, cfg, sample_range=rg, include_direct=False)
        return d["ray_bounces"]

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as pool:
        rb = sum(pool.map(run, ranges))
    dt = time.perf_counter() - t0
    return rb / dt, rb, per * pieces, dt


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, rank, world):
    if rank != 0:
        return
    threads = cpu_threads()
    target = 400_000 * threads  # ~15 s of CPU work per step on this port
    target = min(target, SAMPLES_PER_GPU)
    for _ in range(args.warmup):
        cpu_port_rate(threads, max(target // 10, 4000))
    rates, rbs, dts = [], [], []
    for _ in range(args.steps):
        r, rb, ns, dt = cpu_port_rate(threads, target)
        rates.append(r)
        rbs.append(rb)
        dts.append(dt)
    rate = float(np.sum(rbs) / np.sum(dts))
    meshes, _, _, _ = workload(SAMPLES_PER_GPU)
    ntri = sum(len(m.triangles) for m in meshes)
    sample = (f"{ns} of the 1e7 rays (400 evenly spaced slices), "
              f"{int(np.mean(rbs))} ray-bounces per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.mean(dts) * 1e3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args.gpus, ntri),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference is Python/Cython (no compiled C path to build); timed port = "
                "oracle/sbr_oracle.c, a scalar C restatement pinned bit-exact to the "
                "reference's golden maps, threaded over sample slices",
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU: our implementation

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2504_21719_b200 import SceneModel, _abi, _native
    from paper_2504_21719_b200.radiomap import compute_radio_map_sbr, pack_map_params

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n_total = SAMPLES_PER_GPU * world
    meshes, mats, grid, cfg = workload(n_total)
    ntri = sum(len(m.triangles) for m in meshes)
    scene = SceneModel(meshes, mats, device=dev)
    scene.bind_frequency(cfg.frequency)
    L = _native.lib()
    lo, hi = rank * SAMPLES_PER_GPU, (rank + 1) * SAMPLES_PER_GPU
    params, _, _ = pack_map_params(scene, np.array(TX), grid, cfg)
    nx, ny = grid.shape
    values = torch.zeros((ny, nx), dtype=torch.float64, device=dev)
    direct = torch.zeros((ny, nx), dtype=torch.float64, device=dev)
    counters = torch.zeros(_abi.SBR_MC_COUNT, dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = ctypes.c_void_p(stream.cuda_stream)

    def step(kernel_events=None):
        values.zero_()
        counters.zero_()
        if kernel_events is not None:
            kernel_events[0].record(stream)
        if world > 1:   # chunk-cyclic shard of the N x 1e7 lattice (balanced over the sphere)
            _native.check(L.sbr_radiomap_bounce_sharded(
                scene.accel.handle, ctypes.byref(params), rank, world, _native.ptr(values),
                _native.ptr(counters), sptr))
        else:
            _native.check(L.sbr_radiomap_bounce(scene.accel.handle, ctypes.byref(params), lo,
                                                hi, _native.ptr(values), _native.ptr(counters),
                                                sptr))
        if kernel_events is not None:
            kernel_events[1].record(stream)
        if rank == 0:
            _native.check(L.sbr_radiomap_direct(scene.accel.handle, ctypes.byref(params),
                                                _native.ptr(direct), _native.ptr(counters),
                                                sptr))
            values.add_(direct)
        if world > 1:
            dist.all_reduce(values)
            dist.all_reduce(counters)

    for _ in range(max(args.warmup, 3) if args.warmup >= 3 else args.warmup):
        step()
    torch.cuda.synchronize()
    scene.accel.check()

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _native.kernel_launches()
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
    kern_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
    rb_counts = []
    with ClockSampler(local_rank) as clocks:
        for k in range(args.steps):
            flush.fill_(float(k))            # evict the scene / grid from L2 (untimed)
            step_ev[k][0].record(stream)
            step(kern_ev[k])
            step_ev[k][1].record(stream)
            rb_counts.append(counters[_abi.MAP_COUNTERS.index("ray_bounces")].clone())
        torch.cuda.synchronize()
    launches = _native.kernel_launches() - launches0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = np.array([a.elapsed_time(b) for a, b in step_ev])
    kern_ms = np.array([a.elapsed_time(b) for a, b in kern_ev])
    rb_total = int(sum(int(c.item()) for c in rb_counts))  # all ranks (all-reduced)
    t_local = float(step_ms.sum())
    if world > 1:
        tt = torch.tensor([t_local], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    else:
        t_max = t_local
    value = rb_total / (t_max / 1e3)
    rb_per_step_local = rb_total / args.steps / world

    # ---- per-kernel split (CUDA events around each library launch, on the
    # ---- launching stream), measured on extra untimed steps
    prof_steps = max(1, min(args.steps, 3))
    _native.profile_enable(True)
    for k in range(prof_steps):
        flush.fill_(float(k))
        step()
    torch.cuda.synchronize()
    kernels = {}
    for name in ("k_map_trace", "k_map_shade", "k_map_scatter"):
        ms, nl = _native.profile_kernel_ms(name)
        kernels[name] = {"ms_per_step": ms / prof_steps, "launches_per_step": nl / prof_steps}
    _native.profile_enable(False)
    dom = max(kernels, key=lambda k: kernels[k]["ms_per_step"])
    dom_ms_step = kernels[dom]["ms_per_step"]
    dom_launches = kernels[dom]["launches_per_step"]
    # algorithmic bytes: 176 B per ray-bounce x the rays the kernel
    # processed, over the kernel's own summed launch time
    achieved = rb_per_step_local * BYTES_PER_RB / (dom_ms_step / 1e3) / 1e9
    peak, peak_kind = peaks()
    traffic = profiled_traffic(dom)

    # ---- end to end through the public API (host buffers) ----
    e2e_ms = []
    h2d = ctypes.sizeof(_abi.SbrMapParams)
    d2h = nx * ny * 8 + _abi.SBR_MC_COUNT * 8
    for k in range(max(1, args.steps)):
        flush.fill_(float(k))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        if world == 1:
            host_vals, diag = compute_radio_map_sbr(scene, np.array(TX), grid, cfg,
                                                    sample_range=(lo, hi))
            rb_e2e = diag["ray_bounces"]
        else:
            v, c = compute_radio_map_sbr(scene, np.array(TX), grid, cfg, shard=(rank, world),
                                         include_direct=(rank == 0), return_tensors=True)
            dist.all_reduce(v)
            dist.all_reduce(c)
            host_vals = v.cpu().numpy()
            rb_e2e = int(c[_abi.MAP_COUNTERS.index("ray_bounces")].item())
        t1.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(t0.elapsed_time(t1))
    e_local = float(np.sum(e2e_ms))
    if world > 1:
        tt = torch.tensor([e_local], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e_local = float(tt.item())
    e2e_value = rb_e2e * len(e2e_ms) / (e_local / 1e3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = cpu_threads()
        rate, rb_cpu, ns, dt = cpu_port_rate(threads, min(400_000 * threads, SAMPLES_PER_GPU))
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{ns} of the 1e7 rays (400 evenly spaced slices), {rb_cpu} "
                         f"ray-bounces in {dt:.2f} s on {threads} threads"}

    cir = None
    if not args.no_cir:
        cir = bench_cir(args, dev, rank, world)
    c4 = None
    if not args.no_config4:
        c4 = bench_config4(args, dev, rank, world)
    c5 = None
    if not args.no_config5:
        c5 = bench_config5(args, dev, rank, world)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(t_max / args.steps), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(world, ntri),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
                         "traffic_kernel": traffic.get("kernel") if traffic else None,
                         "kernel": dom, "bytes_per_unit": BYTES_PER_RB,
                         "units_per_launch": rb_per_step_local / max(dom_launches, 1),
                         "kernel_ms": dom_ms_step / max(dom_launches, 1),
                         "kernel_ms_per_step": dom_ms_step,
                         "bounce_call_ms_per_step": float(kern_ms.mean()),
                         "kernels": kernels, "peak_source": peak_kind},
            "cir": cir,
            "config4": c4,
            "config5": c5,
            "cpu_baseline": cpu,
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
            "ray_bounces_per_step": rb_total // args.steps,
        }
        print(json.dumps(line), flush=True)


def bench_config4(args, dev, rank=0, world=1):
    """Config 4: city radio map, 1e9 rays over all N GPUs (strong scaling), 1 m cells.

    1000 x 1000 cells at z = 1.5, Tx (0, 0, 30), {R, S} depth 5.  Each rank
    traces its contiguous shard of the 1e9 global sample ids; one NCCL
    all-reduce of the float64 grid (8 MB) and the counters; rank 0 adds the
    direct term.  Device time per map (max over ranks), CUDA events.
    """
    import torch
    import torch.distributed as dist
    from paper_2504_21719_b200 import SceneModel, _abi, scenes
    from paper_2504_21719_b200.radiomap import (MeasurementGrid, RadioMapConfig,
                                                compute_radio_map_sbr)
    from paper_2504_21719_b200.sampling import Interaction
    from paper_2504_21719_b200.sharding import allreduce_map
    meshes = scenes.city()
    scene = SceneModel(meshes, scenes.uniform_materials(meshes, scenes.concrete(scattering=0.3)),
                       device=dev)
    grid = MeasurementGrid((0.0, 0.0, 1.5), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (1000, 1000))
    cfg = RadioMapConfig(num_samples=C4_SAMPLES, max_depth=5, seed=0,
                         enabled=frozenset({Interaction.REFLECTION, Interaction.SCATTERING}))
    stream = torch.cuda.current_stream(dev)

    def one():   # chunk-cyclic shards of the 1e9 ids: every GPU sees the whole sphere
        v, c = compute_radio_map_sbr(scene, (0.0, 0.0, 30.0), grid, cfg, shard=(rank, world),
                                     include_direct=(rank == 0), return_tensors=True)
        allreduce_map(v, c)
        return v, c

    one()
    torch.cuda.synchronize()
    times, rbs = [], []
    for _ in range(max(1, min(args.steps, 2))):
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        v, c = one()
        b.record(stream)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
        rbs.append(int(c[_abi.MAP_COUNTERS.index("ray_bounces")].item()))
    ms = float(np.mean(times))
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    return {"workload": "config4: procedural city (483,200 tris) radio map, 1e9 rays sharded "
                        "over the N GPUs, 1000x1000 cells of 1 m, {R,S} depth 5, Tx (0,0,30)",
            "value": rbs[-1] / (ms / 1e3), "unit": "ray-bounces/s", "ms_per_map": ms,
            "ray_bounces_per_map": rbs[-1], "n_gpus": world, "scaling": "strong",
            "maps": len(times)}


def bench_cir(args, dev, rank=0, world=1):
    """Config 3: city CIR, 1 Tx x 1024 Rx, N_S = 1e6, depth 5, {R} (BASELINE configs[2]).

    ms per solve (generation + dedup + refinement + fields, host PathTensors
    out) timed with CUDA events on the current stream, max over ranks.  With
    N > 1 GPUs the solve is compute_paths_sharded: sample shards per rank,
    all-gathered candidate rows, replicated global selection (strong scaling:
    the same 1e6-sample solve split over the ranks).
    """
    import torch
    import torch.distributed as dist
    from paper_2504_21719_b200 import (PathConfig, RadioDevice, SceneModel, _native, scenes)
    from paper_2504_21719_b200.cir import compute_paths_sharded as compute_paths
    from paper_2504_21719_b200.sampling import Interaction
    t0 = time.perf_counter()
    meshes = scenes.city()
    scene = SceneModel(meshes, scenes.uniform_materials(meshes, scenes.concrete()), device=dev)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    rxs = [RadioDevice(position=p) for p in scenes.city_receivers(1024)]
    tx = RadioDevice(position=np.array([0.0, 0.0, 30.0]))
    cfg = PathConfig(num_samples=CIR_SAMPLES, max_depth=5, q_diffraction=0.0,
                     enabled=frozenset({Interaction.REFLECTION}), buffer_capacity=2 ** 24)
    compute_paths(scene, [tx], rxs, cfg)  # warm-up
    stream = torch.cuda.current_stream(dev)
    _native.profile_enable(True)
    times, ps = [], None
    for _ in range(max(1, min(args.steps, 3))):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ps = compute_paths(scene, [tx], rxs, cfg)
        b.record(stream)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    n = len(times)
    split = {k: _native.profile_kernel_ms(k)[0] / n for k in ("k_cir_sweep", "k_cir_visibility")}
    _native.profile_enable(False)
    ms = float(np.mean(times))
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    d = ps.diagnostics
    cpu = None
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        # oracle port (oracle/sbr_oracle.c, single thread like the reference's
        # default workers=1) on a bounded sample, extrapolated linearly in N_S
        import oracle
        osc = oracle.OracleScene(meshes, scenes.uniform_materials(meshes, scenes.concrete()))
        small = PathConfig(num_samples=CIR_CPU_SAMPLES, max_depth=5, q_diffraction=0.0,
                           enabled=frozenset({Interaction.REFLECTION}), buffer_capacity=2 ** 24)
        t0 = time.perf_counter()
        osc.compute_paths([tx], rxs, small)
        dt = time.perf_counter() - t0
        cpu = {"value": dt * 1e3 * (CIR_SAMPLES / CIR_CPU_SAMPLES), "unit": "ms per Tx-Rx set",
               "cores": 1, "kind": "port",
               "sample": f"N_S={CIR_CPU_SAMPLES} of {CIR_SAMPLES} in {dt:.2f} s, "
                         f"extrapolated linearly in N_S"}
    return {"workload": "config3: procedural city (483,200 tris) CIR, 1 Tx x 1024 Rx, "
                        "N_S=1e6, depth 5, {R}, hash dedup + image-method refine",
            "ms_per_solve": ms, "solves": n, "paths": d["paths"], "n_gpus": world,
            "scaling": "strong",
            "candidates": d["candidates"], "duplicates": d["duplicates"],
            "refinement_rejections": d["refinement_rejections"],
            "kernel_ms_per_solve": split, "scene_build_s": build_s, "cpu_baseline": cpu,
            "unit": "ms per Tx-Rx set (1 Tx x 1024 Rx)", "higher_is_better": False}


def bench_config5(args, dev, rank=0, world=1):
    """Config 5: city, 8x8 TR 38.901 Tx panel (lambda/2), 4x4 Rx panel, depth 6, N_S = 1e6,
    CIR + CFR over 1024 subcarriers (BASELINE configs[4]); synthetic arrays.

    ms per solve = compute_paths (sharded over the ranks like config 3) +
    frequency_response to a host (16, 64, 1024) complex128 array, CUDA events,
    max over ranks; k_cfr_contract timed separately with its output-write
    roofline (16 B per H entry).
    """
    import torch
    import torch.distributed as dist
    from paper_2504_21719_b200 import (PathConfig, RadioDevice, SceneModel, _native, make_pattern,
                                       scenes)
    from paper_2504_21719_b200.cir import compute_paths_sharded as compute_paths
    from paper_2504_21719_b200.cir import frequency_response
    from paper_2504_21719_b200.em import planar_array
    from paper_2504_21719_b200.sampling import Interaction
    meshes = scenes.city()
    scene = SceneModel(meshes, scenes.uniform_materials(meshes, scenes.concrete()), device=dev)
    lam = 299792458.0 / 3.5e9
    tx = RadioDevice(position=np.array([0.0, 0.0, 30.0]), pattern=make_pattern("tr38901"),
                     array=planar_array(8, 8, lam / 2, lam / 2))
    rx = RadioDevice(position=np.array([2.0, 60.0, 1.5]),
                     array=planar_array(4, 4, lam / 2, lam / 2))
    cfg = PathConfig(num_samples=1_000_000, max_depth=6, q_diffraction=0.0,
                     enabled=frozenset({Interaction.REFLECTION}))
    freqs = 3.5e9 + (np.arange(1024) - 512) * 30e3

    def solve():
        ps = compute_paths(scene, [tx], [rx], cfg)
        return ps, frequency_response(ps, freqs)

    held = [solve() for _ in range(max(args.warmup, 2))]  # warm-up; the held results keep
    del held                                              # two pinned H buffers cached
    stream = torch.cuda.current_stream(dev)
    _native.profile_enable(True)
    times, ps, H = [], None, None
    for _ in range(max(1, min(args.steps, 3))):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ps, H = solve()
        b.record(stream)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    n = len(times)
    cfr_ms = _native.profile_kernel_ms("k_cfr_contract")[0] / n
    _native.profile_enable(False)
    ms = float(np.mean(times))
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    out_bytes = H.size * 16
    return {"workload": "config5: procedural city CIR + CFR, 8x8 TR 38.901 Tx x 4x4 Rx "
                        "(synthetic arrays), depth 6, N_S=1e6, 1024 subcarriers",
            "ms_per_solve": ms, "solves": n, "paths": len(ps.tensors), "H_shape": list(H.shape),
            "n_gpus": world, "scaling": "strong",
            "k_cfr_contract_ms": cfr_ms,
            "k_cfr_contract_write_gbs": out_bytes / (cfr_ms / 1e3) / 1e9 if cfr_ms > 0 else None,
            "unit": "ms per Tx-Rx set", "higher_is_better": False}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cir", action="store_true")
    ap.add_argument("--no-config4", action="store_true")
    ap.add_argument("--no-config5", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if os.environ.get("SBR_BENCH_GLOO") == "1":
            # functional check of the N > 1 code paths on a one-GPU box (gloo,
            # ranks share the device): the numbers are meaningless
            local_rank = local_rank % torch.cuda.device_count()
            torch.cuda.set_device(local_rank)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
