"""Benchmark: radio-map SBR ray-bounces/s on the config-4 city map (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

Headline workload (BASELINE.json configs[3], the radio-map config the metric's
"at 1/2/4/8 B200" is quoted on; it fits one GPU): procedural city (483,200
triangles, SURVEY §8d config 3/4 recipe), 1e9 Fibonacci rays, {R, S} depth 5,
concrete with S = 0.3, 1000 x 1000 cells of 1 m at z = 1.5 centred on the
scene, Tx (0, 0, 30).  A step = one full 1e9-ray map: the wavefront SBR
kernels over the rank's chunk-cyclic shard of the global sample ids, the
direct term (rank 0) and (N > 1) one NCCL all-reduce of the float64 grid +
counters.  Strong scaling: the 1e9 rays are split over the N GPUs.

value       : total ray-bounces of the map / max-over-ranks device time
e2e         : same metric through the public API compute_radio_map_sbr with
              host output (params H2D, 8 MB grid + counters D2H every step)
roofline    : dominant kernel of the map (k_map_trace / k_map_shade, timed with
              CUDA events inside libsbr on the launching stream), 176
              algorithmic bytes per ray-bounce x the
              ray-bounces it processed / its summed launch time, vs the
              measured HBM GB/s
cpu_baseline: the CPU oracle port (oracle/, scalar C restatement of the
              reference loop, pinned to the reference's golden maps) on this
              host's cores over evenly spaced slices of the same 1e9 lattice
config2     : config 2 (street canyon, 1e7 rays per GPU, weak scaling)
cir         : config 3 (city, 1 Tx x 1024 Rx, N_S = 1e6, depth 5): ms per
              compute_paths solve (the CIR half of the BASELINE metric)
config5     : config 5 (8x8 / 4x4 arrays, depth 6, CIR + CFR over 1024 subcarriers)
--impl reference: the CPU port alone on all host threads, same metric and
              config (bounded slices per step), plus one timed map of the
              real reference package (emtrace + its Cython kernel, installed
              in baseline/_ref) on the same scene when it is importable.
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
C4_SAMPLES = 1_000_000_000
C4_TX = (0.0, 0.0, 30.0)
C2_SAMPLES_PER_GPU = 10_000_000
C2_TX = (0.0, 5.0, 20.0)
CIR_SAMPLES = 1_000_000
CIR_CPU_SAMPLES = 2_000
BYTES_PER_RB = 176      # 64 B ray state in + 64 B out + 48 B hit triangle
BYTES_PER_VIS = 32      # 24 B segment in + result, per visibility ray
CPU_SAMPLES_PER_THREAD = 1_500_000   # cpu_baseline leg: ~6 s of port work per thread
REF_SAMPLES_PER_THREAD = 1_000_000   # --impl reference: ~4 s per step
EMTRACE_SAMPLES = 1 << 20            # real-reference map (2 RNG chunks)


def _rs():
    from paper_2504_21719_b200.radiomap import MeasurementGrid, RadioMapConfig
    from paper_2504_21719_b200.sampling import Interaction
    return MeasurementGrid, RadioMapConfig, Interaction


def c4_workload(n_samples=C4_SAMPLES):
    from paper_2504_21719_b200 import scenes
    MeasurementGrid, RadioMapConfig, Interaction = _rs()
    meshes = scenes.city()
    mats = scenes.uniform_materials(meshes, scenes.concrete(scattering=0.3))
    grid = MeasurementGrid((0.0, 0.0, 1.5), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (1000, 1000))
    cfg = RadioMapConfig(num_samples=n_samples, max_depth=5, seed=0,
                         enabled=frozenset({Interaction.REFLECTION, Interaction.SCATTERING}))
    return meshes, mats, grid, cfg


def c2_workload(n_total):
    from paper_2504_21719_b200 import scenes
    MeasurementGrid, RadioMapConfig, Interaction = _rs()
    meshes = scenes.street_canyon()
    mats = scenes.uniform_materials(meshes, scenes.concrete(scattering=0.3))
    grid = MeasurementGrid((0.0, 0.0, 1.5), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (200, 200))
    cfg = RadioMapConfig(num_samples=n_total, max_depth=5, seed=0,
                         enabled=frozenset({Interaction.REFLECTION, Interaction.SCATTERING}))
    return meshes, mats, grid, cfg


def config_dict(n_gpus, ntri):
    return {
        "workload": "config4: procedural city radio map, 1e9 rays sharded over the N GPUs, "
                    "1000x1000 cells of 1 m at z=1.5, {R,S} depth 5, concrete S=0.3, "
                    "Tx (0,0,30)",
        "scene_triangles": ntri,
        "samples": C4_SAMPLES,
        "max_depth": 5,
        "grid_cells": 1_000_000,
        "l2": "inputs larger than L2 (ray queues of ~7 GB per pass) and L2 flushed between "
              "timed steps (256 MiB write, outside the per-step events)",
        "parallelism": f"dp{n_gpus}: chunk-cyclic global sample-id shards (2^19-id RNG chunks "
                       "dealt round-robin), scene replicated, NCCL all-reduce of the grid",
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
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def profiled_traffic(kernel, tag):
    """Mean dram bytes per launch of `kernel` from the committed ncu capture of
    workload `tag` (profiles/traffic_<tag>_<kernel>.json, tools/ncu_summary.py traffic)."""
    for name in (f"traffic_{tag}_{kernel}.json", f"traffic_{kernel}.json" if tag == "c2" else ""):
        if not name:
            continue
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                return json.load(f)
        except (OSError, ValueError):
            continue
    return None


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def max_over_ranks(x, dev, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_floats(vals, dev, world):
    """All ranks' copies of a small float vector (rank order)."""
    if world == 1:
        return [list(vals)]
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [o.cpu().tolist() for o in out]


# ---------------------------------------------------------------------------
# CPU: the oracle port (cpu_baseline legs and --impl reference)

def port_map_rate(scene, grid, cfg, tx, threads, target_samples, pieces=1000):
    """Oracle map over `target_samples` rays in `pieces` evenly spaced slices of
    cfg's lattice, on `threads` host threads (the C code releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    pieces = max(1, min(pieces, target_samples))
    per = max(1, target_samples // pieces)
    stride = cfg.num_samples // pieces
    ranges = [(i * stride, i * stride + per) for i in range(pieces)]

    def run(rg):
        _, d = scene.radiomap(np.array(tx), grid, cfg, sample_range=rg, include_direct=False)
        return d["ray_bounces"]

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as pool:
        rb = sum(pool.map(run, ranges))
    dt = time.perf_counter() - t0
    return rb / dt, rb, per * pieces, dt


def emtrace_map(threads):
    """One timed map of the REAL reference (emtrace from baseline/_ref, Cython
    _core kernel) on the config-4 scene / grid / config at EMTRACE_SAMPLES rays
    through its public API compute_radio_map_sbr.  None when not installed."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "emtrace")):
        return None
    sys.path.insert(0, ref)
    try:
        import emtrace._kernels as ek
        from emtrace.geometry import Mesh
        from emtrace.materials import RadioMaterial
        from emtrace.paths import SceneModel
        from emtrace.radiomap import MeasurementGrid, RadioMapConfig, compute_radio_map_sbr
        from emtrace.sampling import Interaction
    except Exception as exc:  # noqa: BLE001
        return {"unavailable": f"emtrace import failed: {exc!r}"}
    finally:
        sys.path.remove(ref)
    meshes, _, _, _ = c4_workload()
    em = [Mesh(np.asarray(m.vertices), np.asarray(m.triangles), object_id=m.object_id)
          for m in meshes]
    mat = RadioMaterial(eps_r=5.24, sigma=0.0462, thickness=0.1, scattering=0.3)
    t0 = time.perf_counter()
    scene = SceneModel(em, {m.object_id: mat for m in em})
    build_s = time.perf_counter() - t0
    grid = MeasurementGrid((0.0, 0.0, 1.5), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (1000, 1000))
    cfg = RadioMapConfig(num_samples=EMTRACE_SAMPLES, max_depth=5, seed=0, workers=threads,
                         enabled=frozenset({Interaction.REFLECTION, Interaction.SCATTERING}))
    # ray-bounces = rows passed to Accel.trace_batch inside _map_chunk (SURVEY
    # §8d); the reference does not count them, so the instance's bound method
    # is wrapped with a row counter (its arithmetic is untouched)
    rows = [0]
    lock = threading.Lock()
    inner = scene.accel.trace_batch

    def counting_trace_batch(origins, directions, *a, **kw):
        with lock:
            rows[0] += len(origins)
        return inner(origins, directions, *a, **kw)

    scene.accel.trace_batch = counting_trace_batch
    t0 = time.perf_counter()
    _, diag = compute_radio_map_sbr(scene, np.array(C4_TX), grid, cfg)
    dt = time.perf_counter() - t0
    diag["ray_bounces"] = rows[0]
    chunks = -(-EMTRACE_SAMPLES // (1 << 19))
    return {"value": diag["ray_bounces"] / dt, "unit": UNIT, "kind": "reference",
            "cores": min(threads, chunks), "kernel": getattr(ek.active(), "__name__", "?"),
            "sample": f"compute_radio_map_sbr of emtrace on the config-4 scene, grid and "
                      f"config at num_samples={EMTRACE_SAMPLES} (its own Fibonacci lattice), "
                      f"workers={threads}; {diag['ray_bounces']} ray-bounces + 1e6-cell "
                      f"direct term in {dt:.1f} s; the reference parallelises over 2^19-ray "
                      f"chunks, so {chunks} chunks use at most {chunks} threads",
            "scene_build_s": build_s, "ray_bounces": int(diag["ray_bounces"]), "seconds": dt}


def run_reference(args, rank, world):
    if rank != 0:
        return
    import oracle
    threads = cpu_threads()
    meshes, mats, grid, cfg = c4_workload()
    ntri = sum(len(m.triangles) for m in meshes)
    t0 = time.perf_counter()
    sc = oracle.OracleScene(meshes, mats)
    sc.bind_frequency(cfg.frequency)
    build_s = time.perf_counter() - t0
    target = REF_SAMPLES_PER_THREAD * threads
    for _ in range(args.warmup):
        port_map_rate(sc, grid, cfg, C4_TX, threads, max(target // 20, 4000), pieces=200)
    rbs, dts, ns = [], [], 0
    for _ in range(args.steps):
        _, rb, ns, dt = port_map_rate(sc, grid, cfg, C4_TX, threads, target)
        rbs.append(rb)
        dts.append(dt)
    rate = float(np.sum(rbs) / np.sum(dts))
    sample = (f"{ns} of the 1e9 rays per step (1000 evenly spaced slices of the lattice), "
              f"{int(np.mean(rbs))} ray-bounces per step on {threads} threads; "
              f"scene (SAH BVH) build {build_s:.1f} s outside the timing")
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.mean(dts) * 1e3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args.gpus, ntri),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "timed arm = oracle/sbr_oracle.c, the scalar C restatement of the reference's "
                "_map_chunk loop pinned bit-exact to the real reference's golden maps "
                "(tests/golden), threaded over lattice slices; the reference package itself "
                "(Python + Cython) is timed once below under 'emtrace'",
    }
    if not args.no_emtrace:
        line["emtrace"] = emtrace_map(threads)
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU: our implementation

class MapRunner:
    """One radio map per call over this rank's chunk-cyclic shard (device only)."""

    def __init__(self, scene, grid, cfg, tx, dev, rank, world):
        import torch
        from paper_2504_21719_b200 import _abi, _native
        from paper_2504_21719_b200.radiomap import pack_map_params
        self.torch, self._abi, self._native = torch, _abi, _native
        self.scene, self.rank, self.world = scene, rank, world
        scene.bind_frequency(cfg.frequency)
        self.L = _native.lib()
        self.params, _, _ = pack_map_params(scene, np.array(tx), grid, cfg)
        nx, ny = grid.shape
        self.values = torch.zeros((ny, nx), dtype=torch.float64, device=dev)
        self.direct = torch.zeros((ny, nx), dtype=torch.float64, device=dev)
        self.counters = torch.zeros(_abi.SBR_MC_COUNT, dtype=torch.int64, device=dev)
        self.stream = torch.cuda.current_stream(dev)
        self.sptr = ctypes.c_void_p(self.stream.cuda_stream)
        self.rb_idx = _abi.MAP_COUNTERS.index("ray_bounces")

    def step(self, kernel_events=None, local_rb=None):
        import torch.distributed as dist
        N, L = self._native, self.L
        self.values.zero_()
        self.counters.zero_()
        if kernel_events is not None:
            kernel_events[0].record(self.stream)
        N.check(L.sbr_radiomap_bounce_sharded(
            self.scene.accel.handle, ctypes.byref(self.params), self.rank, self.world,
            N.ptr(self.values), N.ptr(self.counters), self.sptr))
        if kernel_events is not None:
            kernel_events[1].record(self.stream)
        if local_rb is not None:
            local_rb.append(self.counters[self.rb_idx].clone())
        if self.rank == 0:
            N.check(L.sbr_radiomap_direct(self.scene.accel.handle, ctypes.byref(self.params),
                                          N.ptr(self.direct), N.ptr(self.counters), self.sptr))
            self.values.add_(self.direct)
        if self.world > 1:
            dist.all_reduce(self.values)
            dist.all_reduce(self.counters)


def kernel_split(runner, flush, steps, names=("k_map_trace", "k_map_shade", "k_map_scatter")):
    """Per-kernel ms per map from libsbr's CUDA events on the launching stream,
    measured on extra untimed steps with the wavefront passes serialised (one
    stream: the timed steps overlap consecutive passes on two streams, which
    would make summed launch times exceed the wall time); also the local
    ray-bounces of one step."""
    import torch
    N = runner._native
    N.check(N.lib().sbr_set_wave_streams(1))
    N.profile_enable(True)
    local = []
    for k in range(steps):
        flush.fill_(float(k))
        runner.step(local_rb=local)
    torch.cuda.synchronize()
    kernels = {}
    for name in names:
        ms, nl = N.profile_kernel_ms(name)
        kernels[name] = {"ms_per_step": ms / steps, "launches_per_step": nl / steps}
    N.profile_enable(False)
    N.check(N.lib().sbr_set_wave_streams(2))
    return kernels, int(local[-1].item())


def roofline(kernels, rb_local, tag):
    dom = max(kernels, key=lambda k: kernels[k]["ms_per_step"])
    ms = kernels[dom]["ms_per_step"]
    nl = max(kernels[dom]["launches_per_step"], 1)
    achieved = rb_local * BYTES_PER_RB / (ms / 1e3) / 1e9
    peak, src = peaks()
    tr = profiled_traffic(dom, tag)
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": tr.get("dram_bytes_per_launch") if tr else None,
            "traffic_source": tr.get("source") if tr else None,
            "kernel": dom, "bytes_per_unit": BYTES_PER_RB, "unit_name": "ray-bounce",
            "units_per_launch": rb_local / nl, "kernel_ms": ms / nl,
            "kernel_ms_per_step": ms, "launches_per_step": nl,
            "kernels": kernels, "peak_source": src}


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2504_21719_b200 import SceneModel, _native
    from paper_2504_21719_b200.radiomap import compute_radio_map_sbr

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    meshes, mats, grid, cfg = c4_workload()
    ntri = sum(len(m.triangles) for m in meshes)
    t0 = time.perf_counter()
    scene = SceneModel(meshes, mats, device=dev)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    run = MapRunner(scene, grid, cfg, C4_TX, dev, rank, world)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = run.stream

    for _ in range(args.warmup):
        run.step()
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
            run.step(kern_ev[k])
            step_ev[k][1].record(stream)
            rb_counts.append(run.counters[run.rb_idx].clone())
        torch.cuda.synchronize()
    launches = _native.kernel_launches() - launches0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = np.array([a.elapsed_time(b) for a, b in step_ev])
    kern_ms = np.array([a.elapsed_time(b) for a, b in kern_ev])
    rb_total = int(sum(int(c.item()) for c in rb_counts))  # all ranks (all-reduced)
    t_max = max_over_ranks(float(step_ms.sum()), dev, world)
    value = rb_total / (t_max / 1e3)

    # ---- per-kernel split and roofline (extra untimed steps) ----
    kernels, rb_local = kernel_split(run, flush, 1)
    roof = roofline(kernels, rb_local, "c4")
    per_rank = None
    if world > 1:
        rows = gather_floats([float(rb_local), float(kern_ms.mean()),
                              roof["kernel_ms_per_step"]], dev, world)
        rbs = [r[0] for r in rows]
        kms = [r[1] for r in rows]
        per_rank = {"ray_bounces": rbs, "bounce_ms": kms,
                    "dominant_kernel_ms": [r[2] for r in rows],
                    "rb_max_over_mean": max(rbs) / (sum(rbs) / len(rbs)),
                    "ms_max_over_mean": max(kms) / (sum(kms) / len(kms))}

    # ---- end to end through the public API (host buffers) ----
    from paper_2504_21719_b200 import _abi
    e2e_ms = []
    rb_e2e = 0
    h2d = ctypes.sizeof(_abi.SbrMapParams)
    nx, ny = grid.shape
    d2h = nx * ny * 8 + _abi.SBR_MC_COUNT * 8
    n_e2e = max(1, min(args.steps, 5))
    for k in range(n_e2e + 1):  # first call untimed (warm-up, like the device-timed loop)
        flush.fill_(float(k))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0e.record(stream)
        if world == 1:
            host_vals, diag = compute_radio_map_sbr(scene, np.array(C4_TX), grid, cfg)
            rb_e2e = diag["ray_bounces"]
        else:
            v, c = compute_radio_map_sbr(scene, np.array(C4_TX), grid, cfg, shard=(rank, world),
                                         include_direct=(rank == 0), return_tensors=True)
            dist.all_reduce(v)
            dist.all_reduce(c)
            host_vals = v.cpu().numpy()
            rb_e2e = int(c[run.rb_idx].item())
        t1e.record(stream)
        torch.cuda.synchronize()
        if k > 0:
            e2e_ms.append(t0e.elapsed_time(t1e))
    e_max = max_over_ranks(float(np.sum(e2e_ms)), dev, world)
    e2e_value = rb_e2e * len(e2e_ms) / (e_max / 1e3)
    del host_vals

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        threads = cpu_threads()
        osc = oracle.OracleScene(meshes, mats)
        osc.bind_frequency(cfg.frequency)
        rate, rb_cpu, ns, dt = port_map_rate(osc, grid, cfg, C4_TX, threads,
                                             CPU_SAMPLES_PER_THREAD * threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{ns} of the 1e9 rays (1000 evenly spaced slices of the lattice), "
                         f"{rb_cpu} ray-bounces in {dt:.2f} s on {threads} threads"}

    c2 = None if args.no_config2 else bench_config2(args, dev, rank, world)
    cir = None if args.no_cir else bench_cir(args, dev, rank, world)
    c5 = None if args.no_config5 else bench_config5(args, dev, rank, world)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(t_max / args.steps), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(world, ntri),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": len(e2e_ms), "warmup": 1,
                    "ms_per_step": [round(x, 2) for x in e2e_ms]},
            "roofline": roof,
            "cpu_baseline": cpu,
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
            "ray_bounces_per_step": rb_total // args.steps,
            "bounce_call_ms_per_step": float(kern_ms.mean()),
            "scene_build_s": build_s,
            "per_rank": per_rank,
            "config2": c2,
            "cir": cir,
            "config5": c5,
        }
        print(json.dumps(line), flush=True)


def bench_config2(args, dev, rank=0, world=1):
    """Config 2: street canyon (11,600 tris) radio map, 1e7 rays per GPU (weak
    scaling: rank r traces its chunk-cyclic shard of an N*1e7 lattice), {R,S}
    depth 5, 200 x 200 cells.  Device ms per map (max over ranks), kernel split,
    roofline, e2e through compute_radio_map_sbr, and the port on a subsample."""
    import torch
    import torch.distributed as dist
    from paper_2504_21719_b200 import SceneModel
    from paper_2504_21719_b200.radiomap import compute_radio_map_sbr
    meshes, mats, grid, cfg = c2_workload(C2_SAMPLES_PER_GPU * world)
    scene = SceneModel(meshes, mats, device=dev)
    run = MapRunner(scene, grid, cfg, C2_TX, dev, rank, world)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(max(args.warmup, 2)):
        run.step()
    torch.cuda.synchronize()
    n = max(1, min(args.steps, 10))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(n)]
    rbs = []
    if world > 1:
        dist.barrier()
    for k in range(n):
        flush.fill_(float(k))
        evs[k][0].record(run.stream)
        run.step()
        evs[k][1].record(run.stream)
        rbs.append(run.counters[run.rb_idx].clone())
    torch.cuda.synchronize()
    times = [a.elapsed_time(b) for a, b in evs]
    ms = max_over_ranks(float(np.mean(times)), dev, world)
    rb = int(rbs[-1].item())
    kernels, rb_local = kernel_split(run, flush, 2)
    roof = roofline(kernels, rb_local, "c2")
    e2e = []
    for k in range(min(n, 5) + 1):  # first call untimed
        flush.fill_(float(k))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(run.stream)
        if world == 1:
            _, diag = compute_radio_map_sbr(scene, np.array(C2_TX), grid, cfg)
        else:
            v, c = compute_radio_map_sbr(scene, np.array(C2_TX), grid, cfg, shard=(rank, world),
                                         include_direct=(rank == 0), return_tensors=True)
            dist.all_reduce(v)
            dist.all_reduce(c)
            v.cpu()
        b.record(run.stream)
        torch.cuda.synchronize()
        if k > 0:
            e2e.append(a.elapsed_time(b))
    e_ms = max_over_ranks(float(np.mean(e2e)), dev, world)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        threads = cpu_threads()
        osc = oracle.OracleScene(meshes, mats)
        osc.bind_frequency(cfg.frequency)
        rate, rb_cpu, ns, dt = port_map_rate(osc, grid, cfg, C2_TX, threads,
                                             min(400_000 * threads, C2_SAMPLES_PER_GPU),
                                             pieces=400)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{ns} of the 1e7 rays (400 evenly spaced slices), {rb_cpu} "
                         f"ray-bounces in {dt:.2f} s on {threads} threads"}
    return {"workload": "config2: procedural street canyon (11,600 tris) radio map, 1e7 rays "
                        "per GPU, {R,S} depth 5, 200x200 cells of 1 m, Tx (0,5,20)",
            "value": rb / (ms / 1e3), "unit": UNIT, "ms_per_map": ms,
            "ray_bounces_per_map": rb, "n_gpus": world, "scaling": "weak", "maps": n,
            "e2e": {"value": rb / (e_ms / 1e3), "unit": UNIT, "ms_per_map": e_ms},
            "roofline": roof, "cpu_baseline": cpu}


def bench_cir(args, dev, rank=0, world=1):
    """Config 3: city CIR, 1 Tx x 1024 Rx, N_S = 1e6, depth 5, {R} (BASELINE configs[2]).

    ms per solve (generation + dedup + refinement + fields, host PathTensors
    out) timed with CUDA events on the current stream, max over ranks.  With
    N > 1 GPUs the solve is compute_paths_sharded: sample shards per rank,
    all-gathered candidate rows, replicated global selection (strong scaling:
    the same 1e6-sample solve split over the ranks).  Roofline of the dominant
    kernel k_cir_visibility at SURVEY §8d's 32 B per visibility ray.
    """
    import torch
    from paper_2504_21719_b200 import (PathConfig, RadioDevice, SceneModel, _native, scenes)
    from paper_2504_21719_b200.cir import _generate_device
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
    split = {}
    for k in ("k_cir_sweep", "k_cir_visibility"):
        ms_k, nl = _native.profile_kernel_ms(k)
        split[k] = {"ms_per_solve": ms_k / n, "launches_per_solve": nl / n}
    _native.profile_enable(False)
    ms = max_over_ranks(float(np.mean(times)), dev, world)
    d = ps.diagnostics
    roof = None
    if world == 1:
        # device counters of one (untimed) generation pass: closest-hit and visibility rays
        _, c, _ = _generate_device(scene, tx.position, np.array([r.position for r in rxs]), cfg)
        vis = split["k_cir_visibility"]
        peak, src = peaks()
        ach = c["visibility_rays"] * BYTES_PER_VIS / (vis["ms_per_solve"] / 1e3) / 1e9
        tr = profiled_traffic("k_cir_visibility", "c3")
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak, "kernel": "k_cir_visibility",
                "bytes_per_unit": BYTES_PER_VIS, "unit_name": "visibility ray",
                "units_per_launch": c["visibility_rays"] / max(vis["launches_per_solve"], 1),
                "kernel_ms": vis["ms_per_solve"] / max(vis["launches_per_solve"], 1),
                "traffic": tr.get("dram_bytes_per_launch") if tr else None,
                "visibility_rays": c["visibility_rays"],
                "visibility_rays_per_s": c["visibility_rays"] / (vis["ms_per_solve"] / 1e3),
                "closest_hit_ray_bounces": c["ray_bounces"], "rows_emitted": c["rows"],
                "algorithmic_bytes_per_solve": (BYTES_PER_RB * c["ray_bounces"]
                                                + BYTES_PER_VIS * c["visibility_rays"]
                                                + 64 * c["rows"]
                                                + 96 * d["candidates"] * cfg.max_depth),
                "peak_source": src}
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
            "kernel_ms_per_solve": split, "roofline": roof, "scene_build_s": build_s,
            "cpu_baseline": cpu,
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
    ms = max_over_ranks(float(np.mean(times)), dev, world)
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
    ap.add_argument("--no-config2", action="store_true")
    ap.add_argument("--no-cir", action="store_true")
    ap.add_argument("--no-config5", action="store_true")
    ap.add_argument("--no-emtrace", action="store_true")
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
