"""Radio maps by shooting and bouncing rays on the GPU.

Drop-in for emtrace/radiomap.py:65-633 and 972-1023 (bounce estimator plus
the analytic direct term).  The whole per-segment loop of `_map_chunk`
(trace, plane crossing + deposit, culling, Fresnel/slab energies,
interaction draw, R/S/T field and direction update) runs in one persistent
sm_100a kernel (csrc/sbr_radiomap.cu) over global sample ids; the direct
term is a second kernel.  Python only packs parameters and reads back the
(ny, nx) float64 grid and the diagnostics counters.

Multi-GPU: `compute_radio_map_sbr(..., sample_range=(lo, hi))` traces a
shard of the global sample ids; the map is the sum of the shard maps
(`bench.py` all-reduces them over NCCL).  The RNG is keyed by global id,
so any sharding reproduces the single-GPU map up to float64 summation
order.
"""

import ctypes
import math
from collections import Counter
from dataclasses import dataclass

import numpy as np

from . import _abi, _native
from .em import SPEED_OF_LIGHT, make_pattern
from .sampling import Interaction, allow_mask

CHUNK_SAMPLES = 1 << _abi.SBR_CHUNK_LOG2
PLANE_TOLERANCE = 1e-6


@dataclass(eq=False)
class MeasurementGrid:
    """Planar rectangle of equal cells (radiomap.py:65-152); maps are indexed [j, i]."""

    center: np.ndarray
    u_hat: np.ndarray
    v_hat: np.ndarray
    cell_size: tuple
    shape: tuple

    def __post_init__(self):
        self.center = np.asarray(self.center, dtype=np.float64)
        self.u_hat = np.asarray(self.u_hat, dtype=np.float64)
        self.v_hat = np.asarray(self.v_hat, dtype=np.float64)
        for axis in (self.u_hat, self.v_hat):
            if abs(np.linalg.norm(axis) - 1.0) > 1e-9:
                raise ValueError("grid axes must be unit vectors")
        if abs(float(self.u_hat @ self.v_hat)) > 1e-9:
            raise ValueError("grid axes must be orthogonal")
        w, h = self.cell_size
        nx, ny = self.shape
        if w <= 0.0 or h <= 0.0:
            raise ValueError("cell size must be positive")
        if nx < 1 or ny < 1:
            raise ValueError("grid shape must be positive")
        self.cell_size = (float(w), float(h))
        self.shape = (int(nx), int(ny))

    @classmethod
    def horizontal(cls, center, extent, cell_size):
        w, h = cell_size
        nx = max(1, int(round(extent[0] / w)))
        ny = max(1, int(round(extent[1] / h)))
        return cls(center, (1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (float(w), float(h)),
                   (nx, ny))

    @property
    def normal(self):
        return np.cross(self.u_hat, self.v_hat)

    @property
    def cell_area(self):
        return self.cell_size[0] * self.cell_size[1]

    @property
    def corner(self):
        nx, ny = self.shape
        w, h = self.cell_size
        return (self.center - (0.5 * nx * w) * self.u_hat - (0.5 * ny * h) * self.v_hat)

    def cell_centers(self):
        nx, ny = self.shape
        w, h = self.cell_size
        u = (np.arange(nx) + 0.5) * w
        v = (np.arange(ny) + 0.5) * h
        return (self.corner + u[None, :, None] * self.u_hat
                + v[:, None, None] * self.v_hat)

    def cell_lookup(self, point):
        """Cell (i, j) containing a point on the plane, or None (higher index on ties)."""
        p = np.asarray(point, dtype=np.float64)
        rel = p - self.corner
        if abs(float(rel @ self.normal)) >= PLANE_TOLERANCE:
            return None
        i = math.floor(float(rel @ self.u_hat) / self.cell_size[0])
        j = math.floor(float(rel @ self.v_hat) / self.cell_size[1])
        nx, ny = self.shape
        if 0 <= i < nx and 0 <= j < ny:
            return (i, j)
        return None


@dataclass(frozen=True)
class RadioMapConfig:
    """Knobs of the map estimators (radiomap.py:169-215)."""

    frequency: float = 3.5e9
    num_samples: int = 10_000_000
    wedge_samples: int = 100_000
    max_depth: int = 3
    enabled: frozenset = frozenset(Interaction)
    seed: int = 0
    workers: int = 1
    rr_depth: int = None
    rr_max: float = 0.95
    gain_threshold: float = 0.0
    wedge_radius: float = None

    def __post_init__(self):
        if self.frequency <= 0.0:
            raise ValueError("frequency must be positive")
        if self.num_samples < 1:
            raise ValueError("num_samples must be positive")
        if self.wedge_samples < 1:
            raise ValueError("wedge_samples must be positive")
        if self.max_depth < 0:
            raise ValueError("max_depth must be >= 0")
        if self.workers < 1:
            raise ValueError("workers must be positive")
        if not 0.0 < self.rr_max <= 1.0:
            raise ValueError("rr_max must lie in (0, 1]")
        if self.rr_depth is not None and not 0 <= self.rr_depth <= self.max_depth:
            raise ValueError("rr_depth must lie in [0, max_depth]")
        if self.gain_threshold < 0.0:
            raise ValueError("gain_threshold must be >= 0")
        if self.wedge_radius is not None and self.wedge_radius <= 0.0:
            raise ValueError("wedge_radius must be positive")

    @property
    def wavelength(self):
        return SPEED_OF_LIGHT / self.frequency


@dataclass(eq=False)
class RadioMapResult:
    """Per-source cell gains on a shared grid (radiomap.py:969-980)."""

    grid: MeasurementGrid
    values: np.ndarray
    diagnostics: list

    def total(self):
        return self.values.sum(axis=0)


class exact_maps:
    """Context manager (and switch) for bitwise-reproducible maps.

    Inside `with exact_maps():` the map kernels accumulate cells as 192-bit
    fixed-point integers (sbr_set_exact_maps), so a map is bitwise identical
    for any deposit order, wave-stream count or run -- the reference's
    worker-count determinism (tests/test_radiomap.py:335-346).  Outside,
    float64 atomics: ~3 % faster, cells equal to ~1e-16 relative.
    """

    def __init__(self, enabled=True):
        self.enabled = bool(enabled)

    def __enter__(self):
        _native.check(_native.lib().sbr_set_exact_maps(int(self.enabled)))
        return self

    def __exit__(self, *exc):
        _native.check(_native.lib().sbr_set_exact_maps(0))
        return False


def russian_roulette_probability(distance, field_energy, p_max):
    return min(distance * distance * field_energy, p_max)


def _resolve_precoder(geometry, precoder):
    if geometry is None:
        return None
    m = len(geometry.offsets)
    if precoder is None:
        return np.full(m, 1.0 / math.sqrt(m), dtype=np.complex128)
    u_p = np.asarray(precoder, dtype=np.complex128)
    if u_p.shape != (m,):
        raise ValueError("precoder length must match the array")
    return u_p


def pack_map_params(scene, source, grid, cfg, pattern=None, array=None, precoder=None):
    """SbrMapParams plus the host arrays the pointers must reference.

    Returns (params, offsets (M,3) f64 or None, precoder (M,2) f64 or None);
    the caller uploads the arrays and patches elem_offsets_dev/precoder_dev.
    """
    if pattern is None:
        pattern = make_pattern("isotropic")
    precoder = _resolve_precoder(array, precoder)
    p = _abi.SbrMapParams()
    p.source = _abi.vec3(np.asarray(source, dtype=np.float64))
    p.corner = _abi.vec3(grid.corner)
    p.u_hat = _abi.vec3(grid.u_hat)
    p.v_hat = _abi.vec3(grid.v_hat)
    n_hat = grid.normal
    p.normal = _abi.vec3(n_hat)
    p.plane_off = float(n_hat @ grid.center)
    p.cell_w, p.cell_h = grid.cell_size
    lam = cfg.wavelength
    p.scale = (lam / (4.0 * np.pi)) ** 2 / grid.cell_area
    p.wavelength = lam
    p.omega0 = 4.0 * np.pi / cfg.num_samples
    p.rr_max = float(cfg.rr_max)
    p.gain_threshold = float(cfg.gain_threshold)
    p.num_samples = int(cfg.num_samples)
    p.seed = int(cfg.seed) & 0xFFFFFFFFFFFFFFFF
    p.nx, p.ny = grid.shape
    p.max_depth = int(cfg.max_depth)
    p.allow_mask = allow_mask(cfg.enabled) & 0x7  # D never inside the bounce loop
    p.rr_depth = -1 if cfg.rr_depth is None else int(cfg.rr_depth)
    p.cull_from = int(cfg.rr_depth) if cfg.rr_depth is not None else 0
    mats = scene._object_materials
    p.any_random_phase = int(any(m.random_phases for m in mats))
    p.pattern = pattern.to_abi()
    offs = prec = None
    if array is not None:
        offs = np.ascontiguousarray(array.offsets, dtype=np.float64)
        prec = np.ascontiguousarray(
            np.stack([precoder.real, precoder.imag], axis=1), dtype=np.float64)
        p.n_elements = len(offs)
    else:
        p.n_elements = 0
    return p, offs, prec


def _counters_to_diag(counts):
    return {name: int(counts[i]) for i, name in enumerate(_abi.MAP_COUNTERS)}


def compute_radio_map_sbr(scene, source, grid, cfg, *, pattern=None, array=None,
                          precoder=None, sample_range=None, shard=None, return_tensors=False,
                          include_direct=True):
    """Bounce-traced power map of one source, direct term included (radiomap.py:586-633).

    Returns (values (ny, nx) float64 numpy, diagnostics dict) like the
    reference.  Multi-GPU: `shard=(rank, world)` restricts the bounce
    estimator to a chunk-cyclic shard of the global sample ids (balanced: every
    shard spans the whole sphere), `sample_range=(lo, hi)` to a contiguous
    range; `include_direct=False` skips the analytic term (added once by one
    shard owner).  With `return_tensors=True` the device tensors are returned
    without a host copy.
    """
    import torch
    source = np.asarray(source, dtype=np.float64)
    accel = scene.accel
    dev = accel.device
    L = _native.lib()
    scene.bind_frequency(cfg.frequency)
    params, offs, prec = pack_map_params(scene, source, grid, cfg, pattern, array,
                                         precoder)
    keep = []
    if offs is not None:
        t_off = torch.from_numpy(offs).to(dev)
        t_pre = torch.from_numpy(prec).to(dev)
        keep += [t_off, t_pre]
        params.elem_offsets_dev = t_off.data_ptr()
        params.precoder_dev = t_pre.data_ptr()
    nx, ny = grid.shape
    lo, hi = (0, cfg.num_samples) if sample_range is None else sample_range
    values = torch.zeros((ny, nx), dtype=torch.float64, device=dev)
    counters = torch.zeros(_abi.SBR_MC_COUNT, dtype=torch.int64, device=dev)
    stream = _native.stream_ptr(dev)
    with torch.cuda.device(dev):
        if shard is not None:
            if sample_range is not None:
                raise ValueError("give either shard or sample_range")
            _native.check(L.sbr_radiomap_bounce_sharded(
                accel.handle, ctypes.byref(params), int(shard[0]), int(shard[1]),
                _native.ptr(values), _native.ptr(counters), stream))
        elif hi > lo:
            _native.check(L.sbr_radiomap_bounce(
                accel.handle, ctypes.byref(params), int(lo), int(hi),
                _native.ptr(values), _native.ptr(counters), stream))
        if include_direct:
            direct = torch.empty((ny, nx), dtype=torch.float64, device=dev)
            _native.check(L.sbr_radiomap_direct(
                accel.handle, ctypes.byref(params), _native.ptr(direct),
                _native.ptr(counters), stream))
            values += direct
    accel.check()
    if return_tensors:
        return values, counters
    counts = counters.cpu().numpy()
    if counts[_abi.MAP_COUNTERS.index("stack_overflow")]:
        raise RuntimeError("BVH traversal stack overflow")
    diag = Counter(samples=cfg.num_samples,
                   chunks=-(-cfg.num_samples // CHUNK_SAMPLES))
    for k, v in _counters_to_diag(counts).items():
        if k in ("stack_overflow",):
            continue
        if v or k in ("escaped", "ray_bounces"):
            diag[k] = v
    if include_direct:
        diag["direct_visible"] = int(counts[_abi.MAP_COUNTERS.index("direct_visible")])
    return values.cpu().numpy(), dict(diag)


PROBE_POINTS = 8


def _scene_diameter(scene):
    lo, hi = scene.accel.bounds
    return float(np.linalg.norm(hi - lo))


def collect_wedges_near_source(scene, source, radius):
    """Wedges within `radius` of the source, not hidden at all 8 probes (radiomap.py:645-671).

    The probe occlusion rays run on the GPU (Accel.occluded_batch).
    """
    source = np.asarray(source, dtype=np.float64)
    if not scene.wedges:
        return []
    W = scene._wedge_host
    origin, e_hat, length = W["origin"], W["e_hat"], W["length"]
    x = np.clip(np.sum((source - origin) * e_hat, axis=1), 0.0, length)
    foot = origin + x[:, None] * e_hat
    idx = np.nonzero(np.linalg.norm(source - foot, axis=1) <= radius)[0]
    if len(idx) == 0:
        return []
    frac = (np.arange(PROBE_POINTS) + 0.5) / PROBE_POINTS
    probes = (origin[idx, None, :] + (frac[None, :, None] * length[idx, None, None])
              * e_hat[idx, None, :]).reshape(-1, 3)
    blocked = scene.accel.occluded_batch(np.broadcast_to(source, probes.shape).copy(),
                                         probes).reshape(len(idx), PROBE_POINTS)
    return [int(i) for i in idx[~np.all(blocked, axis=1)]]


def compute_radio_map_diffraction(scene, source, grid, wedges, cfg, *, pattern=None, array=None,
                                  precoder=None, return_tensors=False):
    """Edge-diffracted power map of one source over the listed wedges (radiomap.py:842-965).

    One sm_100a kernel over all (wedge, sample) pairs: uniform (offset, cone
    azimuth) draws from the `map-wedge` stream keyed by (seed, wedge, block),
    plane crossing, exterior-region and occlusion tests, UTD transfer and the
    finite-difference area weighting; float64 atomic deposits.  Returns
    (values (ny, nx), diagnostics {wedges, cone_samples, deposits}).
    """
    import torch
    source = np.asarray(source, dtype=np.float64)
    scene.wedges  # noqa: B018  (wedge tables on the device)
    accel = scene.accel
    dev = accel.device
    L = _native.lib()
    scene.bind_frequency(cfg.frequency)
    params, offs, prec = pack_map_params(scene, source, grid, cfg, pattern, array, precoder)
    keep = []
    if offs is not None:
        t_off = torch.from_numpy(offs).to(dev)
        t_pre = torch.from_numpy(prec).to(dev)
        keep += [t_off, t_pre]
        params.elem_offsets_dev = t_off.data_ptr()
        params.precoder_dev = t_pre.data_ptr()
    nx, ny = grid.shape
    values = torch.zeros((ny, nx), dtype=torch.float64, device=dev)
    counters = torch.zeros(_abi.SBR_MC_COUNT, dtype=torch.int64, device=dev)
    ids = torch.tensor([int(w) for w in wedges], dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        if len(ids):
            _native.check(L.sbr_radiomap_wedges(
                accel.handle, ctypes.byref(params), _native.ptr(ids), len(ids),
                int(cfg.wedge_samples), _native.ptr(values), _native.ptr(counters),
                _native.stream_ptr(dev)))
    accel.check()
    if return_tensors:
        return values, counters
    c = counters.cpu().numpy()
    diag = {"wedges": len(ids), "cone_samples": int(c[_abi.MAP_COUNTERS.index("cone_samples")])}
    dep = int(c[_abi.MAP_COUNTERS.index("deposits")])
    if dep:
        diag["deposits"] = dep
    return values.cpu().numpy(), diag


def compute_radio_map(scene, transmitters, grid, cfg, *, precoders=None):
    """One value layer per transmitter (radiomap.py:985-1023).

    Transmitters may be RadioDevice instances or bare positions.  The
    bounce estimator always runs; with diffraction enabled the edge term
    (compute_radio_map_diffraction) is added over the wedges within
    `cfg.wedge_radius` (scene diameter when unset), as the reference does.
    """
    from .paths import RadioDevice
    devices = [t if isinstance(t, RadioDevice)
               else RadioDevice(position=np.asarray(t, dtype=np.float64))
               for t in transmitters]
    if precoders is not None and len(precoders) != len(devices):
        raise ValueError("need one precoder per transmitter")
    nx, ny = grid.shape
    values = np.zeros((len(devices), ny, nx))
    diagnostics = []
    for ti, dev in enumerate(devices):
        pre = None if precoders is None else precoders[ti]
        vals, diag = compute_radio_map_sbr(scene, dev.position, grid, cfg,
                                           pattern=dev.pattern, array=dev.array,
                                           precoder=pre)
        if Interaction.DIFFRACTION in cfg.enabled and scene.wedges:
            radius = (cfg.wedge_radius if cfg.wedge_radius is not None
                      else _scene_diameter(scene))
            ids = collect_wedges_near_source(scene, dev.position, radius)
            if ids:
                dvals, ddiag = compute_radio_map_diffraction(
                    scene, dev.position, grid, ids, cfg, pattern=dev.pattern, array=dev.array,
                    precoder=pre)
                vals = vals + dvals
                for key, count in ddiag.items():
                    diag[key] = diag.get(key, 0) + count
        values[ti] = vals
        diagnostics.append(diag)
    return RadioMapResult(grid=grid, values=values, diagnostics=diagnostics)
