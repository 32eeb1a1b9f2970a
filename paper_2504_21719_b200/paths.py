"""Scene container, path-solver configuration and geometry hashing (host side).

Mirrors emtrace/paths.py:52-510 for the parts the device kernels consume:
`SceneModel` (BVH + per-slot plane hashes + per-object material rows),
`PathConfig`, `RadioDevice`, and the FNV-1a plane hashing that keys
candidate deduplication.  Plane hashes are computed here in float64 with the
reference's own vectorised expression (paths.py:156-171) and uploaded, so the
device hash chains are bit-identical to the reference's.

The CIR pipeline itself (generation, dedup, refinement, field replay, CFR)
lives in `cir.py` on top of csrc/sbr_cir.cu and csrc/sbr_fields.cu.
"""

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from .em import SPEED_OF_LIGHT, ArrayGeometry, make_pattern
from .errors import UnresolvedMaterial
from .geometry import EPS_COPLANAR, build_scene_accel  # noqa: F401
from .materials import pack_materials
from .sampling import Interaction

QUANT_RESOLUTION = 1e-4
MIN_HASH_CAPACITY = 1_000_000
HASH_CHAIN_BASE = 1373

_FNV_OFFSET = 0xCBF29CE484222325
_FNV_PRIME = 0x100000001B3
_MASK64 = 0xFFFFFFFFFFFFFFFF
_CANON_EPS = 1e-8


# ---------------------------------------------------------------------------
# hashing (paths.py:68-171)

def fnv1a_u64(value, seed=_FNV_OFFSET):
    """Fold the eight little-endian bytes of a 64-bit value into seed."""
    h = seed & _MASK64
    v = value & _MASK64
    for _ in range(8):
        h = ((h ^ (v & 0xFF)) * _FNV_PRIME) & _MASK64
        v >>= 8
    return h


def quantize_round(x):
    return int(math.floor(x / QUANT_RESOLUTION + 0.5))


def quantize_floor(x):
    return int(math.floor(x / QUANT_RESOLUTION))


def hash_update(current, contribution):
    return (HASH_CHAIN_BASE * current + contribution) & _MASK64


def pair_with_target(chain_hash, target_index):
    return fnv1a_u64(chain_hash, target_index)


def fnv1a_rows(values, seeds):
    """Vectorised fnv1a_u64 over uint64 arrays."""
    h = np.asarray(seeds, dtype=np.uint64).copy()
    v = np.asarray(values, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for shift in range(0, 64, 8):
            byte = (v >> np.uint64(shift)) & np.uint64(0xFF)
            h = (h ^ byte) * np.uint64(_FNV_PRIME)
    return h


def hash_plane(normal, point):
    """(round, floor) hashes of the plane through point (paths.py:86-108)."""
    n = np.asarray(normal, dtype=np.float64)
    n = n / np.linalg.norm(n)
    for c in n:
        if abs(c) > _CANON_EPS:
            if c < 0.0:
                n = -n
            break
    d = float(n @ np.asarray(point, dtype=np.float64))
    h_r, h_f = _FNV_OFFSET, _FNV_OFFSET
    for comp in (n[0], n[1], n[2], d):
        h_r = fnv1a_u64(quantize_round(comp) & _MASK64, h_r)
        h_f = fnv1a_u64(quantize_floor(comp) & _MASK64, h_f)
    return h_r, h_f


def plane_hash_rows(normals, points):
    """Vectorised hash_plane over row-aligned normals and points (paths.py:156-171)."""
    n = np.asarray(normals, dtype=np.float64)
    n = n / np.linalg.norm(n, axis=1, keepdims=True)
    significant = np.abs(n) > _CANON_EPS
    lead_idx = np.argmax(significant, axis=1)
    lead = n[np.arange(len(n)), lead_idx]
    n = np.where((lead < 0.0)[:, None], -n, n)
    d = np.sum(n * np.asarray(points, dtype=np.float64), axis=1)
    h_r = np.full(len(n), _FNV_OFFSET, dtype=np.uint64)
    h_f = h_r.copy()
    for comp in (n[:, 0], n[:, 1], n[:, 2], d):
        h_r = fnv1a_rows(np.floor(comp / QUANT_RESOLUTION + 0.5).astype(np.int64)
                         .astype(np.uint64), h_r)
        h_f = fnv1a_rows(np.floor(comp / QUANT_RESOLUTION).astype(np.int64)
                         .astype(np.uint64), h_f)
    return h_r, h_f


# ---------------------------------------------------------------------------
# configuration and devices

@dataclass(frozen=True)
class PathConfig:
    """Knobs of the path solver (paths.py:356-395)."""

    frequency: float = 3.5e9
    num_samples: int = 1_000_000
    max_depth: int = 3
    q_diffraction: float = 0.2
    enabled: frozenset = frozenset(Interaction)
    seed: int = 0
    buffer_capacity: int = None
    hash_capacity: int = None
    workers: int = 1
    synthetic_arrays: bool = True

    def __post_init__(self):
        if self.frequency <= 0.0:
            raise ValueError("frequency must be positive")
        if self.num_samples < 1:
            raise ValueError("num_samples must be positive")
        if self.max_depth < 0:
            raise ValueError("max_depth must be >= 0")
        if not 0.0 <= self.q_diffraction <= 1.0:
            raise ValueError("q_diffraction must lie in [0, 1]")
        if self.workers < 1:
            raise ValueError("workers must be positive")

    @property
    def wavelength(self):
        return SPEED_OF_LIGHT / self.frequency

    def resolved_buffer_capacity(self):
        if self.buffer_capacity is not None:
            return int(self.buffer_capacity)
        return int(self.num_samples)

    def resolved_hash_capacity(self):
        if self.hash_capacity is not None:
            return int(self.hash_capacity)
        return max(self.resolved_buffer_capacity(), MIN_HASH_CAPACITY)


def _default_array():
    return ArrayGeometry(np.zeros((1, 3)))


@dataclass(eq=False)
class RadioDevice:
    """Transmitter or receiver (paths.py:332-353)."""

    position: np.ndarray
    pattern: object = None
    array: ArrayGeometry = None
    velocity: np.ndarray = None
    name: str = ""

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=np.float64)
        if self.pattern is None:
            self.pattern = make_pattern("isotropic")
        if self.array is None:
            self.array = _default_array()
        if self.velocity is None:
            self.velocity = np.zeros(3)
        self.velocity = np.asarray(self.velocity, dtype=np.float64)

    def element_positions(self):
        return self.position[None, :] + self.array.offsets


# ---------------------------------------------------------------------------
# scene container

class SceneModel:
    """Meshes, materials and the device acceleration structures (paths.py:419-510).

    Differences from the reference, both deliberate:
      * the BVH is the device LBVH (slot order = Morton order);
      * diffraction wedges (wedges.py, the reference's extract_wedges) are
        extracted lazily on first use -- only configurations that enable
        diffraction pay for it -- and uploaded to the device with the
        per-slot wedge CSR (paths.py:452-475).
    """

    def __init__(self, meshes, materials, velocities=None,
                 dihedral_threshold_deg=1.0, device=None):
        self.meshes = list(meshes)
        self.materials = dict(materials)
        self.velocities = {k: np.asarray(v, dtype=np.float64)
                           for k, v in (velocities or {}).items()}
        for mesh in self.meshes:
            if mesh.object_id not in self.materials:
                raise UnresolvedMaterial(f"object {mesh.object_id} has no material")
        self.accel = build_scene_accel(self.meshes, device=device)
        self.dihedral_threshold_deg = dihedral_threshold_deg
        self._wedges = None
        self._build_tables()
        self._material_freq = None

    @property
    def wedges(self):
        """Diffracting edges (geometry.py:400-494), extracted and uploaded on first use."""
        if self._wedges is None:
            self._build_wedge_tables()
        return self._wedges

    def _build_wedge_tables(self):
        """Wedges, edge hashes and the per-slot wedge CSR (paths.py:452-475).

        Extraction and edge hashes run on the GPU (wedges.extract_wedges_device);
        the per-slot lists of owned wedges are built from the owners' input
        triangle indices through the BVH slot permutation.
        """
        from . import _abi, _native
        from .wedges import extract_wedges_device
        acc = self.accel
        W, t = extract_wedges_device(self.meshes, self.dihedral_threshold_deg, acc.device,
                                     accel=acc)
        nt = acc.num_triangles
        nw = len(W)
        if nw:
            # owners (o, m) of every wedge, deduplicated per wedge (set(w.owners()))
            wid0 = np.repeat(np.arange(nw), np.diff(t["off0"]))
            widn = np.repeat(np.arange(nw), np.diff(t["offn"]))
            tri = np.concatenate([t["tri0"], t["trin"]])
            wid = np.concatenate([wid0, widn])
            ids = sorted({m.object_id for m in self.meshes})
            if len(ids) == len(self.meshes):
                # input triangle -> slot (object ids identify the mesh)
                inv = np.empty(nt, np.int64)
                inv[acc.perm] = np.arange(nt)
                slot = inv[tri]
            else:   # shared object ids: the reference's (o, m) -> last slot mapping
                keys = zip(t["obj"][tri].tolist(), t["prim"][tri].tolist())
                slot = np.array([self._tri_slot.get(k, -1) for k in keys], np.int64)
            pairs = np.unique(np.stack([slot, wid], 1)[slot >= 0], axis=0)  # sorted (slot, wid)
            counts = np.bincount(pairs[:, 0], minlength=nt)
            self.tri_wedge_offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
            self.tri_wedge_ids = pairs[:, 1].astype(np.int64)
        else:
            counts = np.zeros(nt, np.int64)
            self.tri_wedge_offsets = np.zeros(nt + 1, np.int64)
            self.tri_wedge_ids = np.zeros(0, np.int64)
        self.tri_has_wedge = counts > 0
        self.wedge_hash_round = t["hash_r"] if nw else np.zeros(0, np.uint64)
        self.wedge_hash_floor = t["hash_f"] if nw else np.zeros(0, np.uint64)
        row = np.searchsorted(self._object_ids, t["obj"]) if nw else np.zeros(0, np.int64)
        if nw:
            first0 = t["tri0"][t["off0"][:-1]]                    # face0[0] (always present)
            has_n = np.diff(t["offn"]) > 0
            firstn = np.where(has_n, t["trin"][np.minimum(t["offn"][:-1], len(t["trin"]) - 1)]
                              if len(t["trin"]) else first0, first0)
            mat0, matn = row[first0], row[firstn]
        else:
            mat0 = matn = np.zeros(0, np.int64)
        keep = {
            "origin": t["origin"] if nw else np.zeros((0, 3)),
            "e_hat": t["e_hat"] if nw else np.zeros((0, 3)),
            "t0_hat": t["t0_hat"] if nw else np.zeros((0, 3)),
            "n0_hat": t["n0_hat"] if nw else np.zeros((0, 3)),
            "nn_hat": t["nn_hat"] if nw else np.zeros((0, 3)),
            "length": t["length"] if nw else np.zeros(0),
            "n_open": t["n_open"] if nw else np.zeros(0),
            "hash_r": self.wedge_hash_round, "hash_f": self.wedge_hash_floor,
            "mat0": np.asarray(mat0, np.int32), "matn": np.asarray(matn, np.int32),
            "slot_offsets": self.tri_wedge_offsets.astype(np.int32),
            "slot_ids": self.tri_wedge_ids.astype(np.int32),
        }
        keep = {k: np.ascontiguousarray(v) for k, v in keep.items()}
        tab = _abi.SbrWedgeTable()
        tab.n_wedges = nw
        for k, v in keep.items():
            setattr(tab, k, v.ctypes.data)
        _native.check(_native.load_library().sbr_scene_set_wedges(acc.handle, ctypes.byref(tab)))
        self._wedge_host = keep
        self._wedges = W

    def _build_tables(self):
        # the per-slot plane hashes (paths.py:449-450) are derived on the device
        # by sbr_scene_create from the float64 corners; host copies on demand
        accel = self.accel
        self._object_ids = np.array(sorted(m.object_id for m in self.meshes),
                                    dtype=np.int64)
        self._object_materials = [self.materials[oid] for oid in self._object_ids]
        # material row per slot (paths.py:497-499): one searchsorted per mesh
        mesh_row = np.searchsorted(self._object_ids, [m.object_id for m in self.meshes])
        sizes = [len(m.triangles) for m in self.meshes]
        self.tri_material_row = np.repeat(mesh_row, sizes)[accel.perm]
        self._slot_map = None
        accel.set_attributes(matrow=self.tri_material_row)

    @property
    def tri_plane_hash_round(self):
        return self.accel.tri_plane_hashes[0]

    @property
    def tri_plane_hash_floor(self):
        return self.accel.tri_plane_hashes[1]

    @property
    def _tri_slot(self):
        """{(object_id, primitive_id): slot} (paths.py:452-455), built on first use."""
        if self._slot_map is None:
            acc = self.accel
            self._slot_map = {(int(o), int(p)): i for i, (o, p) in
                              enumerate(zip(acc.tri_object_id.tolist(),
                                            acc.tri_primitive_id.tolist()))}
        return self._slot_map

    def bind_frequency(self, frequency):
        """Upload the per-object material rows frozen at `frequency`."""
        if self._material_freq != frequency:
            rows = pack_materials(self._object_materials, frequency)
            self.accel.set_materials(rows, len(self._object_materials))
            self._material_freq = frequency

    def material_of(self, object_id):
        return self.materials[object_id]

    def velocity_of(self, object_id):
        v = self.velocities.get(object_id)
        return v if v is not None else np.zeros(3)

    def primitive_owns_wedge(self, object_id, primitive_id):
        slot = self._tri_slot.get((int(object_id), int(primitive_id)))
        self.wedges  # noqa: B018  (ensure tables)
        return slot is not None and bool(self.tri_has_wedge[slot])
