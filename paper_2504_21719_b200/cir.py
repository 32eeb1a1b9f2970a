"""Path solver (CIR) on the GPU: candidate generation, dedup, refinement, fields, CFR.

Drop-in for emtrace/paths.py:174-1563 (diffraction branches excluded, SURVEY
§8f).  Every stage runs sm_100a kernels through the C ABI (include/sbr.h):

  generate_candidates   sbr_cir_sweep -> sbr_cir_visibility -> sbr_cir_select
                        -> sbr_cir_records   (paths.py:1019-1103)
  refine                sbr_cir_refine       (paths.py:1123-1252)
  fields                sbr_cir_fields       (paths.py:1302-1426)
  frequency_response    sbr_cfr              (paths.py:1519-1547)

Results stay on the device as structure-of-arrays tensors (`PathTensors`);
the reference's Python objects (`CandidateRecord`, `ValidPath`) are built
lazily, only when a caller touches `.records` / `.paths`.
"""

import ctypes
from collections import Counter
from dataclasses import dataclass, field

import numpy as np

from . import _abi, _native
from .paths import PathConfig
from .sampling import INTERACTION_ORDER, Interaction, allow_mask

_KIND_OF = {0: Interaction.REFLECTION, 1: Interaction.SCATTERING, 2: Interaction.TRANSMISSION,
            3: Interaction.DIFFRACTION}


# ---------------------------------------------------------------------------
# data model (paths.py:174-226, 233-412)

class DedupTable:
    """Fixed-size counting table deciding chain uniqueness (paths.py:174-204).

    Host data structure kept for API parity; the GPU pipeline resolves the
    same both-slot rule in bulk inside sbr_cir_select.
    """

    def __init__(self, capacity):
        if capacity < 1:
            raise ValueError("capacity must be positive")
        self.capacity = int(capacity)
        self.counts = np.zeros(self.capacity, dtype=np.int32)
        self.registered = 0
        self.duplicates = 0

    def register(self, paired_round, paired_floor):
        i1 = int(paired_round) % self.capacity
        i2 = int(paired_floor) % self.capacity
        if self.counts[i1] == 0 and self.counts[i2] == 0:
            self.counts[i1] += 1
            self.counts[i2] += 1
            self.registered += 1
            return True
        self.duplicates += 1
        return False

    def load_factor(self):
        return float(np.count_nonzero(self.counts)) / self.capacity


class PathBuffer:
    """Bounded candidate store that drops on overflow, never evicts (paths.py:207-226)."""

    def __init__(self, capacity):
        if capacity < 1:
            raise ValueError("capacity must be positive")
        self.capacity = int(capacity)
        self.items = []
        self.discarded = 0

    @property
    def full(self):
        return len(self.items) >= self.capacity

    def append(self, item):
        if self.full:
            self.discarded += 1
            return False
        self.items.append(item)
        return True


@dataclass(eq=False)
class InteractionStep:
    kind: Interaction
    object_id: int
    primitive_id: int
    vertex: np.ndarray
    normal: np.ndarray
    wedge_index: int = -1

    def __post_init__(self):
        self.vertex = np.asarray(self.vertex, dtype=np.float64)
        self.normal = np.asarray(self.normal, dtype=np.float64)


@dataclass(eq=False)
class CandidateRecord:
    source_id: int
    target_id: int
    source: np.ndarray
    target: np.ndarray
    sample_id: int
    steps: tuple
    suffix_start: int
    anchor: np.ndarray
    prefix_probability: float
    chain_hash: int
    diffuse_terminal: bool = False

    @property
    def depth(self):
        return len(self.steps)


@dataclass(eq=False)
class Rejection:
    reason: str
    detail: str = ""


@dataclass(eq=False)
class PathGeometry:
    source_id: int
    target_id: int
    sample_id: int
    vertices: np.ndarray
    steps: tuple
    chain_hash: int
    diffuse_terminal: bool = False

    @property
    def depth(self):
        return len(self.steps)


@dataclass(eq=False)
class ValidPath:
    tx_index: int
    tx_element: int
    rx_index: int
    rx_element: int
    gain: complex
    delay: float
    doppler: float
    departure: np.ndarray
    arrival: np.ndarray
    vertices: np.ndarray
    steps: tuple
    chain_hash: int
    sample_id: int

    @property
    def depth(self):
        return len(self.steps)

    @property
    def kinds(self):
        return "".join(step.kind.value for step in self.steps)


@dataclass(eq=False)
class GenerationResult:
    """Candidate records of one source; `records` is materialised lazily."""

    diagnostics: dict
    _device: object = None
    _records: list = None

    @property
    def records(self):
        if self._records is None:
            self._records = self._device.to_records() if self._device is not None else []
        return self._records


@dataclass(eq=False)
class PathTensors:
    """Structure-of-arrays view of a path set (host numpy, sorted like the reference)."""

    tx: np.ndarray
    tx_el: np.ndarray
    rx: np.ndarray
    rx_el: np.ndarray
    gain: np.ndarray          # complex128
    delay: np.ndarray
    doppler: np.ndarray
    departure: np.ndarray     # (n, 3)
    arrival: np.ndarray       # (n, 3)
    depth: np.ndarray
    chain_hash: np.ndarray    # uint64
    sample: np.ndarray
    kind: np.ndarray          # (n, L) int8, -1 unused
    obj: np.ndarray           # (n, L)
    prim: np.ndarray          # (n, L)
    wedge: np.ndarray         # (n, L) wedge index of D steps, -1
    normal: np.ndarray        # (n, L, 3)
    vertices: np.ndarray      # (n, L + 2, 3), rows padded after depth + 2

    def __len__(self):
        return len(self.delay)


@dataclass(eq=False)
class PathSet:
    """All paths of one solver run (paths.py:404-412); `paths` is built lazily."""

    tensors: PathTensors
    transmitters: list
    receivers: list
    config: PathConfig
    diagnostics: dict
    _paths: list = field(default=None)

    @property
    def paths(self):
        if self._paths is None:
            self._paths = _paths_from_tensors(self.tensors)
        return self._paths


def _paths_from_tensors(T):
    out = []
    for i in range(len(T)):
        d = int(T.depth[i])
        steps = tuple(
            InteractionStep(kind=_KIND_OF[int(T.kind[i, j])], object_id=int(T.obj[i, j]),
                            primitive_id=int(T.prim[i, j]), vertex=T.vertices[i, j + 1].copy(),
                            normal=T.normal[i, j].copy(), wedge_index=int(T.wedge[i, j]))
            for j in range(d))
        out.append(ValidPath(
            tx_index=int(T.tx[i]), tx_element=int(T.tx_el[i]), rx_index=int(T.rx[i]),
            rx_element=int(T.rx_el[i]), gain=complex(T.gain[i]), delay=float(T.delay[i]),
            doppler=float(T.doppler[i]), departure=T.departure[i].copy(),
            arrival=T.arrival[i].copy(), vertices=T.vertices[i, :d + 2].copy(), steps=steps,
            chain_hash=int(T.chain_hash[i]), sample_id=int(T.sample[i])))
    return out


# ---------------------------------------------------------------------------
# device pipeline

def _torch():
    import torch
    return torch


class _PhaseTimer:
    """SBR_TIMING=1: print wall time of each host phase (synchronising)."""

    def __init__(self, name):
        import os
        import time
        self.on = os.environ.get("SBR_TIMING") == "1"
        self.name, self.t, self.time = name, time.perf_counter(), time.perf_counter
        self.parts = []

    def mark(self, label):
        if self.on:
            _torch().cuda.synchronize()
            now = self.time()
            self.parts.append((label, now - self.t))
            self.t = now

    def report(self):
        if self.on:
            print(self.name, " ".join(f"{k}={v * 1e3:.1f}ms" for k, v in self.parts), flush=True)


def _check_cfg(cfg, scene=None):
    if cfg.max_depth > 15:
        raise ValueError("max_depth must be <= 15")
    if scene is not None and Interaction.DIFFRACTION in cfg.enabled:
        scene.wedges  # noqa: B018  -- extract + upload the wedge tables once


def _cir_params(source, targets_t, cfg):
    p = _abi.SbrCirParams()
    p.source = _abi.vec3(np.asarray(source, dtype=np.float64))
    p.q_diffraction = float(cfg.q_diffraction)
    p.num_samples = int(cfg.num_samples)
    p.seed = int(cfg.seed) & 0xFFFFFFFFFFFFFFFF
    p.max_depth = int(cfg.max_depth)
    p.allow_mask = allow_mask(cfg.enabled) & 0xF
    p.n_targets = int(targets_t.shape[0])
    p.targets_dev = targets_t.data_ptr()
    return p


class _VertexBuf:
    def __init__(self, capacity, dev):
        torch = _torch()
        c = max(int(capacity), 1)
        self.t = {
            "point": torch.empty((c, 3), dtype=torch.float64, device=dev),
            "normal": torch.empty((c, 3), dtype=torch.float64, device=dev),
            "run_prob": torch.empty(c, dtype=torch.float64, device=dev),
            "sample": torch.empty(c, dtype=torch.int64, device=dev),
            "hash_r": torch.empty(c, dtype=torch.uint64, device=dev),
            "hash_f": torch.empty(c, dtype=torch.uint64, device=dev),
            "parent": torch.empty(c, dtype=torch.int32, device=dev),
            "tri": torch.empty(c, dtype=torch.int32, device=dev),
            "code": torch.empty(c, dtype=torch.uint8, device=dev),
            "depth": torch.empty(c, dtype=torch.uint8, device=dev),
            "suffix_start": torch.empty(c, dtype=torch.uint8, device=dev),
            "wedge": torch.empty(c, dtype=torch.int32, device=dev),
        }
        self.abi = _abi.SbrVertexBuf()
        for k, v in self.t.items():
            setattr(self.abi, k, v.data_ptr())
        self.abi.capacity = c


class _RecordBuf:
    def __init__(self, n, L, dev):
        torch = _torch()
        n = max(int(n), 1)
        self.n, self.L = n, L
        self.t = {
            "target": torch.empty(n, dtype=torch.int32, device=dev),
            "sample": torch.empty(n, dtype=torch.int64, device=dev),
            "depth": torch.empty(n, dtype=torch.int32, device=dev),
            "suffix_start": torch.empty(n, dtype=torch.int32, device=dev),
            "diffuse": torch.empty(n, dtype=torch.uint8, device=dev),
            "chain_hash": torch.empty(n, dtype=torch.uint64, device=dev),
            "prefix_prob": torch.empty(n, dtype=torch.float64, device=dev),
            "anchor": torch.empty((n, 3), dtype=torch.float64, device=dev),
            "kind": torch.empty((n, L), dtype=torch.int8, device=dev),
            "tri": torch.empty((n, L), dtype=torch.int32, device=dev),
            "vertex": torch.zeros((n, L, 3), dtype=torch.float64, device=dev),
            "normal": torch.zeros((n, L, 3), dtype=torch.float64, device=dev),
            "wedge": torch.full((n, L), -1, dtype=torch.int32, device=dev),
        }
        self.abi = _abi.SbrRecordBuf()
        for k, v in self.t.items():
            setattr(self.abi, k, v.data_ptr())
        self.abi.max_depth = L


class DeviceCandidates:
    """Device-resident candidate records of one source (output of generation)."""

    def __init__(self, scene, source, targets, targets_t, cfg, recbuf, n, source_id):
        self.scene, self.source, self.targets = scene, source, targets
        self.targets_t, self.cfg, self.rec, self.n = targets_t, cfg, recbuf, n
        self.source_id = source_id

    def to_records(self):
        """Materialise CandidateRecord objects (paths.py:990-1016)."""
        if self.n == 0:
            return []
        h = {k: v[:self.n].cpu().numpy() for k, v in self.rec.t.items()}
        acc = self.scene.accel
        out = []
        for i in range(self.n):
            d = int(h["depth"][i])
            steps = []
            for j in range(d):
                slot = int(h["tri"][i, j])
                steps.append(InteractionStep(
                    kind=_KIND_OF[int(h["kind"][i, j])],
                    object_id=int(acc.tri_object_id[slot]),
                    primitive_id=int(acc.tri_primitive_id[slot]),
                    vertex=h["vertex"][i, j].copy(), normal=h["normal"][i, j].copy(),
                    wedge_index=int(h["wedge"][i, j])))
            k = int(h["target"][i])
            out.append(CandidateRecord(
                source_id=self.source_id, target_id=k, source=np.asarray(self.source),
                target=self.targets[k], sample_id=int(h["sample"][i]), steps=tuple(steps),
                suffix_start=int(h["suffix_start"][i]), anchor=h["anchor"][i].copy(),
                prefix_probability=float(h["prefix_prob"][i]),
                chain_hash=int(h["chain_hash"][i]), diffuse_terminal=bool(h["diffuse"][i])))
        return out


def _counters_dict(c):
    return {name: int(c[i]) for i, name in enumerate(_abi.CIR_COUNTERS)}


class _Rows:
    """Visible (vertex, target) rows of one source on this device."""


def _sweep_rows(scene, source, targets, cfg, lo, hi, shard=None):
    """Sweep global sample ids [lo, hi) -- or, with shard=(rank, world), the
    chunk-cyclic shard sbr_cir_sweep_sharded owns -- and collect visible rows
    + dedup keys.

    _sweep_chunk's trace/draw/continue loop (paths.py:704-828) and
    _visible_pairs (657-683) on the GPU; the rows carry the ordinal key
    (depth, sample, target), the vertex index and the pair hashes.
    """
    torch = _torch()
    L_ = _native.lib()
    acc = scene.accel
    dev = acc.device
    R = _Rows()
    R.dev = dev
    stream = _native.stream_ptr(dev)
    R.targets_t = torch.from_numpy(np.ascontiguousarray(targets)).to(dev)
    R.params = _cir_params(source, R.targets_t, cfg)
    R.counters = counters = torch.zeros(_abi.SBR_CC_COUNT, dtype=torch.int64, device=dev)
    # line of sight (generate_candidates 1036-1049)
    occ = acc.occluded_batch(torch.from_numpy(np.broadcast_to(source, targets.shape).copy())
                             .to(dev), R.targets_t)
    R.los_vis = (~occ).to(torch.uint8).contiguous()
    gt = _PhaseTimer("  generate")
    gt.mark("los")
    if shard is not None:
        from .sharding import cyclic_chunks
        n_ids = sum(b - a for a, b in cyclic_chunks(cfg.num_samples, shard[0], shard[1],
                                                    chunk=1 << _abi.SBR_CIR_SHARD_LOG2))
    else:
        n_ids = hi - lo
    R.vb = vb = _VertexBuf(n_ids * cfg.max_depth, dev)
    if n_ids > 0 and cfg.max_depth > 0:
        if shard is not None:
            _native.check(L_.sbr_cir_sweep_sharded(acc.handle, ctypes.byref(R.params),
                                                   int(shard[0]), int(shard[1]),
                                                   ctypes.byref(vb.abi), _native.ptr(counters),
                                                   stream))
        else:
            _native.check(L_.sbr_cir_sweep(acc.handle, ctypes.byref(R.params), lo, hi,
                                           ctypes.byref(vb.abi), _native.ptr(counters), stream))
    nv = int(counters[_abi.CC["vertices"]].item())
    gt.mark("sweep")
    # visibility rows, vertex slabs of <= 2^26 (vertex, target) pairs; before
    # each slab the row buffer is grown (geometrically) to hold the slab's
    # worst case, so no slab is ever traced twice
    nt = len(targets)
    order = torch.empty(max(nv, 1), dtype=torch.int32, device=dev)
    if nv:
        _native.check(L_.sbr_cir_vertex_order(acc.handle, ctypes.byref(vb.abi), nv,
                                              _native.ptr(order), stream))
    slab = max(32, ((1 << 26) // nt) // 32 * 32)
    # room for several slabs' worst case, so the row count is read back (a
    # host sync) only when the slabs launched since the last read could
    # overflow the buffer, not after every slab
    cap = max(1 << 20, min(nv * nt, max(int(nv * nt * 0.03), 4 * slab * nt)))
    row_key = torch.empty(cap, dtype=torch.uint64, device=dev)
    row_vtx = torch.empty(cap, dtype=torch.int32, device=dev)
    nrows = 0  # rows known after the last read-back
    bound = 0  # nrows + worst case of the slabs launched since
    for v0 in range(0, nv, slab):
        v1 = min(nv, v0 + slab)
        if bound + (v1 - v0) * nt > cap:
            nrows = int(counters[_abi.CC["rows"]].item())
            bound = nrows
            need = nrows + (v1 - v0) * nt
            if need > cap:
                cap = max(need, int(cap * 1.5))
                nk = torch.empty(cap, dtype=torch.uint64, device=dev)
                nv_ = torch.empty(cap, dtype=torch.int32, device=dev)
                nk[:nrows].copy_(row_key[:nrows])
                nv_[:nrows].copy_(row_vtx[:nrows])
                row_key, row_vtx = nk, nv_
        _native.check(L_.sbr_cir_visibility(
            acc.handle, ctypes.byref(R.params), ctypes.byref(vb.abi), v0, v1,
            _native.ptr(order), _native.ptr(row_key), _native.ptr(row_vtx), cap,
            _native.ptr(counters), stream))
        bound += (v1 - v0) * nt
    nrows = int(counters[_abi.CC["rows"]].item())
    if nrows > cap:
        raise RuntimeError("visibility row buffer overflow")  # cannot happen
    acc.check()
    gt.mark("visibility")
    R.n = nrows
    R.key, R.vtx = row_key[:nrows], row_vtx[:nrows]
    m = max(nrows, 1)
    R.pr = torch.empty(m, dtype=torch.uint64, device=dev)
    R.pf = torch.empty(m, dtype=torch.uint64, device=dev)
    R.chain = torch.empty(m, dtype=torch.uint8, device=dev)
    if nrows:
        _native.check(L_.sbr_cir_row_pairs(ctypes.byref(vb.abi), _native.ptr(R.key),
                                           _native.ptr(R.vtx), nrows, _native.ptr(R.pr),
                                           _native.ptr(R.pf), _native.ptr(R.chain), stream))
    R.timer = gt
    return R


def _select_rows(params, key, pr, pf, chain, n, los_vis, cfg, counters, dev):
    """sbr_cir_select over (possibly all-gathered) rows -> rec_row tensor, count."""
    torch = _torch()
    L_ = _native.lib()
    n_buffer = cfg.resolved_buffer_capacity()
    rec_cap = max(1, min(n_buffer, n + int(los_vis.numel())))
    rec_row = torch.empty(rec_cap, dtype=torch.int64, device=dev)
    n_rec = ctypes.c_int64(0)
    _native.check(L_.sbr_cir_select(
        ctypes.byref(params), _native.ptr(key), _native.ptr(pr), _native.ptr(pf),
        _native.ptr(chain), n, _native.ptr(los_vis), cfg.resolved_hash_capacity(), n_buffer,
        _native.ptr(rec_row), ctypes.byref(n_rec), _native.ptr(counters),
        _native.stream_ptr(dev)))
    return rec_row, int(n_rec.value)


def _local_rows(R):
    """Shard-local pre-selection (sbr_cir_local_dedup): the rows worth
    all-gathering, as (dict of row tensors, kept row indices, dropped count)."""
    torch = _torch()
    L_ = _native.lib()
    n = R.n
    kept = torch.empty(max(n, 1), dtype=torch.int64, device=R.dev)
    nk, nd = ctypes.c_int64(0), ctypes.c_uint64(0)
    _native.check(L_.sbr_cir_local_dedup(
        ctypes.byref(R.params), _native.ptr(R.key), _native.ptr(R.pr), _native.ptr(R.pf),
        _native.ptr(R.chain), n, _native.ptr(kept), ctypes.byref(nk), ctypes.byref(nd),
        _native.stream_ptr(R.dev)))
    kept = kept[:int(nk.value)]
    rows = {"key": R.key[:n].index_select(0, kept), "pr": R.pr[:n].index_select(0, kept),
            "pf": R.pf[:n].index_select(0, kept), "chain": R.chain[:n].index_select(0, kept)}
    return rows, kept, int(nd.value)


def _materialize(R, rec_row, n, cfg):
    """CandidateRecord arrays for rec_row entries that index R's own rows."""
    torch = _torch()
    L_ = _native.lib()
    dev = R.dev
    L = max(int(cfg.max_depth), 1)
    recbuf = _RecordBuf(n, L, dev)
    if n:
        stream = _native.stream_ptr(dev)
        rec_vtx = torch.empty(n, dtype=torch.int32, device=dev)
        rec_tgt = torch.empty(n, dtype=torch.int32, device=dev)
        _native.check(L_.sbr_cir_resolve_records(_native.ptr(rec_row), n, _native.ptr(R.key),
                                                 _native.ptr(R.vtx), _native.ptr(rec_vtx),
                                                 _native.ptr(rec_tgt), stream))
        _native.check(L_.sbr_cir_records(ctypes.byref(R.params), ctypes.byref(R.vb.abi),
                                         _native.ptr(rec_vtx), _native.ptr(rec_tgt), n,
                                         ctypes.byref(recbuf.abi), stream))
    return recbuf


def _gen_diag(c, cfg):
    return {
        "samples_escaped": c["samples_escaped"],
        "samples_terminated": c["samples_terminated"],
        "duplicates": c["duplicates"],
        "chunk_truncated": c["chunk_truncated"],
        "buffer_overflow": c["buffer_overflow"],
        "candidates": c["candidates"],
        "hash_load_factor": c["hash_slots"] / float(cfg.resolved_hash_capacity()),
        "hash_registered": c["hash_registered"],
    }


def _generate_device(scene, source, targets, cfg, source_id=0, sample_range=None):
    """Run sweep -> visibility -> select -> records on the scene's device.

    Returns (DeviceCandidates, counters dict, generation diagnostics dict).
    """
    torch = _torch()
    _check_cfg(cfg, scene)
    acc = scene.accel
    dev = acc.device
    scene.bind_frequency(cfg.frequency)
    source = np.asarray(source, dtype=np.float64)
    targets = np.atleast_2d(np.asarray(targets, dtype=np.float64))
    if len(targets) == 0:
        raise ValueError("at least one target is required")
    lo, hi = (0, int(cfg.num_samples)) if sample_range is None else map(int, sample_range)
    with torch.cuda.device(dev):
        R = _sweep_rows(scene, source, targets, cfg, lo, hi)
        rec_row, n = _select_rows(R.params, R.key, R.pr, R.pf, R.chain, R.n, R.los_vis, cfg,
                                  R.counters, dev)
        R.timer.mark("select")
        recbuf = _materialize(R, rec_row, n, cfg)
        c = _counters_dict(R.counters.cpu().numpy())
        R.timer.mark("records")
        R.timer.report()
    if c["stack_overflow"]:
        raise RuntimeError("BVH traversal stack overflow")
    cand = DeviceCandidates(scene, source, targets, R.targets_t, cfg, recbuf, n, source_id)
    cand.params = R.params
    return cand, c, _gen_diag(c, cfg)


def generate_candidates(scene, source, targets, cfg, source_id=0):
    """Shoot the sample lattice from one source and collect candidates (paths.py:1019).

    Same semantics as the reference at workers=1 (and, without buffer
    overflow, at any worker count): LoS records first, then chain and
    diffuse records in (depth, sample, target) order, deduplicated by the
    both-slot hash rule and capped at the buffer capacity.
    """
    cand, _, diag = _generate_device(scene, source, targets, cfg, source_id)
    return GenerationResult(diagnostics=diag, _device=cand)


def _refine_device(scene, cand):
    """Image-method refinement of every candidate (paths.py:1123-1252)."""
    torch = _torch()
    L_ = _native.lib()
    dev = scene.accel.device
    n, L = cand.n, cand.rec.L
    pv = torch.zeros((max(n, 1), L + 2, 3), dtype=torch.float64, device=dev)
    status = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
    counters = torch.zeros(_abi.SBR_CC_COUNT, dtype=torch.int64, device=dev)
    if n:
        with torch.cuda.device(dev):
            _native.check(L_.sbr_cir_refine(scene.accel.handle, ctypes.byref(cand.params),
                                            ctypes.byref(cand.rec.abi), n, _native.ptr(pv),
                                            _native.ptr(status), _native.ptr(counters),
                                            _native.stream_ptr(dev)))
    return pv, status, counters


def refine_candidate(record, scene):
    """Exact geometry of one candidate or the reason it fails (paths.py:1123-1245).

    Runs the device refinement kernel on a single packed record.
    """
    torch = _torch()
    dev = scene.accel.device
    steps = record.steps
    if any(st.kind is Interaction.DIFFRACTION for st in steps):
        scene.wedges  # noqa: B018  (wedge tables on the device)
    L = max(len(steps), 1)
    rec = _RecordBuf(1, L, dev)
    acc = scene.accel
    kinds = np.full(L, -1, np.int8)
    tris = np.full(L, -1, np.int32)
    wed = np.full(L, -1, np.int32)
    verts = np.zeros((L, 3))
    norms = np.zeros((L, 3))
    for j, st in enumerate(steps):
        kinds[j] = INTERACTION_ORDER.index(st.kind)
        tris[j] = scene._tri_slot[(int(st.object_id), int(st.primitive_id))]
        verts[j] = st.vertex
        norms[j] = st.normal
        wed[j] = st.wedge_index
    vals = {
        "target": np.array([0], np.int32), "sample": np.array([record.sample_id], np.int64),
        "depth": np.array([len(steps)], np.int32),
        "suffix_start": np.array([record.suffix_start], np.int32),
        "diffuse": np.array([bool(record.diffuse_terminal)], np.uint8),
        "chain_hash": np.array([record.chain_hash & 0xFFFFFFFFFFFFFFFF], np.uint64),
        "prefix_prob": np.array([record.prefix_probability]),
        "anchor": np.asarray(record.anchor, np.float64)[None, :],
        "kind": kinds[None, :], "tri": tris[None, :], "vertex": verts[None], "normal": norms[None],
        "wedge": wed[None, :],
    }
    for k, v in vals.items():
        rec.t[k].copy_(torch.from_numpy(np.ascontiguousarray(v)).reshape(rec.t[k].shape))
    tgt = torch.from_numpy(np.asarray(record.target, np.float64)[None, :].copy()).to(dev)
    cfg = PathConfig(num_samples=1, max_depth=L)
    if scene._material_freq is None:
        # refinement is geometric, but the kernel reads the material table; a
        # fresh scene (no solver run yet) binds the default frequency, as the
        # reference's refine_candidate needs no prior solve
        scene.bind_frequency(cfg.frequency)
    cand = DeviceCandidates(scene, record.source, np.asarray(record.target)[None, :], tgt, cfg,
                            rec, 1, record.source_id)
    cand.params = _cir_params(record.source, tgt, cfg)
    pv, status, _ = _refine_device(scene, cand)
    st = int(status[0].item())
    if st != _abi.SBR_REFINE_OK:
        return Rejection(_abi.REJECTION_NAMES[st])
    d = len(steps)
    v = pv[0, :d + 2].cpu().numpy()
    new_steps = tuple(InteractionStep(kind=s.kind, object_id=s.object_id,
                                      primitive_id=s.primitive_id, vertex=v[j + 1].copy(),
                                      normal=s.normal, wedge_index=s.wedge_index)
                      for j, s in enumerate(steps))
    return PathGeometry(source_id=record.source_id, target_id=record.target_id,
                        sample_id=record.sample_id, vertices=v, steps=new_steps,
                        chain_hash=record.chain_hash,
                        diffuse_terminal=record.diffuse_terminal)


def _antenna_table(patterns, dev):
    """Device array of SbrAntenna descriptors, one per target; patterns are packed
    once per distinct (name, orientation) -- 1024 receivers usually share one."""
    torch = _torch()
    packed, rows = {}, []
    for p in patterns:
        key = (p.name, tuple(float(x) for x in p.orientation))
        if key not in packed:
            packed[key] = bytes(p.to_abi())
        rows.append(packed[key])
    raw = np.frombuffer(b"".join(rows), dtype=np.uint8).copy()
    return torch.from_numpy(raw).to(dev)


def _fields_device(scene, cand, pv, status, tx_dev, target_devices, cfg):
    """Algorithm-2 field replay for every refined candidate (paths.py:1302-1426)."""
    torch = _torch()
    L_ = _native.lib()
    dev = scene.accel.device
    n = cand.n
    fp = _abi.SbrFieldParams()
    fp.wavelength = cfg.wavelength
    fp.q_diffraction = float(cfg.q_diffraction)
    fp.tx_velocity = _abi.vec3(tx_dev.velocity)
    fp.num_samples = int(cfg.num_samples)
    fp.seed = int(cfg.seed) & 0xFFFFFFFFFFFFFFFF
    fp.allow_mask = allow_mask(cfg.enabled) & 0xF
    fp.tx_pattern = tx_dev.pattern.to_abi()
    rx_pat = _antenna_table([d.pattern for d in target_devices], dev)
    rx_vel = torch.from_numpy(np.array([d.velocity for d in target_devices],
                                       dtype=np.float64).reshape(-1, 3)).to(dev)
    obj_ids = scene._object_ids
    vel = np.zeros((len(obj_ids), 3))
    if scene.velocities:
        vel = np.array([scene.velocity_of(int(o)) for o in obj_ids],
                       dtype=np.float64).reshape(-1, 3)
    obj_vel = torch.from_numpy(vel).to(dev)
    fp.rx_pattern_dev = rx_pat.data_ptr()
    fp.rx_velocity_dev = rx_vel.data_ptr()
    fp.obj_velocity_dev = obj_vel.data_ptr()
    fp.n_objects = len(obj_ids) if np.any(vel) else 0
    m = max(n, 1)
    out = {
        "gain": torch.zeros((m, 2), dtype=torch.float64, device=dev),
        "delay": torch.zeros(m, dtype=torch.float64, device=dev),
        "doppler": torch.zeros(m, dtype=torch.float64, device=dev),
        "departure": torch.zeros((m, 3), dtype=torch.float64, device=dev),
        "arrival": torch.zeros((m, 3), dtype=torch.float64, device=dev),
    }
    if n:
        with torch.cuda.device(dev):
            _native.check(L_.sbr_cir_fields(
                scene.accel.handle, ctypes.byref(fp), ctypes.byref(cand.rec.abi),
                _native.ptr(pv), _native.ptr(status), n, _native.ptr(out["gain"]),
                _native.ptr(out["delay"]), _native.ptr(out["doppler"]),
                _native.ptr(out["departure"]), _native.ptr(out["arrival"]),
                _native.stream_ptr(dev)))
    return out


def _flatten_devices(devices, synthetic):
    flat = []
    for di, d in enumerate(devices):
        if synthetic:
            flat.append((di, 0, d.position))
        else:
            for ei, pos in enumerate(d.element_positions()):
                flat.append((di, ei, pos))
    return flat


def _paths_for_source(scene, cand, cfg, ti, te, tx_dev, target_devices, rx_index, rx_elem,
                      timer=None):
    """Refine + replay the candidates of one source; SoA part of valid paths."""
    torch = _torch()
    acc = scene.accel
    rejections = Counter()
    pv, status, rc = _refine_device(scene, cand)
    if timer:
        timer.mark("refine")
    rcount = rc.cpu().numpy()
    for code, name in _abi.REJECTION_NAMES.items():
        cnt = int(rcount[_abi.CC[_abi.REJECTION_COUNTERS[code]]])
        if cnt:
            rejections[name] += cnt
    f = _fields_device(scene, cand, pv, status, tx_dev, target_devices, cfg)
    if timer:
        timer.mark("fields")
    n = cand.n
    if n == 0:
        return None, rejections
    ok_idx = torch.nonzero(status[:n] == _abi.SBR_REFINE_OK).squeeze(1)
    m = int(ok_idx.numel())
    h = {k: v[:n].index_select(0, ok_idx).cpu().numpy() for k, v in cand.rec.t.items()
         if k != "chain_hash"}
    h["chain_hash"] = cand.rec.t["chain_hash"][:n].cpu().numpy()[ok_idx.cpu().numpy()]
    fh = {k: v[:n].index_select(0, ok_idx).cpu().numpy() for k, v in f.items()}
    pvh = pv[:n].index_select(0, ok_idx).cpu().numpy()
    tri = h["tri"]
    valid = tri >= 0
    obj = np.where(valid, acc.tri_object_id[np.maximum(tri, 0)], -1)
    prim = np.where(valid, acc.tri_primitive_id[np.maximum(tri, 0)], -1)
    tg = h["target"].astype(np.int64)
    part = dict(
        tx=np.full(m, ti, np.int64), tx_el=np.full(m, te, np.int64),
        rx=rx_index[tg], rx_el=rx_elem[tg],
        gain=fh["gain"][:, 0] + 1j * fh["gain"][:, 1], delay=fh["delay"],
        doppler=fh["doppler"], departure=fh["departure"], arrival=fh["arrival"],
        depth=h["depth"].astype(np.int64), chain_hash=h["chain_hash"], sample=h["sample"],
        kind=h["kind"], obj=obj, prim=prim, wedge=np.where(valid, h["wedge"], -1),
        normal=h["normal"], vertices=pvh)
    if timer:
        timer.mark("host_copy")
    return part, rejections


def _device_plan(transmitters, receivers, cfg):
    tx_flat = _flatten_devices(transmitters, cfg.synthetic_arrays)
    rx_flat = _flatten_devices(receivers, cfg.synthetic_arrays)
    targets = np.array([pos for _, _, pos in rx_flat])
    target_devices = [receivers[ri] for ri, _, _ in rx_flat]
    rx_index = np.array([ri for ri, _, _ in rx_flat], np.int64)
    rx_elem = np.array([re for _, re, _ in rx_flat], np.int64)
    return tx_flat, targets, target_devices, rx_index, rx_elem


def compute_paths(scene, transmitters, receivers, cfg):
    """All propagation paths between the given devices (paths.py:1444-1516).

    Sorted by (rx, rx_element, tx, tx_element, depth, chain_hash, sample).
    Returns a PathSet whose `tensors` holds the SoA arrays; `paths` builds
    the reference's ValidPath objects on first access.
    """
    transmitters = list(transmitters)
    receivers = list(receivers)
    if not transmitters or not receivers:
        raise ValueError("need at least one transmitter and one receiver")
    _check_cfg(cfg, scene)
    tx_flat, targets, target_devices, rx_index, rx_elem = _device_plan(transmitters, receivers,
                                                                       cfg)
    diagnostics = Counter()
    rejections = Counter()
    load_factor = 0.0
    parts = []
    timer = _PhaseTimer("compute_paths")
    for src_idx, (ti, te, tx_pos) in enumerate(tx_flat):
        cand, _, gdiag = _generate_device(scene, tx_pos, targets, cfg, source_id=src_idx)
        timer.mark("generate")
        load_factor = max(load_factor, gdiag["hash_load_factor"])
        for k, v in gdiag.items():
            if k != "hash_load_factor":
                diagnostics[k] += v
        part, rej = _paths_for_source(scene, cand, cfg, ti, te, transmitters[ti],
                                      target_devices, rx_index, rx_elem, timer)
        rejections.update(rej)
        if part is not None:
            parts.append(part)
    tensors = _concat_sorted(parts, max(int(cfg.max_depth), 1))
    timer.mark("sort")
    timer.report()
    result = dict(diagnostics)
    result["hash_load_factor"] = load_factor
    result["refinement_rejections"] = dict(rejections)
    result["paths"] = len(tensors)
    return PathSet(tensors=tensors, transmitters=transmitters, receivers=receivers, config=cfg,
                   diagnostics=result)


def compute_paths_sharded(scene, transmitters, receivers, cfg, group=None):
    """compute_paths over all ranks of a torch.distributed group, one GPU per rank.

    Multi-GPU CIR: every rank sweeps its contiguous shard of the
    global sample ids (RNG keyed by global id) and casts its occlusion rays;
    the candidate rows (ordinal key, pair hashes, chain flag; 25 B each) are
    all-gathered; every rank runs the same deterministic selection
    (sbr_cir_select) over all rows, so the deduplicated candidate set is
    replicated; each rank then refines and replays only the records whose
    rows it produced (LoS records on rank 0), and the valid paths are
    gathered.  The result equals compute_paths on one GPU.
    """
    import torch.distributed as dist

    from .sharding import gather_rows, owned_records_device, shard_range
    torch = _torch()
    transmitters = list(transmitters)
    receivers = list(receivers)
    if not transmitters or not receivers:
        raise ValueError("need at least one transmitter and one receiver")
    _check_cfg(cfg, scene)
    on = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank(group) if on else 0
    world = dist.get_world_size(group) if on else 1
    tx_flat, targets, target_devices, rx_index, rx_elem = _device_plan(transmitters, receivers,
                                                                       cfg)
    acc = scene.accel
    dev = acc.device
    scene.bind_frequency(cfg.frequency)
    diagnostics = Counter()
    rejections = Counter()
    load_factor = 0.0
    parts = []
    lo, hi = shard_range(cfg.num_samples, rank, world)
    for src_idx, (ti, te, tx_pos) in enumerate(tx_flat):
        source = np.asarray(tx_pos, dtype=np.float64)
        with torch.cuda.device(dev):
            # chunk-cyclic sample shards: contiguous ones differ 2x in visibility work
            R = _sweep_rows(scene, source, targets, cfg, lo, hi,
                            shard=(rank, world) if world > 1 else None)
            n = R.n
            kept, n_dup = None, 0
            if world > 1:
                # only each shard's first occurrences travel (same selection,
                # ~100x fewer rows on config 3); the rest are duplicates
                local, kept, n_dup = _local_rows(R)
            else:
                local = {"key": R.key, "pr": R.pr[:n], "pf": R.pf[:n], "chain": R.chain[:n]}
            g, offsets = gather_rows(local, group)
            sel_counters = torch.zeros(_abi.SBR_CC_COUNT, dtype=torch.int64, device=dev)
            rec_row, nrec = _select_rows(R.params, g["key"], g["pr"], g["pf"], g["chain"],
                                         offsets[-1], R.los_vis, cfg, sel_counters, dev)
            if world > 1:
                dup = torch.tensor([n_dup], dtype=torch.int64, device=dev)
                dist.all_reduce(dup, group=group)
                sel_counters[_abi.CIR_COUNTERS.index("duplicates")] += dup[0]
            # records whose rows this rank produced (LoS on rank 0), on the device
            loc_t, n_loc = owned_records_device(rec_row[:nrec], offsets, rank, kept)
            recbuf = _materialize(R, loc_t, n_loc, cfg)
            sweep = R.counters.clone()
            if on and world > 1:
                dist.all_reduce(sweep, group=group)
        c_sweep = _counters_dict(sweep.cpu().numpy())
        c_sel = _counters_dict(sel_counters.cpu().numpy())
        if c_sweep["stack_overflow"]:
            raise RuntimeError("BVH traversal stack overflow")
        c_sel["samples_escaped"] = c_sweep["samples_escaped"]
        c_sel["samples_terminated"] = c_sweep["samples_terminated"]
        c_sel["duplicates"] += c_sweep["duplicates"]   # dropped at row emission
        gdiag = _gen_diag(c_sel, cfg)
        load_factor = max(load_factor, gdiag["hash_load_factor"])
        for k, v in gdiag.items():
            if k != "hash_load_factor":
                diagnostics[k] += v
        cand = DeviceCandidates(scene, source, targets, R.targets_t, cfg, recbuf, n_loc,
                                src_idx)
        cand.params = R.params
        part, rej = _paths_for_source(scene, cand, cfg, ti, te, transmitters[ti],
                                      target_devices, rx_index, rx_elem)
        rejections.update(rej)
        if part is not None:
            parts.append(part)
    if on and world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, (parts, dict(rejections)), group=group)
        parts = [p for ps, _ in gathered for p in ps]
        rejections = Counter()
        for _, rj in gathered:
            rejections.update(rj)
    tensors = _concat_sorted(parts, max(int(cfg.max_depth), 1))
    result = dict(diagnostics)
    result["hash_load_factor"] = load_factor
    result["refinement_rejections"] = dict(rejections)
    result["paths"] = len(tensors)
    return PathSet(tensors=tensors, transmitters=transmitters, receivers=receivers, config=cfg,
                   diagnostics=result)


def _concat_sorted(parts, L):
    keys = ("tx", "tx_el", "rx", "rx_el", "gain", "delay", "doppler", "departure", "arrival",
            "depth", "chain_hash", "sample", "kind", "obj", "prim", "wedge", "normal",
            "vertices")
    if not parts:
        empty = dict(tx=np.zeros(0, np.int64), tx_el=np.zeros(0, np.int64),
                     rx=np.zeros(0, np.int64), rx_el=np.zeros(0, np.int64),
                     gain=np.zeros(0, np.complex128), delay=np.zeros(0), doppler=np.zeros(0),
                     departure=np.zeros((0, 3)), arrival=np.zeros((0, 3)),
                     depth=np.zeros(0, np.int64), chain_hash=np.zeros(0, np.uint64),
                     sample=np.zeros(0, np.int64), kind=np.zeros((0, L), np.int8),
                     obj=np.zeros((0, L), np.int64), prim=np.zeros((0, L), np.int64),
                     wedge=np.zeros((0, L), np.int64), normal=np.zeros((0, L, 3)),
                     vertices=np.zeros((0, L + 2, 3)))
        return PathTensors(**empty)
    cat = {k: np.concatenate([p[k] for p in parts]) for k in keys}
    # paths.sort(key=(rx, rx_el, tx, tx_el, depth, chain_hash, sample))  paths.py:1505-1508
    order = np.lexsort((cat["sample"], cat["chain_hash"], cat["depth"], cat["tx_el"],
                        cat["tx"], cat["rx_el"], cat["rx"]))
    return PathTensors(**{k: v[order] for k, v in cat.items()})


def frequency_response(path_set, frequencies, transmitter=0, receiver=0):
    """H[rx antenna, tx antenna, frequency] of one link (paths.py:1519-1547), on the GPU."""
    freqs = np.atleast_1d(np.asarray(frequencies, dtype=np.float64))
    cfg = path_set.config
    tx = path_set.transmitters[transmitter]
    rx = path_set.receivers[receiver]
    T = path_set.tensors
    sel = np.nonzero((T.tx == transmitter) & (T.rx == receiver))[0]
    return channel_response(T.gain[sel], T.delay[sel], T.departure[sel], T.arrival[sel], freqs,
                            tx.array.offsets, rx.array.offsets, cfg.wavelength,
                            synthetic=cfg.synthetic_arrays, rx_el=T.rx_el[sel],
                            tx_el=T.tx_el[sel])


def channel_response(gain, delay, departure, arrival, freqs, tx_offsets, rx_offsets, wavelength,
                     synthetic=True, rx_el=None, tx_el=None, return_tensor=False):
    """`sbr_cfr` over one link's paths (host arrays in, complex128 (n_rx, n_tx, F) out).

    The body of frequency_response (paths.py:1519-1547) without the PathSet;
    ``return_tensor=True`` leaves H on the device as a float64 (.., 2) tensor.
    """
    torch = _torch()
    L_ = _native.lib()
    freqs = np.atleast_1d(np.asarray(freqs, dtype=np.float64))
    gain = np.asarray(gain, dtype=np.complex128).reshape(-1)
    n = len(gain)
    tx_offsets = np.asarray(tx_offsets, dtype=np.float64).reshape(-1, 3)
    rx_offsets = np.asarray(rx_offsets, dtype=np.float64).reshape(-1, 3)
    n_tx, n_rx = len(tx_offsets), len(rx_offsets)
    if rx_el is None:
        rx_el = np.zeros(n, np.int32)
    if tx_el is None:
        tx_el = np.zeros(n, np.int32)
    dev = torch.device("cuda", torch.cuda.current_device())
    up = lambda a, dt=np.float64: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)  # noqa
    g = np.stack([gain.real, gain.imag], axis=1) if n else np.zeros((0, 2))
    tensors = [up(g.reshape(-1, 2)), up(np.asarray(delay).reshape(-1)),
               up(np.asarray(departure).reshape(-1, 3)), up(np.asarray(arrival).reshape(-1, 3)),
               up(rx_el, np.int32), up(tx_el, np.int32), up(freqs), up(tx_offsets),
               up(rx_offsets)]
    H = torch.empty((n_rx, n_tx, len(freqs), 2), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        _native.check(L_.sbr_cfr(
            _native.ptr(tensors[0]), _native.ptr(tensors[1]), _native.ptr(tensors[2]),
            _native.ptr(tensors[3]), _native.ptr(tensors[4]), _native.ptr(tensors[5]),
            n, _native.ptr(tensors[6]), len(freqs), _native.ptr(tensors[7]), n_tx,
            _native.ptr(tensors[8]), n_rx, float(wavelength), 1 if synthetic else 0,
            _native.ptr(H), _native.stream_ptr(dev)))
    if return_tensor:
        return H
    # (.., 2) float64 is complex128 in memory: one pinned D2H copy, no host arithmetic
    hc = H.view(torch.complex128)[..., 0]
    host = torch.empty(hc.shape, dtype=torch.complex128, pin_memory=True)
    host.copy_(hc)
    return host.numpy()


def baseband_gains(path_set, transmitter=0, receiver=0):
    """Per-path gains at the carrier with the delay phase folded in (paths.py:1550-1563)."""
    cfg = path_set.config
    T = path_set.tensors
    sel = (T.tx == transmitter) & (T.rx == receiver)
    g = T.gain[sel] * np.exp(-2j * np.pi * cfg.frequency * T.delay[sel])
    return np.asarray(g, dtype=np.complex128), np.asarray(T.delay[sel])


__all__ = [
    "DedupTable", "PathBuffer", "InteractionStep", "CandidateRecord", "Rejection",
    "PathGeometry", "ValidPath", "GenerationResult", "PathTensors", "PathSet",
    "generate_candidates", "refine_candidate", "compute_paths", "compute_paths_sharded",
    "frequency_response", "channel_response",
    "baseband_gains",
]
