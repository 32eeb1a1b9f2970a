"""Triangle-mesh world model on the GPU: LBVH build and batched ray queries.

Drop-in for emtrace/geometry.py:31-237.  `Accel` keeps the reference's
attribute names (num_triangles, bounds, perm, tri_v0/1/2, tri_object_id,
tri_primitive_id, tri_mesh_index, tri_normal) but the slot order is the
device LBVH's Morton order instead of the host SAH order.  The BVH lives in
HBM (csrc/sbr_scene.cu); trace_batch / occluded_batch run the sm_100a
traversal kernels (csrc/sbr_trace.cu) and accept numpy arrays (copied
host<->device) or CUDA tensors (zero-copy).

Closest-hit semantics are the reference's exactly (_core.pyx:115-195): the
hit is the minimum over triangles of (t, object_id, primitive_id) with
t_min < t < t_max, computed with the same float64 watertight test, so the
result does not depend on the BVH shape.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import EmptyScene

EPS_RAY = 1e-4
EPS_AREA = 1e-12
EPS_COPLANAR = 1e-6


@dataclass(eq=False)
class Mesh:
    """One object: vertex table plus triangle index triples (geometry.py:31-71)."""

    vertices: np.ndarray
    triangles: np.ndarray
    object_id: int
    material_ref: str = ""

    def __post_init__(self):
        self.vertices = np.ascontiguousarray(self.vertices, dtype=np.float64)
        self.triangles = np.ascontiguousarray(self.triangles, dtype=np.int64)
        if self.vertices.ndim != 2 or self.vertices.shape[1] != 3:
            raise ValueError("vertices must be (n, 3)")
        if self.triangles.ndim != 2 or self.triangles.shape[1] != 3:
            raise ValueError("triangles must be (m, 3)")
        if len(self.triangles) and (self.triangles.min() < 0
                                    or self.triangles.max() >= len(self.vertices)):
            raise ValueError("triangle index out of range")
        areas = self.triangle_areas()
        if np.any(areas <= EPS_AREA):
            bad = int(np.argmax(areas <= EPS_AREA))
            raise ValueError(f"degenerate triangle {bad} (area {areas[bad]:.3e})")

    def triangle_corners(self):
        v, t = self.vertices, self.triangles
        return v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]

    def triangle_areas(self):
        a, b, c = self.triangle_corners()
        return 0.5 * np.linalg.norm(np.cross(b - a, c - a), axis=1)

    def triangle_normals(self):
        a, b, c = self.triangle_corners()
        n = np.cross(b - a, c - a)
        return n / np.linalg.norm(n, axis=1, keepdims=True)


@dataclass(frozen=True)
class Ray:
    origin: np.ndarray
    direction: np.ndarray
    max_t: float = np.inf

    def __post_init__(self):
        object.__setattr__(self, "origin", np.asarray(self.origin, dtype=np.float64))
        object.__setattr__(self, "direction",
                           np.asarray(self.direction, dtype=np.float64))
        norm = np.linalg.norm(self.direction)
        if abs(norm - 1.0) > 1e-9:
            raise ValueError(f"direction norm {norm} != 1")


@dataclass(frozen=True)
class Hit:
    t: float
    point: np.ndarray
    normal: np.ndarray
    object_id: int
    primitive_id: int
    bary: tuple
    tri_index: int = -1


def _to_device(x, dev, shape_last=None):
    import torch
    if isinstance(x, torch.Tensor):
        t = x.to(device=dev, dtype=torch.float64)
    else:
        t = torch.from_numpy(np.array(x, dtype=np.float64, copy=True)).to(dev)
    return t.contiguous()


class Accel:
    """Immutable LBVH over the flattened triangles of several meshes, in HBM."""

    def __init__(self, meshes, device=None):
        import torch
        tri_count = sum(len(m.triangles) for m in meshes)
        if tri_count == 0:
            raise EmptyScene("no triangles")
        self.meshes = list(meshes)
        v0s, v1s, v2s, objs, prims, mesh_idx = [], [], [], [], [], []
        for i, m in enumerate(self.meshes):
            a, b, c = m.triangle_corners()
            v0s.append(a)
            v1s.append(b)
            v2s.append(c)
            objs.append(np.full(len(a), m.object_id, dtype=np.int64))
            prims.append(np.arange(len(a), dtype=np.int64))
            mesh_idx.append(np.full(len(a), i, dtype=np.int64))
        v0 = np.ascontiguousarray(np.concatenate(v0s))
        v1 = np.ascontiguousarray(np.concatenate(v1s))
        v2 = np.ascontiguousarray(np.concatenate(v2s))

        L = _native.lib()
        self.device = _native.device_of(device)
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _native.check(L.sbr_scene_create(
                v0.ctypes.data_as(ctypes.c_void_p), v1.ctypes.data_as(ctypes.c_void_p),
                v2.ctypes.data_as(ctypes.c_void_p), len(v0), self.device.index,
                _native.stream_ptr(self.device), ctypes.byref(handle)))
        self._handle = handle
        self._lib = L
        perm = np.empty(len(v0), dtype=np.int64)
        _native.check(L.sbr_scene_permutation(handle, perm.ctypes.data_as(ctypes.c_void_p)))
        self.perm = perm
        self.num_nodes = int(L.sbr_scene_num_nodes(handle))
        self._input = (v0, v1, v2)            # input-order corners (wedge extraction)
        sizes = np.array([len(m.triangles) for m in self.meshes], np.int64)
        oid = np.array([m.object_id for m in self.meshes], np.int64)
        obj_in, prim_in = np.concatenate(objs), np.concatenate(prims)
        self._obj_in, self._prim_in = obj_in, prim_in
        self.tri_object_id = obj_in[perm]
        self.tri_primitive_id = prim_in[perm]
        self.tri_mesh_index = np.concatenate(mesh_idx)[perm]
        self._tables = None   # device-derived normals / plane hashes, copied on first use
        self._corners = None  # slot-order host corners, on first use
        lo = np.minimum(np.minimum(v0, v1), v2).min(axis=0)
        hi = np.maximum(np.maximum(v0, v1), v2).max(axis=0)
        self.bounds = (lo - 1e-12 * (1.0 + np.abs(lo)), hi + 1e-12 * (1.0 + np.abs(hi)))
        # closest-hit tie rule: smaller (object_id, primitive_id) wins
        if len(np.unique(oid)) == len(oid):
            # unique object ids: rank = start of the mesh in object-id order + primitive
            start = np.empty(len(oid), np.int64)
            by_id = np.argsort(oid, kind="stable")
            start[by_id] = np.concatenate([[0], np.cumsum(sizes[by_id])[:-1]])
            rank = (np.repeat(start, sizes) + prim_in)[perm].astype(np.int32)
        else:
            order = np.lexsort((self.tri_primitive_id, self.tri_object_id))
            rank = np.empty(len(order), dtype=np.int32)
            rank[order] = np.arange(len(order), dtype=np.int32)
        self.tri_tie_rank = rank
        self.set_attributes(tie_rank=rank)

    def _device_tables(self):
        """Host copies of the per-slot normals and plane hashes that
        sbr_scene_create derived on the device (geometry.py:165-166,
        paths.py:156-171 arithmetic, bit-identical to the numpy expressions)."""
        if self._tables is None:
            n = self.num_triangles
            nrm = np.empty((n, 3), dtype=np.float64)
            hr = np.empty(n, dtype=np.uint64)
            hf = np.empty(n, dtype=np.uint64)
            _native.check(self._lib.sbr_scene_copy_tables(
                self._handle, nrm.ctypes.data_as(ctypes.c_void_p),
                hr.ctypes.data_as(ctypes.c_void_p), hf.ctypes.data_as(ctypes.c_void_p)))
            self._tables = (nrm, hr, hf)
        return self._tables

    def _slot_corners(self):
        if self._corners is None:
            v0, v1, v2 = self._input
            p = self.perm
            self._corners = tuple(np.ascontiguousarray(v[p]) for v in (v0, v1, v2))
        return self._corners

    @property
    def tri_v0(self):
        return self._slot_corners()[0]

    @property
    def tri_v1(self):
        return self._slot_corners()[1]

    @property
    def tri_v2(self):
        return self._slot_corners()[2]

    @property
    def tri_normal(self):
        """(T, 3) geometric normals normalize((v1 - v0) x (v2 - v0)) per slot."""
        return self._device_tables()[0]

    @property
    def tri_plane_hashes(self):
        """(round, floor) plane hashes per slot (paths.py:449-450)."""
        _, hr, hf = self._device_tables()
        return hr, hf

    # -- device tables -----------------------------------------------------
    def set_attributes(self, tie_rank=None, normals=None, matrow=None,
                       hash_r=None, hash_f=None):
        def p(a, dt):
            if a is None:
                return None, ctypes.c_void_p(0)
            a = np.ascontiguousarray(a, dtype=dt)
            return a, a.ctypes.data_as(ctypes.c_void_p)
        keep = [p(tie_rank, np.int32), p(normals, np.float64), p(matrow, np.int32),
                p(hash_r, np.uint64), p(hash_f, np.uint64)]
        _native.check(self._lib.sbr_scene_set_attributes(
            self._handle, *[k[1] for k in keep]))

    def set_materials(self, rows_abi, count):
        _native.check(self._lib.sbr_scene_set_materials(self._handle, rows_abi, count))

    def check(self):
        with _cuda_device(self.device):
            _native.check(self._lib.sbr_scene_check(self._handle,
                                                    _native.stream_ptr(self.device)))

    @property
    def handle(self):
        return self._handle

    def bvh_nodes(self):
        """Host copy of the device BVH2: (boxes (M, 2, 2, 3) [child, lo/hi, xyz], codes (M, 2))."""
        raw = np.empty((self.num_nodes, 16), dtype=np.float32)
        _native.check(self._lib.sbr_scene_copy_nodes(self._handle,
                                                     raw.ctypes.data_as(ctypes.c_void_p)))
        a, b, c = raw[:, 0:4], raw[:, 4:8], raw[:, 8:12]
        codes = raw[:, 12:14].copy().view(np.int32)
        boxes = np.empty((self.num_nodes, 2, 2, 3), dtype=np.float32)
        boxes[:, 0, 0] = np.stack([a[:, 0], a[:, 2], c[:, 0]], 1)
        boxes[:, 0, 1] = np.stack([a[:, 1], a[:, 3], c[:, 1]], 1)
        boxes[:, 1, 0] = np.stack([b[:, 0], b[:, 2], c[:, 2]], 1)
        boxes[:, 1, 1] = np.stack([b[:, 1], b[:, 3], c[:, 3]], 1)
        return boxes, codes

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                self._lib.sbr_scene_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._handle = None

    @property
    def num_triangles(self):
        return len(self.tri_v0)

    # -- queries -----------------------------------------------------------
    def trace_batch(self, origins, directions, t_min=EPS_RAY, t_max=np.inf):
        """Closest hit per ray: (t, tri, u, v), tri = -1 on a miss (geometry.py:178-185).

        numpy in -> numpy out (host copies inside); CUDA tensors in -> tensors out.
        """
        import torch
        host = not isinstance(origins, torch.Tensor)
        dev = self.device
        o = _to_device(origins, dev).reshape(-1, 3)
        d = _to_device(directions, dev).reshape(-1, 3)
        n = o.shape[0]
        if isinstance(t_max, torch.Tensor):
            tm = t_max.to(device=dev, dtype=torch.float64).expand(n).contiguous()
        else:
            tm = torch.from_numpy(np.broadcast_to(np.asarray(t_max, dtype=np.float64),
                                                  (n,)).copy()).to(dev)
        t = torch.empty(n, dtype=torch.float64, device=dev)
        tri = torch.empty(n, dtype=torch.int64, device=dev)
        u = torch.empty(n, dtype=torch.float64, device=dev)
        v = torch.empty(n, dtype=torch.float64, device=dev)
        with _cuda_device(dev):
            _native.check(self._lib.sbr_trace_closest(
                self._handle, _native.ptr(o), _native.ptr(d), float(t_min),
                _native.ptr(tm), n, _native.ptr(t), _native.ptr(tri), _native.ptr(u),
                _native.ptr(v), _native.stream_ptr(dev)))
        self.check()
        if host:
            return t.cpu().numpy(), tri.cpu().numpy(), u.cpu().numpy(), v.cpu().numpy()
        return t, tri, u, v

    def any_hit_batch(self, origins, directions, t_min, t_max):
        """Raw trace_any (_core.pyx:198-253)."""
        import torch
        host = not isinstance(origins, torch.Tensor)
        dev = self.device
        o = _to_device(origins, dev).reshape(-1, 3)
        d = _to_device(directions, dev).reshape(-1, 3)
        n = o.shape[0]
        tm = _to_device(np.broadcast_to(np.asarray(t_max, dtype=np.float64), (n,))
                        if not isinstance(t_max, torch.Tensor) else t_max, dev)
        out = torch.empty(n, dtype=torch.uint8, device=dev)
        with _cuda_device(dev):
            _native.check(self._lib.sbr_trace_any(
                self._handle, _native.ptr(o), _native.ptr(d), float(t_min), _native.ptr(tm),
                n, _native.ptr(out), _native.stream_ptr(dev)))
        self.check()
        out = out.bool()
        return out.cpu().numpy() if host else out

    def occluded_batch(self, a, b, eps=EPS_RAY):
        """Occlusion of open segments (a, b), endpoints offset by eps (geometry.py:187-201)."""
        import torch
        host = not isinstance(a, torch.Tensor)
        dev = self.device
        if host:
            a = np.atleast_2d(a)
            b = np.atleast_2d(b)
        at = _to_device(a, dev).reshape(-1, 3)
        bt = _to_device(b, dev).reshape(-1, 3)
        n = at.shape[0]
        out = torch.empty(n, dtype=torch.uint8, device=dev)
        with _cuda_device(dev):
            _native.check(self._lib.sbr_occluded(
                self._handle, _native.ptr(at), _native.ptr(bt), float(eps), n,
                _native.ptr(out), _native.stream_ptr(dev)))
        self.check()
        out = out.bool()
        return out.cpu().numpy() if host else out


class _cuda_device:
    def __init__(self, dev):
        import torch
        self._ctx = torch.cuda.device(dev)

    def __enter__(self):
        return self._ctx.__enter__()

    def __exit__(self, *exc):
        return self._ctx.__exit__(*exc)


def build_scene_accel(meshes, device=None):
    """Build the shared device BVH for a list of meshes. Raises EmptyScene if empty."""
    return Accel(meshes, device=device)


def hit_from_trace(accel, origin, direction, t, tri, u, v):
    point = origin + t * direction
    normal = accel.tri_normal[tri]
    if float(normal @ direction) > 0.0:
        normal = -normal
    return Hit(t=t, point=point, normal=normal,
               object_id=int(accel.tri_object_id[tri]),
               primitive_id=int(accel.tri_primitive_id[tri]),
               bary=(u, v), tri_index=tri)


def intersect_closest(accel, ray):
    """Closest hit with t in (EPS_RAY, ray.max_t) or None (geometry.py:204-222)."""
    t, tri, u, v = accel.trace_batch(ray.origin[None, :], ray.direction[None, :],
                                     EPS_RAY, ray.max_t)
    if tri[0] < 0:
        return None
    return hit_from_trace(accel, ray.origin, ray.direction, float(t[0]), int(tri[0]),
                          float(u[0]), float(v[0]))


def is_occluded(accel, a, b):
    """True iff geometry blocks the open segment between a and b."""
    return bool(accel.occluded_batch(np.asarray(a)[None, :], np.asarray(b)[None, :])[0])
