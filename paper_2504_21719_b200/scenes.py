"""Deterministic procedural scenes for the benchmark configs.

All generators return lists of `Mesh` (one object id per building / wall),
plus helpers for the test scenes of the reference suite.  Triangles are
wound so geometric normals point out of the material (geometry.py:33-37).

  * `config1_scene`  ground quad (half 50) + one 2x40x15 m box wall
  * `street_canyon`  200x200 m ground (20x20 quads) + 10x10 buildings on a
                     20 m pitch, 12x12 m footprints, heights U(10,40) from
                     default_rng(seed), faces split 3x3 -> 11,600 triangles
  * `city`           1000x1000 m ground (40x40 quads) + 40x40 buildings on a
                     25 m pitch, 15x15 m footprints, heights U(10,60),
                     faces split 5x5 -> 483,200 triangles
"""

import numpy as np

from .geometry import Mesh
from .materials import RadioMaterial, ScatteringPattern

# Outward-wound unit box faces over corners (lo), (hi_x), (hi_xy), (hi_y),
# then the same four lifted to hi_z (reference tests/conftest.py layout).
_BOX_FACES = np.array([
    [0, 2, 1], [0, 3, 2],
    [4, 5, 6], [4, 6, 7],
    [0, 1, 5], [0, 5, 4],
    [2, 3, 7], [2, 7, 6],
    [1, 2, 6], [1, 6, 5],
    [3, 0, 4], [3, 4, 7],
], dtype=np.int64)


def box_mesh(lo, hi, object_id=0, inward=False):
    l = np.asarray(lo, dtype=np.float64)
    h = np.asarray(hi, dtype=np.float64)
    v = np.array([
        [l[0], l[1], l[2]], [h[0], l[1], l[2]], [h[0], h[1], l[2]], [l[0], h[1], l[2]],
        [l[0], l[1], h[2]], [h[0], l[1], h[2]], [h[0], h[1], h[2]], [l[0], h[1], h[2]],
    ])
    f = _BOX_FACES[:, ::-1] if inward else _BOX_FACES
    return Mesh(v, f.copy(), object_id=object_id)


def quad_mesh(half=1.0, z=0.0, object_id=0):
    v = np.array([[-half, -half, z], [half, -half, z], [half, half, z], [-half, half, z]])
    f = np.array([[0, 1, 2], [0, 2, 3]], dtype=np.int64)
    return Mesh(v, f, object_id=object_id)


def _grid_quad(origin, e1, e2, n1, n2):
    """Vertices/triangles of a parallelogram origin + a e1 + b e2 split n1 x n2.

    The normal of every triangle is normalize(e1 x e2).
    """
    o, e1, e2 = (np.asarray(x, dtype=np.float64) for x in (origin, e1, e2))
    a = np.arange(n1 + 1) / n1
    b = np.arange(n2 + 1) / n2
    verts = (o[None, None, :] + a[:, None, None] * e1[None, None, :]
             + b[None, :, None] * e2[None, None, :]).reshape(-1, 3)
    idx = lambda i, j: i * (n2 + 1) + j  # noqa: E731
    tris = []
    for i in range(n1):
        for j in range(n2):
            p00, p10, p11, p01 = idx(i, j), idx(i + 1, j), idx(i + 1, j + 1), idx(i, j + 1)
            tris.append([p00, p10, p11])
            tris.append([p00, p11, p01])
    return verts, np.asarray(tris, dtype=np.int64)


def _merge(parts):
    verts, tris, off = [], [], 0
    for v, t in parts:
        verts.append(v)
        tris.append(t + off)
        off += len(v)
    return np.concatenate(verts), np.concatenate(tris)


def subdivided_box(lo, hi, k, object_id):
    """Closed box with each face split k x k quads, normals outward."""
    x0, y0, z0 = (float(c) for c in lo)
    x1, y1, z1 = (float(c) for c in hi)
    dx, dy, dz = x1 - x0, y1 - y0, z1 - z0
    faces = [
        ((x0, y0, z0), (0, dy, 0), (dx, 0, 0)),   # bottom, normal -z
        ((x0, y0, z1), (dx, 0, 0), (0, dy, 0)),   # top, +z
        ((x0, y0, z0), (dx, 0, 0), (0, 0, dz)),   # front, -y
        ((x0, y1, z0), (0, 0, dz), (dx, 0, 0)),   # back, +y
        ((x1, y0, z0), (0, dy, 0), (0, 0, dz)),   # right, +x
        ((x0, y0, z0), (0, 0, dz), (0, dy, 0)),   # left, -x
    ]
    v, t = _merge([_grid_quad(o, a, b, k, k) for o, a, b in faces])
    return Mesh(v, t, object_id=object_id)


def ground(half, n, object_id=0, z=0.0):
    v, t = _grid_quad((-half, -half, z), (2 * half, 0, 0), (0, 2 * half, 0), n, n)
    return Mesh(v, t, object_id=object_id)


def street_canyon(seed=1):
    """~11.6k-triangle street canyon (config 2)."""
    rng = np.random.default_rng(seed)
    meshes = [ground(100.0, 20, object_id=0)]
    oid = 1
    for bx in range(10):
        for by in range(10):
            h = rng.uniform(10.0, 40.0)
            cx = -100.0 + 20.0 * bx + 10.0
            cy = -100.0 + 20.0 * by + 10.0
            meshes.append(subdivided_box((cx - 6.0, cy - 6.0, 0.0), (cx + 6.0, cy + 6.0, h),
                                         3, oid))
            oid += 1
    return meshes


def city(seed=1, n=40, pitch=25.0, footprint=15.0, k=5, hmin=10.0, hmax=60.0):
    """~483k-triangle procedural city (configs 3-5)."""
    rng = np.random.default_rng(seed)
    half = 0.5 * n * pitch
    meshes = [ground(half, n, object_id=0)]
    oid = 1
    f2 = 0.5 * footprint
    for bx in range(n):
        for by in range(n):
            h = rng.uniform(hmin, hmax)
            cx = -half + pitch * bx + 0.5 * pitch
            cy = -half + pitch * by + 0.5 * pitch
            meshes.append(subdivided_box((cx - f2, cy - f2, 0.0), (cx + f2, cy + f2, h), k, oid))
            oid += 1
    return meshes


def city_receivers(count=1024, seed=2, n=40, pitch=25.0, footprint=15.0, z=1.5):
    """Receivers uniform over the street area (rejected inside footprints)."""
    rng = np.random.default_rng(seed)
    half = 0.5 * n * pitch
    f2 = 0.5 * footprint
    out = []
    while len(out) < count:
        p = rng.uniform(-half + 1.0, half - 1.0, size=2)
        cx = (np.floor((p + half) / pitch) + 0.5) * pitch - half
        if np.all(np.abs(p - cx) < f2 + 0.5):
            continue
        out.append([p[0], p[1], z])
    return np.asarray(out)


def config1_scene():
    """Ground plane + one box wall (config 1)."""
    return [quad_mesh(half=50.0, z=0.0, object_id=0),
            box_mesh([10.0, -20.0, 0.0], [12.0, 20.0, 15.0], object_id=1)]


def box_room_walls(lo=(-3.0, -4.0, 0.0), hi=(3.0, 4.0, 3.0)):
    """Closed room, each wall its own object 1..6 (reference test_radiomap.py:40-66)."""
    xl, yl, zl = lo
    xh, yh, zh = hi

    def wall(a, b, c, d, oid):
        return Mesh(np.array([a, b, c, d], dtype=np.float64),
                    np.array([[0, 1, 2], [0, 2, 3]], dtype=np.int64), object_id=oid)

    return [
        wall([xl, yl, zl], [xh, yl, zl], [xh, yh, zl], [xl, yh, zl], 1),
        wall([xl, yl, zh], [xh, yl, zh], [xh, yh, zh], [xl, yh, zh], 2),
        wall([xl, yl, zl], [xh, yl, zl], [xh, yl, zh], [xl, yl, zh], 3),
        wall([xl, yh, zl], [xh, yh, zl], [xh, yh, zh], [xl, yh, zh], 4),
        wall([xl, yl, zl], [xl, yh, zl], [xl, yh, zh], [xl, yl, zh], 5),
        wall([xh, yl, zl], [xh, yh, zl], [xh, yh, zh], [xh, yl, zh], 6),
    ]


def concrete(scattering=0.0, **kw):
    """The benchmark concrete: RadioMaterial(eps_r=5.24, sigma=0.0462, thickness=0.1)."""
    return RadioMaterial("concrete", eps_r=5.24, sigma=0.0462, thickness=0.1,
                         scattering=scattering, pattern=kw.pop("pattern", ScatteringPattern()),
                         **kw)


def uniform_materials(meshes, material):
    return {m.object_id: material for m in meshes}
