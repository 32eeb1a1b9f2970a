"""Chain scenes x = base^k: BVH depth (PLOC only) and map parity vs the oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from test_gpu_edge_inputs import CONC, R  # noqa: E402
from paper_2504_21719_b200 import (MeasurementGrid, RadioMapConfig, SceneModel,  # noqa: E402
                                   _native, compute_radio_map_sbr)
from paper_2504_21719_b200.geometry import Mesh  # noqa: E402


def chain(n, base):
    verts, tris = [], []
    for k in range(n):
        x = float(base ** k)
        b = len(verts)
        verts += [(x, -1.0, -1.0), (x, 1.0, -1.0), (x, 1.0, 1.0), (x, -1.0, 1.0)]
        tris += [(b, b + 1, b + 2), (b, b + 2, b + 3)]
    return [Mesh(np.array(verts), np.array(tris), object_id=0)]


for n, base in [(int(a), float(b)) for a, b in (x.split(":") for x in (sys.argv[1:] or ["110:2"]))]:
    meshes = chain(n, base)
    L = _native.lib()
    L.sbr_set_bvh_builder(2)
    sc = SceneModel(meshes, {0: CONC})
    acc = sc.accel
    L.sbr_set_bvh_builder(1)
    nodes = np.zeros((int(L.sbr_scene_num_nodes(acc.handle)), 16), np.int32)
    _native.check(L.sbr_scene_copy_nodes(acc.handle, nodes.ctypes.data))
    depth, todo = {0: 1}, [0]
    while todo:
        i = todo.pop()
        for c in nodes[i, 12:14]:
            if c >= 0:
                depth[int(c)] = depth[i] + 1
                todo.append(int(c))
    grid = MeasurementGrid((2.0, 0.0, 0.05), (1, 0, 0), (0, 1, 0), (0.25, 0.25), (32, 8))
    cfg = RadioMapConfig(num_samples=200_000, max_depth=4, enabled=R, seed=5)
    src = (1.5 if base == 2.0 else 0.5 * (base ** 5 + base ** 6), 0.3, 0.2)
    try:
        vals, diag = compute_radio_map_sbr(sc, src, grid, cfg, include_direct=False)
        want, wdiag = oracle.OracleScene(meshes, {0: CONC}).radiomap(np.array(src), grid, cfg,
                                                                     include_direct=False)
        same = all(diag.get(k, 0) == wdiag.get(k, 0) for k in ("deposits", "escaped", "ray_bounces"))
        rel = float(np.max(np.abs(vals - want)) / max(np.max(np.abs(want)), 1e-300))
        print(n, base, "depth", max(depth.values()), "same", same, "rel", rel,
              {k: (diag.get(k, 0), wdiag.get(k, 0)) for k in ("deposits", "escaped", "ray_bounces")}, flush=True)
    except Exception as e:  # noqa: BLE001
        print(n, base, "depth", max(depth.values()), "error", repr(e)[:200], flush=True)
