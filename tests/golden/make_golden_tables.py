"""Golden per-triangle scene tables from the REAL reference (emtrace).

    PYTHONPATH=baseline/_ref python tests/golden/make_golden_tables.py

For the street canyon (config 2) and the golden random soup (trace.npz):
emtrace's SceneModel geometric normals (Accel.tri_normal, geometry.py:165-166)
and plane hashes (tri_plane_hash_round/floor, paths.py:449-450), keyed by
(object_id, primitive_id) because the device slot order differs from the
reference's SAH order.  Pins the device-derived tables (sbr_scene_create's
k_slot_tables) bit-exactly.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(1, ROOT)

from emtrace.geometry import Mesh  # noqa: E402
from emtrace.materials import RadioMaterial  # noqa: E402
from emtrace.paths import SceneModel  # noqa: E402


def tables(meshes):
    em = [Mesh(np.asarray(m.vertices), np.asarray(m.triangles), object_id=int(m.object_id))
          for m in meshes]
    sc = SceneModel(em, {m.object_id: RadioMaterial() for m in em})
    a = sc.accel
    order = np.lexsort((a.tri_primitive_id, a.tri_object_id))
    return dict(obj=a.tri_object_id[order], prim=a.tri_primitive_id[order],
                normal=a.tri_normal[order], hash_r=sc.tri_plane_hash_round[order],
                hash_f=sc.tri_plane_hash_floor[order])


def main():
    from paper_2504_21719_b200 import scenes
    out = {}
    for k, v in tables(scenes.street_canyon()).items():
        out["canyon_" + k] = v
    g = np.load(os.path.join(HERE, "trace.npz"))
    soup = [Mesh(g[f"verts_{i}"], g[f"tris_{i}"], object_id=int(g[f"oid_{i}"]))
            for i in range(int(g["nmesh"]))]
    for k, v in tables(soup).items():
        out["soup_" + k] = v
    np.savez_compressed(os.path.join(HERE, "tables.npz"), **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
