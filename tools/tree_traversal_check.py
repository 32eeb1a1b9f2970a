"""Run the oracle (all 1e5 samples of a 1e5-sample map: the Fibonacci
index runs pole to pole, so a prefix is not a representative sample)'s scalar traversal over OUR device-built tree (converted to the
reference's depth-first node layout) to separate tree quality from traversal effects."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import oracle
from paper_2504_21719_b200 import _native, scenes
from paper_2504_21719_b200.geometry import build_scene_accel
from paper_2504_21719_b200.radiomap import MeasurementGrid, RadioMapConfig
from paper_2504_21719_b200.sampling import Interaction

L = oracle.lib()
L.orc_visit_stats.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]


def convert(acc):
    boxes, codes = acc.bvh_nodes()
    bmin, bmax, right, start, count = [], [], [], [], []

    def emit(lo, hi):
        bmin.append(lo.astype(np.float64)); bmax.append(hi.astype(np.float64))
        right.append(-1); start.append(-1); count.append(0)
        return len(bmin) - 1

    def rec(node, lo, hi):
        me = emit(lo, hi)
        for c in (0, 1):
            code = int(codes[node, c])
            clo, chi = boxes[node, c, 0], boxes[node, c, 1]
            if c == 1:
                right[me] = len(bmin)
            if code >= 0:
                rec(code, clo, chi)
            else:
                k = emit(clo, chi)
                start[k] = (~code) >> 2
                count[k] = ((~code) & 3) + 1
        return me

    sys.setrecursionlimit(100000)
    rec(0, boxes[0, :, 0].min(0), boxes[0, :, 1].max(0))
    return (np.ascontiguousarray(bmin), np.ascontiguousarray(bmax),
            np.array(right, np.int32), np.array(start, np.int32), np.array(count, np.int32))


CITY = "--city" in sys.argv
meshes = scenes.city() if CITY else scenes.street_canyon()
mats = scenes.uniform_materials(meshes, scenes.concrete(scattering=0.3))
TX = (0.0, 0.0, 30.0) if CITY else (0.0, 5.0, 20.0)
grid = MeasurementGrid((0, 0, 1.5), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (200, 200))
cfg = RadioMapConfig(num_samples=100_000, max_depth=5, seed=0,
                     enabled=frozenset({Interaction.REFLECTION, Interaction.SCATTERING}))
n = np.zeros(1, np.uint64); t = np.zeros(1, np.uint64)
for label, builder in (("sah(reference)", None), ("lbvh", 0), ("ploc", 1)):
    sc = oracle.OracleScene(meshes, mats)
    keep = None
    if builder is not None:
        _native.check(_native.lib().sbr_set_bvh_builder(builder))
        acc = build_scene_accel(meshes)
        keep = convert(acc)
        s = sc._s
        s.bmin, s.bmax, s.right, s.start, s.count = [a.ctypes.data for a in keep]
        s.nnodes = len(keep[0])
        # triangles / attributes in OUR slot order
        p = acc.perm
        sc.tri_v0, sc.tri_v1, sc.tri_v2 = acc.tri_v0, acc.tri_v1, acc.tri_v2
        sc.tri_object_id = np.ascontiguousarray(acc.tri_object_id)
        sc.tri_primitive_id = np.ascontiguousarray(acc.tri_primitive_id)
        sc.tri_normal = np.ascontiguousarray(acc.tri_normal)
        sc.tri_material_row = np.ascontiguousarray(
            np.searchsorted(sc._object_ids, sc.tri_object_id).astype(np.int32))
        s.v0, s.v1, s.v2 = sc.tri_v0.ctypes.data, sc.tri_v1.ctypes.data, sc.tri_v2.ctypes.data
        s.obj, s.prim = sc.tri_object_id.ctypes.data, sc.tri_primitive_id.ctypes.data
        s.normal, s.matrow = sc.tri_normal.ctypes.data, sc.tri_material_row.ctypes.data
    L.orc_visit_stats(n.ctypes.data, t.ctypes.data, 1)
    v, d = sc.radiomap(TX, grid, cfg, sample_range=(0, 100000), include_direct=False)
    L.orc_visit_stats(n.ctypes.data, t.ctypes.data, 1)
    print(label, "scalar near-first traversal: nodes/rb %.2f tris/rb %.2f  (rb %d, deposits %d)"
          % (n[0] / d["ray_bounces"], t[0] / d["ray_bounces"], d["ray_bounces"], d["deposits"]))
