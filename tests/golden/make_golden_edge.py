"""Golden diffraction radio maps from the REAL reference (emtrace) -> tests/golden/edge.npz.

    python tests/golden/make_golden_edge.py [--ref /tmp/refpkg/src]

For each case of tests/edge_cases.py: collect_wedges_near_source, the edge
estimator alone (compute_radio_map_diffraction) and the full
compute_radio_map with diffraction enabled, plus diagnostics.
"""

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def main():
    ap = argparse.ArgumentParser()
    default = "/tmp/refpkg/src" if os.path.isdir("/tmp/refpkg/src") else "/root/reference/pkg/src"
    ap.add_argument("--ref", default=default)
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from emtrace.em import ArrayGeometry, make_pattern
    from emtrace.geometry import Mesh as RMesh
    from emtrace.materials import RadioMaterial as RMat
    from emtrace.paths import RadioDevice, SceneModel
    from emtrace.radiomap import (MeasurementGrid, RadioMapConfig, collect_wedges_near_source,
                                  compute_radio_map, compute_radio_map_diffraction,
                                  _scene_diameter)

    from edge_cases import EDGE_CASES, edge_geometry

    out = {}
    for name, c in EDGE_CASES.items():
        meshes, mats = edge_geometry(name)
        scene = SceneModel([RMesh(m.vertices, m.triangles, object_id=m.object_id) for m in meshes],
                           {o: RMat("m%d" % o, **md) for o, md in mats.items()})
        grid = MeasurementGrid(*c["grid"])
        cfg = RadioMapConfig(wedge_radius=c["radius"], **c["cfg"])
        kw = {}
        if c.get("pattern"):
            kw["pattern"] = make_pattern(c["pattern"][0], orientation=c["pattern"][1])
        if c.get("array"):
            kw["array"] = ArrayGeometry(np.asarray(c["array"], dtype=np.float64))
        src = np.asarray(c["src"], dtype=np.float64)
        radius = c["radius"] if c["radius"] is not None else _scene_diameter(scene)
        ids = collect_wedges_near_source(scene, src, radius)
        t0 = time.perf_counter()
        pre = np.asarray(c["precoder"], dtype=np.complex128) if c.get("precoder") else None
        ev, ed = compute_radio_map_diffraction(scene, src, grid, ids, cfg, precoder=pre, **kw)
        dev = RadioDevice(position=src, **kw)
        res = compute_radio_map(scene, [dev], grid, cfg,
                                precoders=None if pre is None else [pre])
        p = f"{name}__"
        out[p + "wedge_ids"] = np.array(ids, dtype=np.int64)
        out[p + "edge_values"] = ev
        out[p + "values"] = res.values[0]
        for k, v in ed.items():
            out[p + "edgediag__" + k] = np.array(v)
        for k, v in res.diagnostics[0].items():
            out[p + "diag__" + k] = np.array(v)
        print(name, len(ids), "wedges", f"{time.perf_counter() - t0:.1f} s", ed,
              {k: v for k, v in res.diagnostics[0].items()})
    np.savez_compressed(os.path.join(HERE, "edge.npz"), **out)


if __name__ == "__main__":
    main()
