"""Golden scene-file / OBJ / writer outcomes from the REAL reference (emtrace.sceneio).

    python tests/golden/make_golden_sceneio.py [--ref /tmp/refpkg/src]

Parses every case of tests/sceneio_cases.py with the reference and records the
description (or the exception class + message), loads the OBJ cases (arrays +
warnings) and records the writers' exact output text.  -> tests/golden/sceneio.json
"""

import argparse
import json
import os
import sys
import tempfile
import types
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/tmp/refpkg/src" if os.path.isdir("/tmp/refpkg/src")
                    else "/root/reference/pkg/src")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from emtrace import sceneio
    from emtrace.radiomap import MeasurementGrid
    import sceneio_cases as C
    from sceneio_cases import as_objects, describe, fake_paths

    out = {"good": describe(sceneio.parse_scene_text(C.GOOD)),
           "minimal": describe(sceneio.parse_scene_text(C.MINIMAL)), "bad": {}, "obj": {},
           "obj_bad": {}}
    for k, text in C.BAD.items():
        try:
            sceneio.parse_scene_text(text)
            out["bad"][k] = None
        except Exception as e:  # noqa: BLE001
            out["bad"][k] = [type(e).__name__, str(e), getattr(e, "line", None),
                             getattr(e, "field", None)]
    with tempfile.TemporaryDirectory() as td:
        for k, text in {**C.OBJ, **C.OBJ_BAD}.items():
            p = os.path.join(td, k + ".obj")
            open(p, "w").write(text)
            with warnings.catch_warnings(record=True) as caught:
                warnings.simplefilter("always")
                try:
                    m = sceneio.load_mesh_obj(p, object_id=3, material_ref="m")
                    res = dict(vertices=m.vertices.tolist(), triangles=m.triangles.tolist(),
                               warnings=[[type(w.message).__name__, str(w.message)]
                                         for w in caught])
                except Exception as e:  # noqa: BLE001
                    res = [type(e).__name__, str(e)]
            out["obj" if k in C.OBJ else "obj_bad"][k] = res
        # writers
        recs = fake_paths()
        for r in recs:
            r["gain"] = [r["gain"].real, r["gain"].imag]
        out["paths_input"] = recs
        res = as_objects(recs)
        for fmt in ("csv", "json"):
            p = os.path.join(td, "paths." + fmt)
            sceneio.write_paths(res, p, fmt=fmt)
            out["paths_" + fmt] = open(p).read()
        out["paths_read"] = sceneio.read_paths_csv(os.path.join(td, "paths.csv"))
        grid = MeasurementGrid((0, 0, 1.5), (1, 0, 0), (0, 1, 0), (1.0, 2.0), (4, 3))
        vals = np.random.default_rng(5).uniform(1e-14, 1e-6, size=(3, 4))
        vals[0, 0] = 0.0
        out["map_values"] = vals.tolist()
        for fmt in ("csv", "pgm"):
            p = os.path.join(td, "map." + fmt)
            sceneio.write_radio_map(grid, vals, p, fmt=fmt)
            out["map_" + fmt] = open(p).read()
        mesh = sceneio.load_mesh_obj(os.path.join(td, "poly.obj"))
        sceneio.write_mesh_obj(mesh, os.path.join(td, "w.obj"))
        out["obj_written"] = open(os.path.join(td, "w.obj")).read()
    with open(os.path.join(HERE, "sceneio.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print("written sceneio.json")


if __name__ == "__main__":
    main()
