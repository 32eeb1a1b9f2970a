"""Scene files, OBJ meshes and writers vs the real reference (emtrace.sceneio).

Golden outcomes: tests/golden/sceneio.json (tests/golden/make_golden_sceneio.py).
CPU-only except the end-to-end load_scene / write_scene round trip, which
builds a SceneModel on the GPU.
"""

import json
import os
import warnings

import numpy as np
import pytest

import sceneio_cases as C
from sceneio_cases import as_objects, describe
from paper_2504_21719_b200 import sceneio
from paper_2504_21719_b200.radiomap import MeasurementGrid

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "sceneio.json")))


def _norm(x):
    return json.loads(json.dumps(x))


def test_parse_good_scene_matches_reference():
    assert _norm(describe(sceneio.parse_scene_text(C.GOOD))) == GOLD["good"]
    assert _norm(describe(sceneio.parse_scene_text(C.MINIMAL))) == GOLD["minimal"]


@pytest.mark.parametrize("name", sorted(C.BAD))
def test_parse_errors_match_reference(name):
    want = GOLD["bad"][name]
    with pytest.raises(Exception) as exc:
        sceneio.parse_scene_text(C.BAD[name])
    e = exc.value
    assert [type(e).__name__, str(e), getattr(e, "line", None), getattr(e, "field", None)] == want


@pytest.mark.parametrize("name", sorted({**C.OBJ, **C.OBJ_BAD}))
def test_obj_loading_matches_reference(tmp_path, name):
    text = {**C.OBJ, **C.OBJ_BAD}[name]
    p = tmp_path / f"{name}.obj"
    p.write_text(text)
    with warnings.catch_warnings(record=True) as caught:
        warnings.simplefilter("always")
        try:
            m = sceneio.load_mesh_obj(p, object_id=3, material_ref="m")
            got = dict(vertices=m.vertices.tolist(), triangles=m.triangles.tolist(),
                       warnings=[[type(w.message).__name__, str(w.message)] for w in caught])
            assert m.object_id == 3 and m.material_ref == "m"
        except Exception as e:  # noqa: BLE001
            got = [type(e).__name__, str(e)]
    want = GOLD["obj"].get(name, GOLD["obj_bad"].get(name))
    assert _norm(got) == want


def test_writers_match_reference(tmp_path):
    res = as_objects(GOLD["paths_input"])
    for fmt in ("csv", "json"):
        p = tmp_path / f"paths.{fmt}"
        sceneio.write_paths(res, p, fmt=fmt)
        assert p.read_text() == GOLD[f"paths_{fmt}"]
    assert _norm(sceneio.read_paths_csv(tmp_path / "paths.csv")) == GOLD["paths_read"]
    grid = MeasurementGrid((0, 0, 1.5), (1, 0, 0), (0, 1, 0), (1.0, 2.0), (4, 3))
    vals = np.array(GOLD["map_values"])
    for fmt in ("csv", "pgm"):
        p = tmp_path / f"map.{fmt}"
        sceneio.write_radio_map(grid, vals, p, fmt=fmt)
        assert p.read_text() == GOLD[f"map_{fmt}"]
    assert np.array_equal(sceneio.read_radio_map_csv(tmp_path / "map.csv"), vals)
    with pytest.raises(ValueError):
        sceneio.write_radio_map(grid, vals[:2], tmp_path / "x.csv")
    with pytest.raises(ValueError):
        sceneio.write_paths(res, tmp_path / "x.txt", fmt="txt")
    (tmp_path / "poly.obj").write_text(C.OBJ["poly"])
    sceneio.write_mesh_obj(sceneio.load_mesh_obj(tmp_path / "poly.obj"), tmp_path / "w.obj")
    assert (tmp_path / "w.obj").read_text() == GOLD["obj_written"]


def _scene_dir(tmp_path):
    (tmp_path / "sub dir").mkdir()
    quad = "v -10 -10 0\nv 10 -10 0\nv 10 10 0\nv -10 10 0\nf 1 2 3 4\n"
    wall = "v 4 -5 0\nv 4 5 0\nv 4 5 6\nv 4 -5 6\nf 1 2 3 4\n"
    (tmp_path / "floor.obj").write_text(quad)
    (tmp_path / "sub dir" / "wall.obj").write_text(wall)
    p = tmp_path / "s.scene"
    p.write_text(C.GOOD)
    return p


@pytest.mark.gpu
def test_load_scene_and_round_trip(cuda, tmp_path):
    from paper_2504_21719_b200.errors import MissingMesh, UnresolvedMaterial
    ls = sceneio.load_scene(_scene_dir(tmp_path))
    assert ls.frequency == 3.5e9 and ls.warnings == []
    assert [m.object_id for m in ls.model.meshes] == [0, 1]
    assert ls.model.accel.num_triangles == 4
    assert np.array_equal(ls.model.velocities[0], [0.0, 0.5, 0.0])
    tx = ls.transmitters[0]
    assert tx.array.offsets.shape == (8, 3) and tx.name == "tx0"
    out = sceneio.write_scene(ls, tmp_path / "copy")
    again = sceneio.load_scene(out)
    assert again.model.accel.num_triangles == 4
    assert describe(again.description)["materials"] == describe(ls.description)["materials"]
    assert np.allclose(again.transmitters[0].array.offsets, tx.array.offsets, atol=1e-15)
    bad = tmp_path / "bad.scene"
    bad.write_text(C.MINIMAL + "object o\n  mesh floor.obj\n  material nope\n")
    with pytest.raises(UnresolvedMaterial):
        sceneio.load_scene(bad)
    bad.write_text(C.MINIMAL + "material m\n  eps_r 3\nobject o\n  mesh none.obj\n  material m\n")
    with pytest.raises(MissingMesh):
        sceneio.load_scene(bad)
