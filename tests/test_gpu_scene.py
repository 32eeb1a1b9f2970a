"""Scene ingestion on the GPU: per-slot tables derived by
sbr_scene_create on the device, pinned to the real reference.

Golden: tests/golden/tables.npz (make_golden_tables.py, emtrace's SceneModel
normals and plane hashes keyed by (object_id, primitive_id)).
"""

import numpy as np
import pytest

from conftest import golden, golden_trace_meshes
from paper_2504_21719_b200 import SceneModel, scenes
from paper_2504_21719_b200.materials import RadioMaterial
from paper_2504_21719_b200.paths import plane_hash_rows

pytestmark = pytest.mark.gpu


def _keyed(scene):
    a = scene.accel
    order = np.lexsort((a.tri_primitive_id, a.tri_object_id))
    return (a.tri_object_id[order], a.tri_primitive_id[order], a.tri_normal[order],
            scene.tri_plane_hash_round[order], scene.tri_plane_hash_floor[order])


@pytest.mark.parametrize("which", ["canyon", "soup"])
def test_device_tables_match_reference(cuda, which):
    g = golden("tables.npz")
    meshes = scenes.street_canyon() if which == "canyon" else golden_trace_meshes()
    sc = SceneModel(meshes, {m.object_id: RadioMaterial() for m in meshes})
    obj, prim, nrm, hr, hf = _keyed(sc)
    assert np.array_equal(obj, g[f"{which}_obj"]) and np.array_equal(prim, g[f"{which}_prim"])
    assert np.array_equal(nrm, g[f"{which}_normal"])          # bit-exact float64
    assert np.array_equal(hr, g[f"{which}_hash_r"])
    assert np.array_equal(hf, g[f"{which}_hash_f"])


def test_device_tables_match_host_expression_on_city(cuda):
    """483,200 triangles: the device normals / hashes equal the reference's numpy
    expressions (np.cross / np.linalg.norm, _plane_hash_rows) evaluated on the
    host over the same slot-ordered corners."""
    meshes = scenes.city()
    sc = SceneModel(meshes, scenes.uniform_materials(meshes, scenes.concrete()))
    a = sc.accel
    n = np.cross(a.tri_v1 - a.tri_v0, a.tri_v2 - a.tri_v0)
    n = n / np.linalg.norm(n, axis=1, keepdims=True)
    assert np.array_equal(a.tri_normal, n)
    hr, hf = plane_hash_rows(n, a.tri_v0)
    assert np.array_equal(sc.tri_plane_hash_round, hr)
    assert np.array_equal(sc.tri_plane_hash_floor, hf)
