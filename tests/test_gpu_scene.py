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


def _check_wedges_equal(got, want, tol=1e-12):
    assert len(got) == len(want)
    for a, b in zip(got, want):
        assert [tuple(x) for x in a.face0] == [tuple(x) for x in b.face0]
        assert [tuple(x) for x in a.facen] == [tuple(x) for x in b.facen]
        for attr in ("origin", "e_hat", "n0_hat", "nn_hat", "t0_hat"):
            np.testing.assert_allclose(getattr(a, attr), getattr(b, attr), rtol=0, atol=tol)
        assert abs(a.length - b.length) <= tol and abs(a.n - b.n) <= tol


def test_device_wedges_match_reference_golden(cuda):
    """GPU wedge extraction + edge hashes vs emtrace's extract_wedges / hash_edge
    on the diffraction cases (tests/golden/cir.npz)."""
    from cir_cases import D_CASES, case_geometry
    from paper_2504_21719_b200.wedges import extract_wedges_device
    g = golden("cir.npz")
    for name in D_CASES:
        p = f"{name}__wedge_"
        meshes, _, _ = case_geometry(name)
        W, t = extract_wedges_device(meshes)
        assert len(W) == len(g[p + "length"]), name
        own = g[p + "owners"]
        for i, w in enumerate(W):
            sel = own[own[:, 0] == i]
            assert [tuple(r[2:]) for r in sel if r[1] == 0] == [tuple(x) for x in w.face0]
            assert [tuple(r[2:]) for r in sel if r[1] == 1] == [tuple(x) for x in w.facen]
            for attr, key in (("origin", "origin"), ("e_hat", "ehat"), ("n0_hat", "n0"),
                              ("nn_hat", "nn"), ("t0_hat", "t0")):
                np.testing.assert_allclose(getattr(w, attr), g[p + key][i], rtol=0, atol=1e-12)
            assert w.length == pytest.approx(float(g[p + "length"][i]), abs=1e-12)
            assert w.n == pytest.approx(float(g[p + "n"][i]), abs=1e-12)
        assert np.array_equal(t["hash_r"], g[p + "hash_r"].astype(np.uint64))
        assert np.array_equal(t["hash_f"], g[p + "hash_f"].astype(np.uint64))


def test_device_wedges_match_host_extraction_on_city(cuda):
    """The 483,200-triangle city (12,964 wedges): GPU extraction equals the
    host restatement (itself pinned to the reference by test_wedges.py) owner
    for owner, frames to 1e-12, edge hashes exactly; and a SceneModel with
    diffraction tables builds fast."""
    import time

    from paper_2504_21719_b200.wedges import extract_wedges, extract_wedges_device, hash_edge
    meshes = scenes.city()
    W, t = extract_wedges_device(meshes)
    ref = extract_wedges(meshes)
    _check_wedges_equal(W, ref)
    hs = np.array([hash_edge(w) for w in ref], dtype=np.uint64)
    assert np.array_equal(t["hash_r"], hs[:, 0]) and np.array_equal(t["hash_f"], hs[:, 1])
    mats = scenes.uniform_materials(meshes, scenes.concrete())
    SceneModel(meshes, mats).wedges  # warm (CUDA context, kernels)
    t0 = time.perf_counter()
    sc = SceneModel(meshes, mats)
    assert len(sc.wedges) == len(ref)
    dt = time.perf_counter() - t0
    print(f"city SceneModel + wedge tables: {dt:.3f} s")
    assert dt < 1.0
