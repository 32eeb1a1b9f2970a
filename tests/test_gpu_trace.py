"""GPU parity of the LBVH + traversal kernels against the oracle and golden vectors."""

import numpy as np
import pytest

import oracle
from conftest import golden, golden_trace_meshes
from paper_2504_21719_b200 import scenes
from paper_2504_21719_b200.errors import EmptyScene
from paper_2504_21719_b200.geometry import Mesh, Ray, build_scene_accel, intersect_closest, is_occluded

pytestmark = pytest.mark.gpu


def _ids(acc, tri):
    return (np.where(tri >= 0, acc.tri_object_id[tri], -1),
            np.where(tri >= 0, acc.tri_primitive_id[tri], -1))


def test_closest_bit_exact_vs_reference_golden(cuda):
    g = golden("trace.npz")
    acc = build_scene_accel(golden_trace_meshes())
    t, tri, u, v = acc.trace_batch(g["origins"], g["dirs"])
    obj, prim = _ids(acc, tri)
    assert np.array_equal(obj, g["obj"]) and np.array_equal(prim, g["prim"])
    assert np.array_equal(t, g["t"])
    assert np.array_equal(u, g["u"]) and np.array_equal(v, g["v"])


def test_any_hit_and_occlusion_vs_golden(cuda):
    g = golden("trace.npz")
    acc = build_scene_accel(golden_trace_meshes())
    assert np.array_equal(acc.any_hit_batch(g["origins"], g["dirs"], 1e-4, g["tmax"]),
                          g["anyhit"])
    assert np.array_equal(acc.occluded_batch(g["seg_a"], g["seg_b"]), g["occluded"])
    # occlusion is symmetric
    assert np.array_equal(acc.occluded_batch(g["seg_b"], g["seg_a"]), g["occluded"])


@pytest.mark.parametrize("scene", ["canyon", "soup"])
def test_closest_bit_exact_vs_oracle_large(cuda, rng, scene):
    if scene == "canyon":
        meshes = scenes.street_canyon()
        o = rng.uniform([-100, -100, 0.5], [100, 100, 45], size=(200_000, 3))
    else:
        meshes = golden_trace_meshes()
        o = rng.normal(size=(200_000, 3)) * 2.5
    d = rng.normal(size=o.shape)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    acc = build_scene_accel(meshes)
    ref = oracle.OracleScene(meshes)
    t, tri, u, v = acc.trace_batch(o, d)
    rt, rtri, ru, rv = ref.trace_batch(o, d)
    assert np.array_equal(_ids(acc, tri)[0], np.where(rtri >= 0, ref.tri_object_id[rtri], -1))
    assert np.array_equal(_ids(acc, tri)[1], np.where(rtri >= 0, ref.tri_primitive_id[rtri], -1))
    assert np.array_equal(t, rt) and np.array_equal(u, ru) and np.array_equal(v, rv)
    tmax = rng.uniform(0.5, 80.0, size=len(o))
    assert np.array_equal(acc.any_hit_batch(o, d, 1e-4, tmax), ref.any_hit_batch(o, d, 1e-4, tmax))


def test_every_triangle_reachable(cuda, rng):
    # reference test_geometry.py:102-118 at 1e5 triangles
    from conftest import ROOT  # noqa: F401
    tris = []
    while len(tris) < 100_000:
        pts = rng.uniform(-5, 5, size=(100_000, 3, 3))
        size = rng.uniform(0.01, 0.2, size=(100_000, 1, 1))
        pts = pts[:, :1, :] + (pts - pts[:, :1, :]) * size
        area = 0.5 * np.linalg.norm(np.cross(pts[:, 1] - pts[:, 0], pts[:, 2] - pts[:, 0]), axis=1)
        tris.extend(pts[area > 1e-6][: 100_000 - len(tris)])
    tris = np.asarray(tris)
    mesh = Mesh(tris.reshape(-1, 3), np.arange(3 * len(tris)).reshape(-1, 3), object_id=0)
    acc = build_scene_accel([mesh])
    a, b, c = mesh.triangle_corners()
    cen = (a + b + c) / 3.0
    nrm = mesh.triangle_normals()
    t, tri, _, _ = acc.trace_batch(cen + 5e-4 * nrm, -nrm)
    assert np.all(tri >= 0)
    assert np.all(t <= 5e-4 + 1e-9)


def test_small_scenes_and_tie_rule(cuda):
    quad = scenes.quad_mesh()
    acc = build_scene_accel([quad])
    h = intersect_closest(acc, Ray(np.array([0.5, 0.5, 2.0]), np.array([0.0, 0.0, -1.0])))
    assert (h.object_id, h.primitive_id) == (0, 0)  # shared diagonal -> lower primitive
    ray = Ray(np.array([0.0, 0.0, 1.0]), np.array([0.0, 0.0, -1.0]))
    assert intersect_closest(acc, ray).t == pytest.approx(1.0, abs=1e-12)
    assert intersect_closest(acc, Ray(ray.origin, ray.direction, max_t=0.5)) is None
    below = intersect_closest(acc, Ray(np.array([0.2, 0.1, -1.0]), np.array([0.0, 0.0, 1.0])))
    assert np.allclose(below.normal, [0, 0, -1])
    ground = build_scene_accel([scenes.quad_mesh()])
    assert is_occluded(ground, np.array([0, 0, -1.0]), np.array([0, 0, 1.0]))
    assert not is_occluded(ground, np.array([0.1, 0.1, 0.0]), np.array([0, 0, 1.0]))
    with pytest.raises(EmptyScene):
        build_scene_accel([])


def test_sampling_kernels_match_golden(cuda):
    from paper_2504_21719_b200.sampling import fibonacci_directions, rng_uniform
    g = golden("fibonacci.npz")
    for n in (1, 2, 7, 1000):
        got = fibonacci_directions(n).cpu().numpy()
        np.testing.assert_allclose(got, g[f"full_{n}"], rtol=0, atol=4e-16)
    for lo in (0, 4_999_968, 9_999_936):
        got = fibonacci_directions(10_000_000, lo, lo + 64).cpu().numpy()
        np.testing.assert_allclose(got, g[f"big_{lo}"], rtol=0, atol=4e-16)
    r = golden("rng.npz")
    for k in range(len(r["draws"])):
        got = rng_uniform(int(r["seeds"][k]), int(r["samples"][k]), int(r["depths"][k]),
                          str(r["purposes"][k]), r["draws"].shape[1]).cpu().numpy()
        assert np.array_equal(got, r["draws"][k])
