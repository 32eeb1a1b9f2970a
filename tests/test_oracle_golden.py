"""Pin the CPU oracle against golden vectors produced by the real reference.

CPU only.  Fixtures come from tests/golden/make_golden.py (emtrace imported
from /root/reference in the build container).
"""

import numpy as np
import pytest

import oracle
from cases import COUNTER_KEYS, MAP_CASES, build_case, case_meshes, golden_map
from conftest import golden, golden_trace_meshes
from paper_2504_21719_b200.materials import RadioMaterial
from paper_2504_21719_b200.paths import plane_hash_rows


def test_rng_streams_bit_exact():
    g = golden("rng.npz")
    for k in range(len(g["draws"])):
        got = oracle.philox_uniform(int(g["seeds"][k]), int(g["samples"][k]),
                                    int(g["depths"][k]), str(g["purposes"][k]),
                                    g["draws"].shape[1])
        assert np.array_equal(got, g["draws"][k])


@pytest.mark.parametrize("key", ["full_1", "full_2", "full_7", "full_1000"])
def test_fibonacci_small_bit_exact(key):
    g = golden("fibonacci.npz")
    n = int(key.split("_")[1])
    assert np.array_equal(oracle.fibonacci(n), g[key])


def test_fibonacci_1e7_slices_bit_exact():
    g = golden("fibonacci.npz")
    for lo in (0, 4_999_968, 9_999_936):
        got = oracle.fibonacci(10_000_000, lo, lo + 64)
        assert np.array_equal(got, g[f"big_{lo}"])


def test_slab_fresnel_matches_reference():
    g = golden("fresnel.npz")
    for k in range(len(g["eps_r"])):
        m = RadioMaterial("m", eps_r=float(g["eps_r"][k]), sigma=float(g["sigma"][k]),
                          thickness=float(g["thickness"][k]))
        got = oracle.slab_fresnel(m.to_abi(3.5e9), g["cos"])
        want = g["coeff"][k]
        finite = np.isfinite(want)
        assert np.array_equal(np.isfinite(got), finite)
        np.testing.assert_allclose(got[finite], want[finite], rtol=1e-13, atol=1e-300)


def test_trace_closest_and_any_bit_exact():
    g = golden("trace.npz")
    sc = oracle.OracleScene(golden_trace_meshes())
    t, tri, u, v = sc.trace_batch(g["origins"], g["dirs"])
    obj = np.where(tri >= 0, sc.tri_object_id[tri], -1)
    prim = np.where(tri >= 0, sc.tri_primitive_id[tri], -1)
    assert np.array_equal(obj, g["obj"]) and np.array_equal(prim, g["prim"])
    assert np.array_equal(t, g["t"]) and np.array_equal(u, g["u"]) and np.array_equal(v, g["v"])
    anyhit = sc.any_hit_batch(g["origins"], g["dirs"], 1e-4, g["tmax"])
    assert np.array_equal(anyhit, g["anyhit"])
    assert np.array_equal(sc.occluded_batch(g["seg_a"], g["seg_b"]), g["occluded"])


def test_plane_hashes_bit_exact():
    g = golden("hashes.npz")
    hr, hf = plane_hash_rows(g["normals"], g["points"])
    assert np.array_equal(hr, g["hash_r"]) and np.array_equal(hf, g["hash_f"])


def test_scene_generators_match_golden_digest():
    import sys, os
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from make_golden import mesh_digest
    g = golden("radiomap.npz")
    assert mesh_digest(case_meshes("canyon_rs")) == str(g["canyon_digest"])
    assert mesh_digest(case_meshes("box_rs")) == str(g["box_digest"])


@pytest.mark.parametrize("name", list(MAP_CASES))
def test_oracle_radio_map_matches_reference(name):
    g = golden("radiomap.npz")
    want, want_diag = golden_map(g, name)
    meshes, mats, src, grid, cfg, kw = build_case(name)
    vals, diag = oracle.OracleScene(meshes, mats).radiomap(src, grid, cfg, **kw)
    for key in COUNTER_KEYS:
        assert diag.get(key, 0) == want_diag.get(key, 0), key
    nz = want != 0
    assert np.array_equal(vals != 0, nz)
    rel = np.abs(vals[nz] - want[nz]) / np.abs(want[nz])
    assert rel.max() < 1e-12, rel.max()
