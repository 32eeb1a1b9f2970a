"""GPU edge (diffraction) radio-map estimator vs the reference (golden) and the oracle."""

import numpy as np
import pytest

import oracle
from edge_cases import EDGE_CASES
from paper_2504_21719_b200 import SceneModel, compute_radio_map
from paper_2504_21719_b200.paths import RadioDevice
from paper_2504_21719_b200.radiomap import (collect_wedges_near_source,
                                            compute_radio_map_diffraction)
from test_oracle_edge import compare_maps, edge_case, gold

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", list(EDGE_CASES))
def test_edge_map_matches_reference(cuda, name):
    meshes, pm, grid, cfg, src, kw = edge_case(name)
    scene = SceneModel(meshes, pm)
    radius = EDGE_CASES[name]["radius"]
    if radius is None:
        lo, hi = scene.accel.bounds
        radius = float(np.linalg.norm(hi - lo))
    ids = collect_wedges_near_source(scene, src, radius)
    assert ids == list(gold(name, "wedge_ids"))
    vals, diag = compute_radio_map_diffraction(scene, src, grid, ids, cfg, **kw)
    assert diag["cone_samples"] == int(gold(name, "edgediag__cone_samples"))
    assert diag.get("deposits", 0) == int(gold(name, "edgediag__deposits"))
    compare_maps(vals, gold(name, "edge_values"))
    # full compute_radio_map with D enabled: bounce + direct + edge terms
    pre = kw.pop("precoder", None)
    dev = RadioDevice(position=src, **kw)
    res = compute_radio_map(scene, [dev], grid, cfg, precoders=None if pre is None else [pre])
    compare_maps(res.values[0], gold(name, "values"))
    from conftest import golden
    g = golden("edge.npz")
    for key in ("deposits", "cone_samples", "wedges", "direct_visible", "respawns", "escaped"):
        want = int(g[f"{name}__diag__{key}"]) if f"{name}__diag__{key}" in g.files else 0
        assert res.diagnostics[0].get(key, 0) == want, key


def test_edge_map_city_vs_oracle(cuda):
    """Beyond the fixtures: 64 city wedges near the Tx, 2e4 samples each."""
    from paper_2504_21719_b200 import scenes
    from paper_2504_21719_b200.radiomap import MeasurementGrid, RadioMapConfig
    meshes = scenes.city(n=8)
    mats = scenes.uniform_materials(meshes, scenes.concrete())
    scene = SceneModel(meshes, mats)
    grid = MeasurementGrid((0.0, 0.0, 1.5), (1, 0, 0), (0, 1, 0), (2.0, 2.0), (100, 100))
    cfg = RadioMapConfig(num_samples=1000, wedge_samples=20_000, max_depth=1, seed=7)
    src = np.array([3.0, -4.0, 30.0])
    ids = collect_wedges_near_source(scene, src, 60.0)[:64]
    assert len(ids) > 10
    vals, diag = compute_radio_map_diffraction(scene, src, grid, ids, cfg)
    osc = oracle.OracleScene(meshes, mats)
    assert osc.collect_wedges_near_source(src, 60.0)[:64] == ids
    want, wdiag = osc.radiomap_edges(src, grid, cfg, ids)
    assert diag.get("deposits", 0) == wdiag["deposits"]
    compare_maps(vals, want)
