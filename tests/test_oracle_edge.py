"""CPU oracle of the edge (diffraction) radio-map estimator vs the reference (golden)."""

import numpy as np
import pytest

import oracle
from conftest import golden
from edge_cases import EDGE_CASES, edge_geometry
from paper_2504_21719_b200.em import ArrayGeometry, make_pattern
from paper_2504_21719_b200.materials import RadioMaterial
from paper_2504_21719_b200.radiomap import MeasurementGrid, RadioMapConfig


def edge_case(name):
    c = EDGE_CASES[name]
    meshes, mats = edge_geometry(name)
    pm = {o: RadioMaterial("m%d" % o, **md) for o, md in mats.items()}
    grid = MeasurementGrid(*c["grid"])
    cfg = RadioMapConfig(wedge_radius=c["radius"], **c["cfg"])
    kw = {}
    if c.get("pattern"):
        kw["pattern"] = make_pattern(c["pattern"][0], orientation=c["pattern"][1])
    if c.get("array"):
        kw["array"] = ArrayGeometry(np.asarray(c["array"], dtype=np.float64))
        kw["precoder"] = np.asarray(c["precoder"], dtype=np.complex128)
    return meshes, pm, grid, cfg, np.asarray(c["src"], dtype=np.float64), kw


def gold(name, key):
    return golden("edge.npz")[f"{name}__{key}"]


def compare_maps(got, want, tight=1e-9, frac=0.99, loose=1e-3):
    nz = (want != 0) | (got != 0)
    rel = np.abs(got[nz] - want[nz]) / np.maximum(np.abs(want[nz]), 1e-300)
    assert np.mean(rel < tight) >= frac, (np.mean(rel < tight), rel.max())
    assert np.quantile(rel, 0.999) < loose, rel.max()
    return rel


@pytest.mark.parametrize("name", list(EDGE_CASES))
def test_oracle_edge_map_matches_reference(name):
    meshes, pm, grid, cfg, src, kw = edge_case(name)
    sc = oracle.OracleScene(meshes, pm)
    radius = EDGE_CASES[name]["radius"]
    if radius is None:
        lo = np.minimum.reduce([m.vertices.min(0) for m in meshes])
        hi = np.maximum.reduce([m.vertices.max(0) for m in meshes])
        radius = float(np.linalg.norm((hi + 1e-12 * (1 + np.abs(hi)))
                                      - (lo - 1e-12 * (1 + np.abs(lo)))))
    ids = sc.collect_wedges_near_source(src, radius)
    assert ids == list(gold(name, "wedge_ids"))
    vals, diag = sc.radiomap_edges(src, grid, cfg, ids, **kw)
    assert diag["cone_samples"] == int(gold(name, "edgediag__cone_samples"))
    assert diag["deposits"] == int(gold(name, "edgediag__deposits"))
    compare_maps(vals, gold(name, "edge_values"))
