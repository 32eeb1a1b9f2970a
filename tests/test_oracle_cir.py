"""Pin the CPU oracle's path-solver restatement against the real reference (CPU only).

Golden fixtures: tests/golden/cir.npz (tests/golden/make_golden_cir.py runs
emtrace's generate_candidates / compute_paths / frequency_response).  The
oracle is the checker the GPU path is compared with at sizes beyond the
fixtures (tests/test_gpu_cir.py) and the CPU baseline of the CIR metric.
"""

import numpy as np
import pytest

import oracle
from cir_cases import CIR_CASES, case_geometry
from conftest import golden
from paper_2504_21719_b200.em import ArrayGeometry, make_pattern
from paper_2504_21719_b200.materials import RadioMaterial, ScatteringPattern
from paper_2504_21719_b200.paths import PathConfig, RadioDevice
from paper_2504_21719_b200.sampling import Interaction

KINDS = {"R": Interaction.REFLECTION, "S": Interaction.SCATTERING,
         "T": Interaction.TRANSMISSION, "D": Interaction.DIFFRACTION}
_SC = {}


def oracle_case(name):
    c = CIR_CASES[name]
    if name not in _SC:
        meshes, mats, vel = case_geometry(name)
        pm = {}
        for oid, md in mats.items():
            md = dict(md)
            pat = md.pop("pattern", None)
            if pat is not None:
                md["pattern"] = ScatteringPattern(kind=pat[0], alpha_r=pat[1], alpha_i=pat[2],
                                                  lambda_mix=pat[3])
            pm[oid] = RadioMaterial("m%d" % oid, **md)
        _SC[name] = oracle.OracleScene(meshes, pm, velocities=vel)
    kw = dict(c["cfg"])
    kw["enabled"] = frozenset(KINDS[k] for k in c["kinds"])
    cfg = PathConfig(**kw)

    def device(d):
        kw = {}
        if d.get("pattern"):
            kw["pattern"] = make_pattern(d["pattern"][0], orientation=d["pattern"][1])
        if d.get("array"):
            kw["array"] = ArrayGeometry(np.asarray(d["array"], dtype=np.float64))
        if d.get("velocity") is not None:
            kw["velocity"] = np.asarray(d["velocity"], dtype=np.float64)
        return RadioDevice(position=np.asarray(d["pos"], dtype=np.float64), **kw)

    return _SC[name], cfg, [device(d) for d in c["tx"]], [device(d) for d in c["rx"]]


def gold(name, prefix):
    g = golden("cir.npz")
    p = f"{name}__{prefix}"
    return {k[len(p):]: g[k] for k in g.files if k.startswith(p)}


@pytest.mark.parametrize("name", list(CIR_CASES))
def test_oracle_generation_matches_reference(name):
    sc, cfg, txs, rxs = oracle_case(name)
    targets = (np.array([r.position for r in rxs]) if cfg.synthetic_arrays
               else np.concatenate([r.element_positions() for r in rxs]))
    src = txs[0].position if cfg.synthetic_arrays else txs[0].element_positions()[0]
    rec, diag = sc.generate_candidates(src, targets, cfg)
    want = gold(name, "gen_")
    for k, v in gold(name, "gendiag__").items():
        if k == "hash_load_factor":
            assert diag[k] == pytest.approx(float(v), rel=1e-12)
        else:
            assert diag.get(k, 0) == int(v), k
    for k in ("sample", "target", "depth", "suffix_start"):
        assert np.array_equal(rec[k], want[k]), k
    assert np.array_equal(rec["diffuse"].astype(bool), want["diffuse"])
    assert np.array_equal(rec["chain_hash"], want["chain_hash"])
    np.testing.assert_allclose(rec["prefix_prob"], want["prefix_prob"], rtol=1e-12)
    np.testing.assert_allclose(rec["anchor"], want["anchor"], rtol=0, atol=1e-12)
    L = want["kind"].shape[1]
    kind = np.where(np.arange(rec["kind"].shape[1])[None, :] < rec["depth"][:, None],
                    rec["kind"], -1)[:, :L]
    assert np.array_equal(kind, want["kind"])
    tri = rec["tri"][:, :L]
    obj = np.where(kind >= 0, sc.tri_object_id[np.maximum(tri, 0)], -1)
    prim = np.where(kind >= 0, sc.tri_primitive_id[np.maximum(tri, 0)], -1)
    assert np.array_equal(obj, want["obj"]) and np.array_equal(prim, want["prim"])
    m = kind >= 0
    assert np.array_equal(np.where(m, rec["wedge"][:, :L], -1), want["wedge"])
    np.testing.assert_allclose(rec["vertex"][:, :L][m], want["vertex"][m], rtol=0, atol=1e-12)
    assert np.array_equal(rec["normal"][:, :L][m], want["normal"][m])


@pytest.mark.parametrize("name", list(CIR_CASES))
def test_oracle_paths_match_reference(name):
    sc, cfg, txs, rxs = oracle_case(name)
    paths, diag = sc.compute_paths(txs, rxs, cfg)
    want = gold(name, "path_")
    n = len(want["delay"])
    assert diag["paths"] == n
    if n == 0:
        return
    for k in ("tx", "tx_el", "rx", "rx_el", "depth", "sample"):
        assert np.array_equal(paths[k], want[k]), k
    assert np.array_equal(paths["chain_hash"], want["chain_hash"])
    L = want["kind"].shape[1]
    assert np.array_equal(paths["kind"][:, :L], want["kind"])
    assert np.array_equal(paths["obj"][:, :L], want["obj"])
    assert np.array_equal(paths["wedge"][:, :L], want["wedge"])
    for i in range(n):
        d = int(want["depth"][i])
        np.testing.assert_allclose(paths["vertices"][i, :d + 2], want["vertices"][i, :d + 2],
                                   rtol=0, atol=1e-9)
    np.testing.assert_allclose(paths["delay"], want["delay"], rtol=1e-12)
    rel = np.abs(paths["gain"] - want["gain"]) / np.abs(want["gain"])
    assert rel.max() < 1e-6, rel.max()
    np.testing.assert_allclose(paths["doppler"], want["doppler"], rtol=1e-9, atol=1e-9)
    for k, v in gold(name, "diag__").items():
        if k.startswith("rej__"):
            assert diag["refinement_rejections"].get(k[5:], 0) == int(v), k
        elif k == "hash_load_factor":
            assert diag[k] == pytest.approx(float(v), rel=1e-12)
        else:
            assert diag.get(k, 0) == int(v), k
    c = CIR_CASES[name]
    if c.get("freqs") is not None:
        H = oracle.frequency_response(paths, cfg, txs[0], rxs[0], c["freqs"])
        wh = golden("cir.npz")[f"{name}__cfr"]
        assert np.abs(H - wh).max() / np.abs(wh).max() < 1e-9
