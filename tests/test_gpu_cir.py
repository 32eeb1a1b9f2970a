"""GPU parity of the path solver (CIR) against golden vectors from the real reference.

Fixtures: tests/golden/cir.npz, made by tests/golden/make_golden_cir.py from
emtrace's own generate_candidates / compute_paths / frequency_response on the
cases of tests/cir_cases.py.

Bars (north star): interaction sequences and deduplicated path sets
bit-exact; gains, delays and angles within 1e-4 relative.  Generation is
float64 in the reference's operation order, so candidate records are
compared exactly (every field, including vertices); refined vertices to
1e-9 m; gains to 1e-6 relative (asserting the 1e-4 contract with margin).
"""

import numpy as np
import pytest

from cir_cases import CIR_CASES, case_geometry, mesh_digest
from conftest import golden
from paper_2504_21719_b200 import (PathConfig, RadioDevice, SceneModel, compute_paths,
                                   frequency_response, generate_candidates, refine_candidate)
from paper_2504_21719_b200.cir import PathGeometry
from paper_2504_21719_b200.em import ArrayGeometry, make_pattern
from paper_2504_21719_b200.materials import RadioMaterial, ScatteringPattern
from paper_2504_21719_b200.sampling import Interaction

pytestmark = pytest.mark.gpu

KINDS = {"R": Interaction.REFLECTION, "S": Interaction.SCATTERING,
         "T": Interaction.TRANSMISSION, "D": Interaction.DIFFRACTION}
KIND_CODE = {Interaction.REFLECTION: 0, Interaction.SCATTERING: 1,
             Interaction.TRANSMISSION: 2, Interaction.DIFFRACTION: 3}

_SCENES = {}


def build(name):
    c = CIR_CASES[name]
    if name not in _SCENES:
        meshes, mats, vel = case_geometry(name)
        pm = {}
        for oid, md in mats.items():
            md = dict(md)
            pat = md.pop("pattern", None)
            if pat is not None:
                md["pattern"] = ScatteringPattern(kind=pat[0], alpha_r=pat[1], alpha_i=pat[2],
                                                  lambda_mix=pat[3])
            pm[oid] = RadioMaterial("m%d" % oid, **md)
        _SCENES[name] = (SceneModel(meshes, pm, velocities=vel), mesh_digest(meshes))
    scene, digest = _SCENES[name]
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

    return scene, digest, cfg, [device(d) for d in c["tx"]], [device(d) for d in c["rx"]]


def gold(name, prefix):
    g = golden("cir.npz")
    p = f"{name}__{prefix}"
    return {k[len(p):]: g[k] for k in g.files if k.startswith(p)}


@pytest.mark.parametrize("name", list(CIR_CASES))
def test_generate_candidates_bit_exact(cuda, name):
    scene, digest, cfg, txs, rxs = build(name)
    assert digest == str(golden("cir.npz")[f"{name}__digest"])
    want = gold(name, "gen_")
    wdiag = gold(name, "gendiag__")
    targets = (np.array([r.position for r in rxs]) if cfg.synthetic_arrays
               else np.concatenate([r.element_positions() for r in rxs]))
    src = txs[0].position if cfg.synthetic_arrays else txs[0].element_positions()[0]
    res = generate_candidates(scene, src, targets, cfg)
    for k, v in wdiag.items():
        if k == "hash_load_factor":
            assert res.diagnostics[k] == pytest.approx(float(v), rel=1e-12)
        else:
            assert res.diagnostics.get(k, 0) == int(v), k
    recs = res.records
    assert len(recs) == len(want["sample"])
    for i, r in enumerate(recs):
        assert r.sample_id == want["sample"][i], i
        assert r.target_id == want["target"][i], i
        assert len(r.steps) == want["depth"][i], i
        assert r.suffix_start == want["suffix_start"][i], i
        assert r.diffuse_terminal == bool(want["diffuse"][i]), i
        assert r.chain_hash == int(want["chain_hash"][i]), i
        assert r.prefix_probability == pytest.approx(want["prefix_prob"][i], rel=1e-12), i
        np.testing.assert_allclose(r.anchor, want["anchor"][i], rtol=0, atol=1e-12)
        for j, st in enumerate(r.steps):
            assert KIND_CODE[st.kind] == want["kind"][i, j]
            assert st.object_id == want["obj"][i, j] and st.primitive_id == want["prim"][i, j]
            assert st.wedge_index == want["wedge"][i, j]
            # CUDA's sin/cos may differ from glibc by 1 ulp in the launch
            # direction; geometry then agrees to ~1e-15 m, decisions exactly
            np.testing.assert_allclose(st.vertex, want["vertex"][i, j], rtol=0, atol=1e-12)
            assert np.array_equal(st.normal, want["normal"][i, j]), (i, j)


@pytest.mark.parametrize("name", list(CIR_CASES))
def test_compute_paths_matches_reference(cuda, name):
    scene, _, cfg, txs, rxs = build(name)
    want = gold(name, "path_")
    ps = compute_paths(scene, txs, rxs, cfg)
    T = ps.tensors
    n = len(want["delay"])
    assert len(T) == n
    for k in ("tx", "tx_el", "rx", "rx_el", "depth", "sample"):
        assert np.array_equal(getattr(T, k), want[k]), k
    assert np.array_equal(T.chain_hash.astype(np.uint64), want["chain_hash"])
    L = want["kind"].shape[1]
    kind = np.where(np.arange(T.kind.shape[1])[None, :] < T.depth[:, None], T.kind, -1)
    assert np.array_equal(kind[:, :L], want["kind"])
    obj = np.where(kind >= 0, T.obj, -1)[:, :L]
    prim = np.where(kind >= 0, T.prim, -1)[:, :L]
    assert np.array_equal(obj, want["obj"]) and np.array_equal(prim, want["prim"])
    assert np.array_equal(np.where(kind >= 0, T.wedge, -1)[:, :L], want["wedge"])
    for i in range(n):
        d = int(want["depth"][i])
        np.testing.assert_allclose(T.vertices[i, :d + 2], want["vertices"][i, :d + 2],
                                   rtol=0, atol=1e-9)
    np.testing.assert_allclose(T.delay, want["delay"], rtol=1e-12)
    np.testing.assert_allclose(T.departure, want["departure"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(T.arrival, want["arrival"], rtol=0, atol=1e-12)
    g, wg = T.gain, want["gain"]
    scale = np.maximum(np.abs(wg), 1e-300)
    rel = np.abs(g - wg) / scale
    assert rel.max(initial=0.0) < 1e-6, rel.max()
    np.testing.assert_allclose(T.doppler, want["doppler"], rtol=1e-9, atol=1e-9)
    wd = gold(name, "diag__")
    for k, v in wd.items():
        if k.startswith("rej__"):
            assert ps.diagnostics["refinement_rejections"].get(k[5:], 0) == int(v), k
        elif k == "hash_load_factor":
            assert ps.diagnostics[k] == pytest.approx(float(v), rel=1e-12)
        else:
            assert ps.diagnostics.get(k, 0) == int(v), k
    # lazily-built reference objects agree with the SoA view
    if n:
        p0 = ps.paths[0]
        assert p0.depth == want["depth"][0] and p0.gain == complex(T.gain[0])


@pytest.mark.parametrize("name", [k for k, c in CIR_CASES.items() if c.get("freqs") is not None])
def test_frequency_response_matches_reference(cuda, name):
    scene, _, cfg, txs, rxs = build(name)
    g = golden("cir.npz")
    ps = compute_paths(scene, txs, rxs, cfg)
    H = frequency_response(ps, CIR_CASES[name]["freqs"], 0, 0)
    want = g[f"{name}__cfr"]
    assert H.shape == want.shape
    err = np.abs(H - want).max() / np.abs(want).max()
    assert err < 1e-9, err


def test_refinement_fixed_point(cuda):
    # reference test_paths.py:379-389
    scene, _, cfg, txs, rxs = build("box_r")
    ps = compute_paths(scene, txs[:1], rxs[:1], cfg)
    from paper_2504_21719_b200.cir import CandidateRecord
    for p in ps.paths[:20]:
        rec = CandidateRecord(source_id=0, target_id=0, source=txs[0].position,
                              target=rxs[0].position, sample_id=p.sample_id, steps=p.steps,
                              suffix_start=0, anchor=txs[0].position, prefix_probability=1.0,
                              chain_hash=p.chain_hash)
        again = refine_candidate(rec, scene)
        assert isinstance(again, PathGeometry)
        np.testing.assert_allclose(again.vertices, p.vertices, atol=1e-9)


def test_screen_diffraction_points_minimize_length(cuda):
    # reference test_paths.py:459-481: four edge paths around a screen, each
    # diffraction point on its edge satisfying the Keller law k_in.e == k_out.e
    scene, _, cfg, txs, rxs = build("screen_d")
    ps = compute_paths(scene, txs, rxs, cfg)
    d_paths = [p for p in ps.paths if p.kinds == "D"]
    assert len(d_paths) == 4
    for p in d_paths:
        w = scene.wedges[p.steps[0].wedge_index]
        v = p.vertices[1]
        x = float((v - w.origin) @ w.e_hat)
        assert -1e-9 <= x <= w.length + 1e-9
        k_in = (v - txs[0].position) / np.linalg.norm(v - txs[0].position)
        k_out = (rxs[0].position - v) / np.linalg.norm(rxs[0].position - v)
        assert k_in @ w.e_hat == pytest.approx(k_out @ w.e_hat, abs=1e-9)


@pytest.mark.parametrize("samples,kinds", [(100_000, "R"), (50_000, "RS")])
def test_canyon_paths_vs_oracle(cuda, samples, kinds):
    """Beyond the golden fixtures: 64 street receivers in the config-2 canyon vs the oracle."""
    import oracle
    from cir_cases import _canyon_targets
    from paper_2504_21719_b200 import scenes
    meshes = scenes.street_canyon()
    mats = scenes.uniform_materials(meshes, scenes.concrete(scattering=0.2))
    rx = [RadioDevice(position=np.array(d["pos"])) for d in _canyon_targets(64, seed=9)]
    tx = RadioDevice(position=np.array([0.0, 5.0, 20.0]))
    cfg = PathConfig(num_samples=samples, max_depth=4, q_diffraction=0.0, seed=3,
                     enabled=frozenset(KINDS[k] for k in kinds))
    want, wdiag = oracle.OracleScene(meshes, mats).compute_paths([tx], rx, cfg)
    ps = compute_paths(SceneModel(meshes, mats), [tx], rx, cfg)
    T = ps.tensors
    for k, v in wdiag.items():
        if k == "refinement_rejections":
            assert ps.diagnostics[k] == v
        elif k == "hash_load_factor":
            assert ps.diagnostics[k] == pytest.approx(v, rel=1e-12)
        else:
            assert ps.diagnostics.get(k, 0) == v, k
    assert len(T) == len(want["delay"])
    for k in ("rx", "depth", "sample"):
        assert np.array_equal(getattr(T, k), want[k]), k
    assert np.array_equal(T.chain_hash.astype(np.uint64), want["chain_hash"].astype(np.uint64))
    L = want["kind"].shape[1]
    kind = np.where(np.arange(T.kind.shape[1])[None, :] < T.depth[:, None], T.kind, -1)[:, :L]
    assert np.array_equal(kind, want["kind"])
    assert np.array_equal(np.where(kind >= 0, T.obj[:, :L], -1), want["obj"])
    np.testing.assert_allclose(T.delay, want["delay"], rtol=1e-12)
    rel = np.abs(T.gain - want["gain"]) / np.maximum(np.abs(want["gain"]), 1e-300)
    assert rel.max(initial=0.0) < 1e-6, rel.max()


def test_city_paths_vs_oracle(cuda):
    """The config-3 city (483k triangles) with 64 street receivers at N_S = 2e4 vs
    the oracle: path set, every diagnostics counter, gains -- exercises the
    visibility kernel's occluder tables, far-first any-hit and emission-time
    duplicate drop on a large scene."""
    import oracle
    from paper_2504_21719_b200 import scenes
    meshes = scenes.city()
    mats = scenes.uniform_materials(meshes, scenes.concrete())
    rx = [RadioDevice(position=p) for p in scenes.city_receivers(64)]
    tx = RadioDevice(position=np.array([0.0, 0.0, 30.0]))
    cfg = PathConfig(num_samples=20_000, max_depth=4, q_diffraction=0.0,
                     enabled=frozenset({Interaction.REFLECTION}))
    want, wdiag = oracle.OracleScene(meshes, mats).compute_paths([tx], rx, cfg)
    ps = compute_paths(SceneModel(meshes, mats), [tx], rx, cfg)
    for k, v in wdiag.items():
        if k == "refinement_rejections":
            assert ps.diagnostics[k] == v
        elif k == "hash_load_factor":
            assert ps.diagnostics[k] == pytest.approx(v, rel=1e-12)
        else:
            assert ps.diagnostics.get(k, 0) == v, k
    T = ps.tensors
    assert len(T) == len(want["delay"]) > 0
    for k in ("rx", "depth", "sample"):
        assert np.array_equal(getattr(T, k), want[k]), k
    assert np.array_equal(T.chain_hash.astype(np.uint64), want["chain_hash"].astype(np.uint64))
    np.testing.assert_allclose(T.delay, want["delay"], rtol=1e-12)
    rel = np.abs(T.gain - want["gain"]) / np.maximum(np.abs(want["gain"]), 1e-300)
    assert rel.max(initial=0.0) < 1e-6, rel.max()


@pytest.mark.parametrize("name", ["box_trunc", "canyon_r", "box_rst"])
def test_sharded_selection_matches_single_gpu(cuda, name):
    """Multi-GPU CIR logic, emulated on one GPU: two sample shards swept
    separately, rows concatenated as the all-gather would, one global
    selection, per-shard materialisation -- must equal compute_paths."""
    import torch
    from paper_2504_21719_b200 import cir
    from paper_2504_21719_b200.sharding import shard_range
    scene, _, cfg, txs, rxs = build(name)
    ref = compute_paths(scene, txs[:1], rxs, cfg).tensors
    tx_flat, targets, tdevs, rx_index, rx_elem = cir._device_plan(txs[:1], rxs, cfg)
    _, _, src = tx_flat[0]
    src = np.asarray(src, np.float64)
    scene.bind_frequency(cfg.frequency)
    # contiguous halves for one case, the chunk-cyclic shards compute_paths_sharded uses
    # (sbr_cir_sweep_sharded, 4096-id chunks) for the others
    if name == "box_trunc":
        shards = [cir._sweep_rows(scene, src, targets, cfg, *shard_range(cfg.num_samples, r, 2))
                  for r in range(2)]
    else:
        shards = [cir._sweep_rows(scene, src, targets, cfg, 0, 0, shard=(r, 2)) for r in range(2)]
    offsets = [0, shards[0].n, shards[0].n + shards[1].n]
    cat = {k: torch.cat([getattr(R, k)[:R.n] for R in shards]) for k in ("key", "pr", "pf",
                                                                          "chain")}
    sel = torch.zeros(len(cir._abi.CIR_COUNTERS), dtype=torch.int64, device=cuda)
    rec_row, nrec = cir._select_rows(shards[0].params, cat["key"], cat["pr"], cat["pf"],
                                     cat["chain"], offsets[-1], shards[0].los_vis, cfg, sel, cuda)
    _check_shards(shards, rec_row, nrec, offsets, sel, scene, src, targets, cfg, txs, tdevs,
                  rx_index, rx_elem, ref, cuda)
    # the same with the shard-local pre-selection compute_paths_sharded uses at N > 1:
    # only each shard's first occurrences are "gathered", dropped rows are duplicates
    loc_rows = [cir._local_rows(R) for R in shards]
    offsets2 = [0, int(loc_rows[0][1].numel()),
                int(loc_rows[0][1].numel()) + int(loc_rows[1][1].numel())]
    cat2 = {k: torch.cat([lr[0][k] for lr in loc_rows]) for k in ("key", "pr", "pf", "chain")}
    sel2 = torch.zeros(len(cir._abi.CIR_COUNTERS), dtype=torch.int64, device=cuda)
    rec_row2, nrec2 = cir._select_rows(shards[0].params, cat2["key"], cat2["pr"], cat2["pf"],
                                       cat2["chain"], offsets2[-1], shards[0].los_vis, cfg,
                                       sel2, cuda)
    dup = cir._abi.CIR_COUNTERS.index("duplicates")
    sel2[dup] += sum(lr[2] for lr in loc_rows)
    assert np.array_equal(sel2.cpu().numpy(), sel.cpu().numpy())
    assert nrec2 == nrec
    _check_shards(shards, rec_row2, nrec2, offsets2, sel2, scene, src, targets, cfg, txs, tdevs,
                  rx_index, rx_elem, ref, cuda, kept=[lr[1] for lr in loc_rows])
    # the public entry point on a single rank
    ps = cir.compute_paths_sharded(scene, txs[:1], rxs, cfg)
    assert np.array_equal(ps.tensors.chain_hash, ref.chain_hash)


def _check_shards(shards, rec_row, nrec, offsets, sel, scene, src, targets, cfg, txs, tdevs,
                  rx_index, rx_elem, ref, cuda, kept=None):
    import torch
    from paper_2504_21719_b200 import cir
    from paper_2504_21719_b200.sharding import owned_records
    parts = []
    for r, R in enumerate(shards):
        pos, loc = owned_records(rec_row[:nrec].cpu().numpy(), offsets, r)
        if kept is not None:
            loc = np.array(loc, dtype=np.int64)
            m = loc >= 0
            loc[m] = kept[r].cpu().numpy()[loc[m]]
        recbuf = cir._materialize(R, torch.from_numpy(loc.astype(np.int64)).to(cuda), len(loc),
                                  cfg)
        cand = cir.DeviceCandidates(scene, src, targets, R.targets_t, cfg, recbuf, len(loc), 0)
        cand.params = R.params
        part, _ = cir._paths_for_source(scene, cand, cfg, 0, 0, txs[0], tdevs, rx_index, rx_elem)
        if part is not None:
            parts.append(part)
    got = cir._concat_sorted(parts, max(cfg.max_depth, 1))
    assert len(got) == len(ref)
    for k in ("rx", "depth", "sample", "chain_hash"):
        assert np.array_equal(getattr(got, k), getattr(ref, k)), k
    np.testing.assert_allclose(got.delay, ref.delay, rtol=1e-12)
    assert np.abs(got.gain - ref.gain).max(initial=0.0) <= 1e-12 * np.abs(ref.gain).max(initial=1)


def test_config5_arrays_cfr_city_vs_oracle(cuda):
    """Config 5: city, 8x8 TR 38.901 Tx panel, 4x4 Rx panel, depth 6, CFR over 1024 subcarriers."""
    import oracle
    from paper_2504_21719_b200 import scenes
    from paper_2504_21719_b200.em import planar_array
    meshes = scenes.city()
    mats = scenes.uniform_materials(meshes, scenes.concrete())
    lam = 299792458.0 / 3.5e9
    tx = RadioDevice(position=np.array([0.0, 0.0, 30.0]), pattern=make_pattern("tr38901"),
                     array=planar_array(8, 8, lam / 2, lam / 2))
    rx = RadioDevice(position=np.array([2.0, 60.0, 1.5]), array=planar_array(4, 4, lam / 2,
                                                                             lam / 2))
    cfg = PathConfig(num_samples=100_000, max_depth=6, q_diffraction=0.0,
                     enabled=frozenset({Interaction.REFLECTION}))
    freqs = 3.5e9 + (np.arange(1024) - 512) * 30e3
    ps = compute_paths(SceneModel(meshes, mats), [tx], [rx], cfg)
    H = frequency_response(ps, freqs)
    want, wdiag = oracle.OracleScene(meshes, mats).compute_paths([tx], [rx], cfg)
    assert len(ps.tensors) == len(want["delay"]) and len(want["delay"]) > 0
    assert np.array_equal(ps.tensors.chain_hash, want["chain_hash"])
    wh = oracle.frequency_response(want, cfg, tx, rx, freqs)
    assert H.shape == (16, 64, 1024)
    assert np.abs(H - wh).max() / np.abs(wh).max() < 1e-9


@pytest.mark.parametrize("synthetic", [True, False])
@pytest.mark.parametrize("dmma_min", [-1, 0, 16])
def test_cfr_contraction_many_paths_vs_oracle(cuda, synthetic, dmma_min):
    """Factorised CFR (steering x spin contraction) against the oracle's path-by-path sum:
    300 random paths (more than one K tile, ragged), 4x4 Rx x 8x8 Tx, 1000 subcarriers
    (ragged frequency tile), element-indexed and synthetic arrays; through the
    path-order SIMT contraction (dmma_min -1) and the FP64 tensor-core one (0, and
    the default threshold 16)."""
    from paper_2504_21719_b200 import _native
    _native.check(_native.lib().sbr_set_cfr_dmma_min_paths(dmma_min))
    try:
        _cfr_many_paths(synthetic)
    finally:
        _native.check(_native.lib().sbr_set_cfr_dmma_min_paths(16))


def _cfr_many_paths(synthetic):
    import types
    import oracle
    from paper_2504_21719_b200.cir import channel_response
    from paper_2504_21719_b200.em import planar_array
    rng = np.random.default_rng(7)
    n = 300
    lam = 299792458.0 / 3.5e9
    d = rng.normal(size=(n, 3)); d /= np.linalg.norm(d, axis=1, keepdims=True)
    a = rng.normal(size=(n, 3)); a /= np.linalg.norm(a, axis=1, keepdims=True)
    paths = {"tx": np.zeros(n, np.int64), "rx": np.zeros(n, np.int64),
             "gain": (rng.normal(size=n) + 1j * rng.normal(size=n)) * 1e-4,
             "delay": rng.uniform(1e-8, 3e-6, n), "departure": d, "arrival": a,
             "rx_el": rng.integers(0, 16, n), "tx_el": rng.integers(0, 64, n)}
    txo = planar_array(8, 8, lam / 2, lam / 2).offsets
    rxo = planar_array(4, 4, lam / 2, lam / 2).offsets
    freqs = 3.5e9 + (np.arange(1000) - 500) * 30e3
    H = channel_response(paths["gain"], paths["delay"], d, a, freqs, txo, rxo, lam,
                         synthetic=synthetic, rx_el=paths["rx_el"], tx_el=paths["tx_el"])
    cfg = types.SimpleNamespace(wavelength=lam, synthetic_arrays=synthetic)
    dev = lambda o: types.SimpleNamespace(array=types.SimpleNamespace(offsets=o))  # noqa
    want = oracle.frequency_response(paths, cfg, dev(txo), dev(rxo), freqs)
    assert H.shape == (16, 64, 1000)
    # same products, same path order: only libm sin/cos ulps differ
    assert np.abs(H - want).max() / np.abs(want).max() < 1e-12
