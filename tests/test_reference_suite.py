"""The reference's own unit tests for the hot path, restated against this API.

Each test states the behaviour of one test in emtrace's test-suite
(`pkg/tests/test_geometry.py`, `test_radiomap.py`, `test_paths.py`; cited per
test), on the same scenes and configurations, so a user moving from the
reference finds the same guarantees.  The host-side validation tests run on
CPU; everything that traces is `gpu`-marked and runs the CUDA path.
"""

import numpy as np
import pytest

from paper_2504_21719_b200 import (MeasurementGrid, Mesh, PathConfig, RadioDevice,
                                   RadioMapConfig, Ray, SceneModel, build_scene_accel,
                                   compute_paths, compute_radio_map_sbr,
                                   generate_candidates, intersect_closest, scenes)
from paper_2504_21719_b200.em import ArrayGeometry
from paper_2504_21719_b200.errors import UnresolvedMaterial
from paper_2504_21719_b200.materials import RadioMaterial
from paper_2504_21719_b200.sampling import Interaction

C0 = 299792458.0
BOX_LO, BOX_HI = np.array([-3.0, -4.0, 0.0]), np.array([3.0, 4.0, 3.0])
TX_POS, RX_POS = np.array([-1.0, -2.0, 1.5]), np.array([1.5, 2.0, 1.5])
CONCRETE = RadioMaterial("concrete", eps_r=5.24, sigma=0.1, thickness=0.3)
R_ONLY = frozenset({Interaction.REFLECTION})
RS = frozenset({Interaction.REFLECTION, Interaction.SCATTERING})


def _walled_room(material=CONCRETE):
    """Closed room, one object per wall (test_radiomap.py:48-66)."""
    (xl, yl, zl), (xh, yh, zh) = BOX_LO, BOX_HI
    quads = [
        ([xl, yl, zl], [xh, yl, zl], [xh, yh, zl], [xl, yh, zl]),
        ([xl, yl, zh], [xh, yl, zh], [xh, yh, zh], [xl, yh, zh]),
        ([xl, yl, zl], [xh, yl, zl], [xh, yl, zh], [xl, yl, zh]),
        ([xl, yh, zl], [xh, yh, zl], [xh, yh, zh], [xl, yh, zh]),
        ([xl, yl, zl], [xl, yh, zl], [xl, yh, zh], [xl, yl, zh]),
        ([xh, yl, zl], [xh, yh, zl], [xh, yh, zh], [xh, yl, zh]),
    ]
    meshes = [Mesh(np.array(q, dtype=np.float64), np.array([[0, 1, 2], [0, 2, 3]]), object_id=i + 1)
              for i, q in enumerate(quads)]
    return SceneModel(meshes, {i: material for i in range(1, 7)})


def _inward_room(material=CONCRETE):
    """One inward-facing box object (test_paths.py:53-55)."""
    return SceneModel([scenes.box_mesh(BOX_LO, BOX_HI, object_id=0, inward=True)], {0: material})


def _small_grid(cell=1.0, n=2):
    return MeasurementGrid((0.5, 1.0, 1.2), (1, 0, 0), (0, 1, 0), (cell, cell), (n, n))


# ---------------------------------------------------------------------------
# host-side validation (CPU)
# ---------------------------------------------------------------------------

def test_mesh_rejects_degenerate_triangle_and_bad_index():
    # test_geometry.py:16-25
    with pytest.raises(ValueError):
        Mesh(np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], float), np.array([[0, 1, 2]]), object_id=0)
    with pytest.raises(ValueError):
        Mesh(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float), np.array([[0, 1, 3]]), object_id=0)


def test_ray_requires_unit_direction():
    # test_geometry.py:28-30
    with pytest.raises(ValueError):
        Ray(np.zeros(3), np.array([0.0, 0.0, 2.0]))


def test_grid_validation_messages():
    # test_radiomap.py:106-114
    with pytest.raises(ValueError, match="unit"):
        MeasurementGrid((0, 0, 0), (2, 0, 0), (0, 1, 0), (1, 1), (2, 2))
    with pytest.raises(ValueError, match="orthogonal"):
        MeasurementGrid((0, 0, 0), (1, 0, 0), (1, 0, 0), (1, 1), (2, 2))
    with pytest.raises(ValueError, match="cell size"):
        MeasurementGrid((0, 0, 0), (1, 0, 0), (0, 1, 0), (0.0, 1), (2, 2))
    with pytest.raises(ValueError, match="shape"):
        MeasurementGrid((0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1), (0, 2))


def test_unresolved_material_raises_before_any_device_work():
    # test_paths.py:625-628
    mesh = scenes.box_mesh(BOX_LO, BOX_HI, object_id=3, inward=True)
    with pytest.raises(UnresolvedMaterial):
        SceneModel([mesh], {0: CONCRETE})


# ---------------------------------------------------------------------------
# closest hit (GPU)
# ---------------------------------------------------------------------------

@pytest.mark.gpu
def test_single_triangle_accel_bounds(cuda):
    # test_geometry.py:38-44
    acc = build_scene_accel([Mesh(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float),
                                  np.array([[0, 1, 2]]), object_id=0)])
    assert acc.num_triangles == 1
    lo, hi = acc.bounds
    assert np.allclose(lo, [0, 0, 0], atol=1e-9) and np.allclose(hi, [1, 1, 0], atol=1e-9)


@pytest.mark.gpu
def test_two_disjoint_boxes_nearer_first(cuda):
    # test_geometry.py:47-55
    acc = build_scene_accel([scenes.box_mesh([0, 0, 0], [1, 1, 1], object_id=0),
                             scenes.box_mesh([3, 0, 0], [4, 1, 1], object_id=1)])
    assert acc.num_triangles == 24
    h = intersect_closest(acc, Ray(np.array([-2.0, 0.5, 0.5]), np.array([1.0, 0.0, 0.0])))
    assert h.object_id == 0
    assert h.t == pytest.approx(2.0, abs=1e-12)


@pytest.mark.gpu
def test_ground_plane_hit_and_cap(cuda):
    # test_geometry.py:58-66
    acc = build_scene_accel([scenes.quad_mesh()])
    ray = Ray(np.array([0.0, 0.0, 1.0]), np.array([0.0, 0.0, -1.0]))
    h = intersect_closest(acc, ray)
    assert h.t == pytest.approx(1.0, abs=1e-12)
    assert np.allclose(h.point, [0, 0, 0], atol=1e-12)
    assert np.allclose(h.normal, [0, 0, 1])
    assert intersect_closest(acc, Ray(ray.origin, ray.direction, max_t=0.5)) is None


@pytest.mark.gpu
def test_shared_diagonal_tie_breaks_to_lower_primitive(cuda):
    # test_geometry.py:69-74: (0.5, 0.5) lies on the diagonal both triangles own
    acc = build_scene_accel([scenes.quad_mesh()])
    h = intersect_closest(acc, Ray(np.array([0.5, 0.5, 2.0]), np.array([0.0, 0.0, -1.0])))
    assert (h.object_id, h.primitive_id) == (0, 0)


@pytest.mark.gpu
def test_normal_faces_incident_side(cuda):
    # test_geometry.py:77-81
    acc = build_scene_accel([scenes.quad_mesh()])
    below = intersect_closest(acc, Ray(np.array([0.2, 0.1, -1.0]), np.array([0.0, 0.0, 1.0])))
    assert np.allclose(below.normal, [0, 0, -1])


@pytest.mark.gpu
def test_hit_point_consistency(cuda):
    # test_geometry.py:144-156 (hypothesis, 50 examples over px, py in
    # [-0.9, 0.9], tilt in [-0.45, 0.45]): 50 seeded draws plus the box corners
    rng = np.random.default_rng(144)
    draws = np.column_stack([rng.uniform(-0.9, 0.9, 50), rng.uniform(-0.9, 0.9, 50),
                             rng.uniform(-0.45, 0.45, 50)])
    corners = np.array([[a, b, c] for a in (-0.9, 0.9) for b in (-0.9, 0.9) for c in (-0.45, 0.45)])
    acc = build_scene_accel([scenes.quad_mesh()])
    hits = 0
    for px, py, tilt in np.vstack([draws, corners, [[0.0, 0.0, 0.0]]]):
        d = np.array([tilt, tilt / 2, -1.0])
        d /= np.linalg.norm(d)
        o = np.array([px, py, 1.0])
        h = intersect_closest(acc, Ray(o, d))
        if h is None:
            continue
        hits += 1
        assert float(h.normal @ d) <= 0.0
        assert np.linalg.norm(h.point - (o + h.t * d)) <= 1e-6 * max(h.t, 1.0)
    assert hits > 40


# ---------------------------------------------------------------------------
# radio map (GPU)
# ---------------------------------------------------------------------------

@pytest.mark.gpu
def test_bounce_map_matches_path_solver(cuda):
    # test_radiomap.py:258-278: cell averages agree with the non-coherent sum
    # over refined paths to the cell centres
    scene = _walled_room()
    grid = _small_grid(cell=0.5)
    vals, diag = compute_radio_map_sbr(scene, TX_POS, grid,
                                       RadioMapConfig(num_samples=800_000, max_depth=3,
                                                      enabled=R_ONLY, seed=0))
    assert diag["deposits"] > 0
    centers = grid.cell_centers().reshape(-1, 3)
    result = compute_paths(scene, [RadioDevice(position=TX_POS)],
                           [RadioDevice(position=c) for c in centers],
                           PathConfig(num_samples=120_000, max_depth=3, enabled=R_ONLY,
                                      q_diffraction=0.0, seed=0))
    truth = np.zeros(len(centers))
    for p in result.paths:
        truth[p.rx_index] += abs(p.gain) ** 2
    truth = truth.reshape(grid.shape[1], grid.shape[0])
    assert np.all(truth > 0.0)
    assert np.max(np.abs(vals - truth) / truth) < 0.06


@pytest.mark.gpu
def test_culling_counters_and_threshold_bias(cuda):
    # test_radiomap.py:299-319
    scene, grid = _walled_room(), _small_grid()
    kw = dict(num_samples=100_000, max_depth=3, enabled=RS, seed=1)
    v0, d0 = compute_radio_map_sbr(scene, TX_POS, grid, RadioMapConfig(**kw))
    assert d0.get("threshold_killed", 0) == 0 and d0.get("roulette_killed", 0) == 0
    _, d1 = compute_radio_map_sbr(scene, TX_POS, grid, RadioMapConfig(rr_depth=1, rr_max=0.9, **kw))
    assert d1["roulette_killed"] > 0
    v2, d2 = compute_radio_map_sbr(scene, TX_POS, grid, RadioMapConfig(gain_threshold=1e-3, **kw))
    assert d2["threshold_killed"] > 0
    assert np.all(v2 <= v0 + 1e-18)  # the threshold only removes energy


@pytest.mark.gpu
def test_roulette_stays_close_to_plain_estimate(cuda):
    # test_radiomap.py:322-332
    scene, grid = _walled_room(), _small_grid()
    kw = dict(num_samples=400_000, max_depth=3, enabled=RS, seed=7)
    v0, _ = compute_radio_map_sbr(scene, TX_POS, grid, RadioMapConfig(**kw))
    v1, _ = compute_radio_map_sbr(scene, TX_POS, grid, RadioMapConfig(rr_depth=1, rr_max=0.9, **kw))
    assert v1.sum() == pytest.approx(v0.sum(), rel=0.12)


# ---------------------------------------------------------------------------
# path solver (GPU)
# ---------------------------------------------------------------------------

@pytest.mark.gpu
def test_specular_paths_invariant_to_extra_interactions(cuda):
    # test_paths.py:548-574: enabling S and T does not change the pure-R paths
    rough = RadioMaterial("rough", eps_r=5.24, sigma=0.1, thickness=0.3, scattering=0.4)
    scene = _inward_room(rough)
    tx, rx = [RadioDevice(position=TX_POS)], [RadioDevice(position=RX_POS)]
    only_r = compute_paths(scene, tx, rx, PathConfig(num_samples=12000, max_depth=2, seed=3,
                                                     q_diffraction=0.0, enabled=R_ONLY))
    everything = compute_paths(scene, tx, rx, PathConfig(num_samples=12000, max_depth=2, seed=3,
                                                         q_diffraction=0.0))
    pure = {p.chain_hash: p for p in everything.paths if set(p.kinds) <= {"R"}}
    assert len(pure) == len(only_r.paths) > 0
    for p in only_r.paths:
        q = pure[p.chain_hash]
        assert q.gain == pytest.approx(p.gain, rel=1e-12)
        assert q.delay == pytest.approx(p.delay, rel=1e-12)
        np.testing.assert_allclose(q.vertices, p.vertices, atol=1e-9)


@pytest.mark.gpu
def test_depth_limited_run_has_no_deeper_paths(cuda):
    # test_paths.py:577-582
    ps = compute_paths(_inward_room(), [RadioDevice(position=TX_POS)], [RadioDevice(position=RX_POS)],
                       PathConfig(num_samples=20000, max_depth=1, enabled=R_ONLY, q_diffraction=0.0))
    assert {p.depth for p in ps.paths} == {0, 1}


@pytest.mark.gpu
def test_all_rows_terminate_when_nothing_enabled_applies(cuda):
    # test_paths.py:585-593: diffraction alone in a wedge-free room
    cfg = PathConfig(num_samples=2000, max_depth=2, seed=0, q_diffraction=0.2,
                     enabled=frozenset({Interaction.DIFFRACTION}))
    result = generate_candidates(_inward_room(), TX_POS, RX_POS[None, :], cfg)
    assert all(not r.steps for r in result.records)
    assert result.diagnostics["samples_terminated"] == 2000


@pytest.mark.gpu
def test_buffer_capacity_keeps_the_first_candidates(cuda):
    # test_paths.py:596-609
    scene = _inward_room()
    kw = dict(num_samples=30000, max_depth=2, enabled=R_ONLY, q_diffraction=0.0)
    capped = generate_candidates(scene, TX_POS, RX_POS[None, :], PathConfig(buffer_capacity=3, **kw))
    free = generate_candidates(scene, TX_POS, RX_POS[None, :], PathConfig(**kw))
    assert len(capped.records) == 3
    assert capped.diagnostics["buffer_overflow"] > 0
    assert [r.chain_hash for r in capped.records] == [r.chain_hash for r in free.records[:3]]


@pytest.mark.gpu
def test_per_element_tracing_offsets_sources(cuda):
    # test_paths.py:701-714: synthetic_arrays=False traces every element
    offsets = np.array([[0.0, 0.0, 0.0], [0.0, 0.0, 0.2]])
    tx = RadioDevice(position=TX_POS, array=ArrayGeometry(offsets))
    cfg = PathConfig(num_samples=1000, max_depth=0, enabled=R_ONLY, q_diffraction=0.0,
                     synthetic_arrays=False)
    ps = compute_paths(_inward_room(), [tx], [RadioDevice(position=RX_POS)], cfg)
    assert sorted(p.tx_element for p in ps.paths) == [0, 1]
    for p in ps.paths:
        dist = float(np.linalg.norm(RX_POS - (TX_POS + offsets[p.tx_element])))
        assert p.delay == pytest.approx(dist / C0, rel=1e-12)


# ---------------------------------------------------------------------------
# launch lattice and random streams (GPU; test_sampling.py)
# ---------------------------------------------------------------------------

def _fib(n, begin=0, end=None):
    from paper_2504_21719_b200.sampling import fibonacci_directions
    return fibonacci_directions(n, begin, end).cpu().numpy()


@pytest.mark.gpu
def test_fibonacci_single_point_and_rejects_empty(cuda):
    # test_sampling.py:32-35, 65-67: n = 0 sits at polar angle pi/2, azimuth 0
    np.testing.assert_allclose(_fib(1), [[1.0, 0.0, 0.0]], atol=1e-15)
    with pytest.raises(ValueError):
        _fib(0)


@pytest.mark.gpu
@pytest.mark.parametrize("count", [2, 17, 1000])
def test_fibonacci_unit_norms(cuda, count):
    # test_sampling.py:38-42
    d = _fib(count)
    assert d.shape == (count, 3)
    np.testing.assert_allclose(np.linalg.norm(d, axis=1), 1.0, atol=1e-12)


@pytest.mark.gpu
def test_fibonacci_near_uniform_and_deterministic(cuda):
    # test_sampling.py:45-47, 61-62
    assert np.linalg.norm(_fib(10 ** 4).mean(axis=0)) < 0.02
    assert np.array_equal(_fib(257), _fib(257))


@pytest.mark.gpu
@pytest.mark.parametrize("count", [100, 1000, 10000])
def test_fibonacci_no_large_holes(cuda, count):
    # test_sampling.py:50-58: no direction is isolated far beyond the mean spacing
    from scipy.spatial import cKDTree
    d = _fib(count)
    dist, _ = cKDTree(d).query(d, k=2)
    gap = 2.0 * np.arcsin(np.clip(dist[:, 1] / 2.0, 0.0, 1.0))
    assert gap.max() <= 4.0 * gap.mean()


@pytest.mark.gpu
def test_fibonacci_slices_are_the_full_lattice(cuda):
    # shards and passes evaluate [begin, end) of one lattice: any slicing
    # reproduces the full evaluation bit for bit
    full = _fib(4099)
    for lo, hi in ((0, 1), (1, 4099), (1000, 1001), (2048, 4099), (17, 3000)):
        assert np.array_equal(_fib(4099, lo, hi), full[lo:hi])


def _draws(seed, sample, depth, purpose, count, first=0):
    from paper_2504_21719_b200.sampling import rng_uniform
    return rng_uniform(seed, sample, depth, purpose, count, first).cpu().numpy()


@pytest.mark.gpu
def test_stream_reproducible_and_distinct_ids(cuda):
    # test_sampling.py:240-256
    ref = _draws(42, 13, 2, "interaction", 100)
    assert np.array_equal(ref, _draws(42, 13, 2, "interaction", 100))
    for other in (_draws(43, 13, 2, "interaction", 10), _draws(42, 14, 2, "interaction", 10),
                  _draws(42, 13, 3, "interaction", 10), _draws(42, 13, 2, "hemisphere", 10)):
        assert not np.array_equal(ref[:10], other)


@pytest.mark.gpu
def test_stream_order_and_offset_independence(cuda):
    # test_sampling.py:259-271: a stream's draws never depend on which streams
    # ran first; on the device the draws are stateless, so any sub-range of a
    # stream equals the same slice of the whole stream
    serial = [_draws(5, i, 0, "interaction", 16) for i in range(8)]
    shuffled = {i: _draws(5, i, 0, "interaction", 16) for i in (5, 2, 7, 0, 6, 1, 4, 3)}
    for i in range(8):
        assert np.array_equal(serial[i], shuffled[i])
        for first, count in ((0, 1), (3, 5), (4, 12), (15, 1)):
            assert np.array_equal(_draws(5, i, 0, "interaction", count, first),
                                  serial[i][first:first + count])


# ---------------------------------------------------------------------------
# box room against closed-form answers (GPU; test_paths.py:92-407, 612-622)
# ---------------------------------------------------------------------------

WALLS = [(a, v) for a in range(3) for v in (BOX_LO[a], BOX_HI[a])]


def _mirror_paths(tx, rx, max_depth):
    """Image-method enumeration of the specular paths inside the box: every
    wall sequence without immediate repeats whose back-traced reflection
    points land strictly inside their walls, in order (the room is convex,
    so nothing else can block them).  Returns {depth: [unfolded length]}."""
    out = {0: [float(np.linalg.norm(rx - tx))]}

    def extend(chain, images):
        if chain:
            p_next, ok = rx, True
            for (a, v), img in zip(reversed(chain), reversed(images)):
                den = p_next[a] - img[a]
                t = (v - img[a]) / den if den != 0.0 else -1.0
                if not 1e-9 < t < 1.0 - 1e-9:
                    ok = False
                    break
                p = img + t * (p_next - img)
                others = [b for b in range(3) if b != a]
                if any(not BOX_LO[b] + 1e-9 < p[b] < BOX_HI[b] - 1e-9 for b in others):
                    ok = False
                    break
                p_next = p
            if ok:
                out.setdefault(len(chain), []).append(float(np.linalg.norm(rx - images[-1])))
        if len(chain) == max_depth:
            return
        last = images[-1] if images else tx
        for w in WALLS:
            if chain and w == chain[-1]:
                continue
            img = last.copy()
            img[w[0]] = 2.0 * w[1] - img[w[0]]
            extend(chain + [w], images + [img])

    extend([], [])
    return out


@pytest.fixture(scope="module")
def box_paths():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = PathConfig(num_samples=120_000, max_depth=3, enabled=R_ONLY, q_diffraction=0.0, seed=0)
    scene = _inward_room()
    return scene, cfg, compute_paths(scene, [RadioDevice(position=TX_POS)],
                                     [RadioDevice(position=RX_POS)], cfg)


@pytest.mark.gpu
def test_box_counts_and_delays_match_image_enumeration(box_paths):
    # test_paths.py:303-317
    _, _, ps = box_paths
    want = _mirror_paths(TX_POS, RX_POS, 3)
    found = {}
    for p in ps.paths:
        found.setdefault(p.depth, []).append(p.delay)
    assert set(found) == set(want)
    for depth, lengths in want.items():
        assert len(found[depth]) == len(lengths), f"depth {depth}"
        np.testing.assert_allclose(np.sort(found[depth]), np.sort(lengths) / C0, rtol=1e-9)


def _slab(cos0, eta, thickness, lam, pol):
    """ITU-R P.2040 slab over vacuum, one polarization (materials.py:163-238)."""
    root = np.sqrt(complex(eta) - (1.0 - cos0 * cos0))
    if root.imag > 0.0:
        root = -root
    r = (cos0 - root) / (cos0 + root) if pol == "perp" else \
        (eta * cos0 - root) / (eta * cos0 + root)
    q = 2.0 * np.pi * thickness / lam * root
    p2, p1 = np.exp(-2j * q), np.exp(-1j * q)
    den = 1.0 - r * r * p2
    return r * (1.0 - p2) / den, (1.0 - r * r) * p1 / den


@pytest.mark.gpu
def test_box_single_bounce_gains_analytic(box_paths):
    # test_paths.py:337-376: devices at equal height, so a floor / ceiling
    # bounce is purely parallel and a side-wall bounce purely perpendicular
    _, cfg, ps = box_paths
    lam = cfg.wavelength
    eta = CONCRETE.complex_permittivity(cfg.frequency)
    singles = [p for p in ps.paths if p.depth == 1]
    assert len(singles) == 6
    for axis, value in WALLS:
        image = TX_POS.copy()
        image[axis] = 2.0 * value - image[axis]
        length = float(np.linalg.norm(RX_POS - image))
        r, _ = _slab(abs((RX_POS - image)[axis]) / length, eta, CONCRETE.thickness, lam,
                     "par" if axis == 2 else "perp")
        match = [p for p in singles if abs(p.delay - length / C0) < 1e-13
                 and abs(p.steps[0].vertex[axis] - value) < 1e-9]
        assert match, f"bounce off axis {axis} at {value} missing"
        for p in match:
            assert abs(p.gain) == pytest.approx(lam / (4.0 * np.pi * length) * abs(r), rel=1e-9)


@pytest.mark.gpu
def test_box_refinement_fixed_point(box_paths):
    # test_paths.py:379-389: refining a refined path returns it
    from paper_2504_21719_b200.cir import CandidateRecord, PathGeometry, refine_candidate
    scene, _, ps = box_paths
    for p in ps.paths[:20]:
        rec = CandidateRecord(source_id=0, target_id=0, source=TX_POS, target=RX_POS,
                              sample_id=p.sample_id, steps=p.steps, suffix_start=0,
                              anchor=TX_POS, prefix_probability=1.0, chain_hash=p.chain_hash)
        again = refine_candidate(rec, scene)
        assert isinstance(again, PathGeometry)
        np.testing.assert_allclose(again.vertices, p.vertices, atol=1e-9)


@pytest.mark.gpu
def test_refinement_rejects_plane_mismatch(cuda):
    # test_paths.py:392-406
    from paper_2504_21719_b200.cir import (CandidateRecord, InteractionStep, Rejection,
                                           refine_candidate)
    bogus = InteractionStep(kind=Interaction.REFLECTION, object_id=0, primitive_id=0,
                            vertex=np.array([0.0, 0.0, 0.0]), normal=np.array([1.0, 0.0, 0.0]))
    rec = CandidateRecord(source_id=0, target_id=0, source=TX_POS, target=RX_POS, sample_id=0,
                          steps=(bogus,), suffix_start=0, anchor=TX_POS, prefix_probability=1.0,
                          chain_hash=0)
    out = refine_candidate(rec, _inward_room())
    assert isinstance(out, Rejection) and out.reason == "coplanar-miss"


@pytest.mark.gpu
def test_doppler_static_scene_is_zero(box_paths):
    # test_paths.py:635-637
    assert all(p.doppler == 0.0 for p in box_paths[2].paths)


@pytest.mark.gpu
def test_generation_diagnostics_account_for_all_rows(cuda):
    # test_paths.py:612-622: closed room, reflection only -- every ray survives
    # both bounces and every bounce vertex sees the single target
    cfg = PathConfig(num_samples=5000, max_depth=2, enabled=R_ONLY, q_diffraction=0.0, seed=0)
    diag = generate_candidates(_inward_room(), TX_POS, RX_POS[None, :], cfg).diagnostics
    assert diag["samples_escaped"] == 0
    assert diag["duplicates"] + (diag["hash_registered"] - 1) == 2 * 5000
    assert diag["candidates"] == diag["hash_registered"]


@pytest.mark.gpu
def test_worker_counts_give_identical_paths(cuda):
    # test_paths.py:513-533: the reference's worker pool is a host knob; the
    # device result must not depend on it either
    rough = RadioMaterial("rough", eps_r=5.24, sigma=0.1, thickness=0.3, scattering=0.15)
    scene = _inward_room(rough)
    tx, rx = [RadioDevice(position=TX_POS)], [RadioDevice(position=RX_POS)]
    runs = [compute_paths(scene, tx, rx, PathConfig(num_samples=8000, max_depth=3, seed=7,
                                                    q_diffraction=0.0, workers=w))
            for w in (1, 2, 4)]
    base = runs[0]
    assert any(p.kinds and "S" in p.kinds for p in base.paths)
    for other in runs[1:]:
        assert len(other.paths) == len(base.paths)
        for a, b in zip(base.paths, other.paths):
            assert a.gain == b.gain and a.delay == b.delay and a.sample_id == b.sample_id
            assert np.array_equal(a.vertices, b.vertices)
        assert other.diagnostics == base.diagnostics


# ---------------------------------------------------------------------------
# grid and configuration (host; test_radiomap.py:117-177)
# ---------------------------------------------------------------------------

def test_grid_geometry():
    g = MeasurementGrid((1.0, 2.0, 3.0), (1, 0, 0), (0, 1, 0), (0.5, 0.25), (4, 8))
    assert np.allclose(g.normal, [0, 0, 1])
    assert g.cell_area == pytest.approx(0.125)
    assert np.allclose(g.corner, [0.0, 1.0, 3.0])
    c = g.cell_centers()
    assert c.shape == (8, 4, 3)
    assert np.allclose(c[0, 0], [0.25, 1.125, 3.0]) and np.allclose(c[-1, -1], [1.75, 2.875, 3.0])
    h = MeasurementGrid.horizontal((0, 0, 1.5), (10.0, 6.0), (2.0, 2.0))
    assert h.shape == (5, 3) and np.allclose(h.normal, [0, 0, 1])


def test_cell_lookup_boundaries_go_to_the_higher_cell():
    g = MeasurementGrid((0.0, 0.0, 2.0), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (2, 2))
    assert g.cell_lookup((0.0, 0.0, 2.0)) == (1, 1)
    assert g.cell_lookup((-0.5, -0.5, 2.0)) == (0, 0)
    assert g.cell_lookup((0.999, 0.2, 2.0)) == (1, 1)
    assert g.cell_lookup((1.001, 0.0, 2.0)) is None
    assert g.cell_lookup((0.0, 0.0, 2.1)) is None


def test_config_validation_and_roulette_probability():
    from paper_2504_21719_b200.radiomap import russian_roulette_probability
    for kw in (dict(num_samples=0), dict(rr_max=0.0), dict(rr_depth=4, max_depth=3),
               dict(gain_threshold=-1.0)):
        with pytest.raises(ValueError):
            RadioMapConfig(**kw)
    assert RadioMapConfig(frequency=3.5e9).wavelength == pytest.approx(C0 / 3.5e9)
    assert russian_roulette_probability(2.0, 0.01, 0.95) == pytest.approx(0.04)
    assert russian_roulette_probability(10.0, 1.0, 0.95) == 0.95


# ---------------------------------------------------------------------------
# screen: occlusion, transmission, diffraction (GPU; test_paths.py:432-510,
# test_radiomap.py:244-255)
# ---------------------------------------------------------------------------

def _screen_scene():
    """Vertical 4 m square screen in the y = 0 plane, x in [-2, 2], z in [0, 4]."""
    quad = scenes.quad_mesh(half=2.0, z=0.0, object_id=5)
    swap = np.array([[1.0, 0, 0], [0, 0, 1.0], [0, 1.0, 0]])
    mesh = Mesh(quad.vertices @ swap + np.array([0.0, 0.0, 2.0]), quad.triangles, object_id=5)
    return SceneModel([mesh], {5: CONCRETE})


SCREEN_TX, SCREEN_RX = np.array([0.0, -3.0, 2.0]), np.array([0.0, 3.0, 2.5])


@pytest.fixture(scope="module")
def screen_paths():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    scene = _screen_scene()
    cfg = PathConfig(num_samples=150_000, max_depth=1, seed=0, q_diffraction=0.3)
    return scene, cfg, compute_paths(scene, [RadioDevice(position=SCREEN_TX)],
                                     [RadioDevice(position=SCREEN_RX)], cfg)


@pytest.mark.gpu
def test_screen_blocks_los_and_transmits(screen_paths):
    _, cfg, ps = screen_paths
    kinds = sorted(p.kinds for p in ps.paths)
    assert "" not in kinds, "blocked line of sight must not appear"
    assert kinds.count("T") == 1 and kinds.count("D") == 4
    t_path = next(p for p in ps.paths if p.kinds == "T")
    a, m, b = t_path.vertices
    assert np.linalg.norm(np.cross(b - a, m - a)) < 1e-9  # straight through
    dist = float(np.linalg.norm(b - a))
    assert t_path.delay == pytest.approx(dist / C0, rel=1e-12)
    # the ray runs in the x = 0 plane, the incidence plane of the y = 0 screen:
    # a zenith-referenced pattern is purely parallel
    _, t_par = _slab(abs((b - a)[1]) / dist, CONCRETE.complex_permittivity(cfg.frequency),
                     CONCRETE.thickness, cfg.wavelength, "par")
    assert abs(t_path.gain) == pytest.approx(cfg.wavelength / (4.0 * np.pi * dist) * abs(t_par),
                                             rel=1e-9)


@pytest.mark.gpu
def test_screen_diffraction_points_minimize_length(screen_paths):
    from scipy.optimize import minimize_scalar
    scene, _, ps = screen_paths
    d_paths = [p for p in ps.paths if p.kinds == "D"]
    assert len(d_paths) == 4
    for p in d_paths:
        w = scene.wedges[p.steps[0].wedge_index]
        v = p.vertices[1]
        x = float((v - w.origin) @ w.e_hat)
        length = lambda s: (np.linalg.norm(w.origin + s * w.e_hat - SCREEN_TX)  # noqa: E731
                            + np.linalg.norm(SCREEN_RX - w.origin - s * w.e_hat))
        ref = minimize_scalar(length, bounds=(0.0, w.length), method="bounded",
                              options={"xatol": 1e-10}).x
        assert x == pytest.approx(ref, abs=1e-6)
        k_in, k_out = v - SCREEN_TX, SCREEN_RX - v
        k_in, k_out = k_in / np.linalg.norm(k_in), k_out / np.linalg.norm(k_out)
        assert k_in @ w.e_hat == pytest.approx(k_out @ w.e_hat, abs=1e-9)  # Keller cone


@pytest.mark.gpu
def test_off_edge_diffraction_rejected(cuda):
    from paper_2504_21719_b200.cir import (CandidateRecord, InteractionStep, Rejection,
                                           refine_candidate)
    scene = _screen_scene()
    top = next(i for i, w in enumerate(scene.wedges)
               if abs(w.origin[2] - 4.0) < 1e-9 and abs(w.e_hat[2]) < 1e-9)
    w = scene.wedges[top]
    source, target = np.array([40.0, -3.0, 6.0]), np.array([41.0, 3.0, 7.0])  # far beyond +x
    step = InteractionStep(kind=Interaction.DIFFRACTION, object_id=5, primitive_id=0,
                           vertex=w.point_at(w.length), normal=w.n0_hat, wedge_index=top)
    rec = CandidateRecord(source_id=0, target_id=0, source=source, target=target, sample_id=0,
                          steps=(step,), suffix_start=0, anchor=source, prefix_probability=1.0,
                          chain_hash=0)
    out = refine_candidate(rec, scene)
    assert isinstance(out, Rejection) and out.reason == "off-edge"


@pytest.mark.gpu
def test_direct_term_respects_occlusion(cuda):
    # test_radiomap.py:244-255: with no bounces the map is the analytic direct
    # term; the screen's shadow is empty, the outer columns see the source
    grid = MeasurementGrid((0.0, 2.0, 1.0), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (10, 2))
    vals, _ = compute_radio_map_sbr(_screen_scene(), np.array([0.0, -3.0, 2.5]), grid,
                                    RadioMapConfig(num_samples=1, max_depth=0))
    shadowed = vals == 0.0
    assert shadowed.any() and (~shadowed).any()
    assert vals[0, 0] > 0.0 and vals[0, 5] == 0.0


# ---------------------------------------------------------------------------
# edge (diffraction) map (GPU; test_radiomap.py:353-373, 502-538)
# ---------------------------------------------------------------------------

@pytest.mark.gpu
def test_collect_wedges_radius_and_visibility(cuda):
    from paper_2504_21719_b200.radiomap import collect_wedges_near_source
    scene = _screen_scene()
    assert len(scene.wedges) == 4
    everything = collect_wedges_near_source(scene, SCREEN_TX, 100.0)
    assert sorted(everything) == [0, 1, 2, 3]
    # a point hovering just off the bottom edge keeps only that wedge
    lows = [wi for wi in everything if abs(scene.wedges[wi].origin[2]) < 1e-9
            and abs(scene.wedges[wi].e_hat[2]) < 0.5]
    assert collect_wedges_near_source(scene, np.array([0.0, -0.4, 0.0]), 0.5) == lows
    # a cage around the source hides the screen's wedges (its own stay visible)
    cage = scenes.box_mesh(SCREEN_TX - 0.2, SCREEN_TX + 0.2, object_id=9)
    caged = SceneModel([scene.meshes[0], cage], {5: CONCRETE, 9: CONCRETE})
    kept = collect_wedges_near_source(caged, SCREEN_TX, 100.0)
    screen_wedges = [wi for wi, w in enumerate(caged.wedges)
                     if abs(w.origin[1]) < 1e-9 and abs(w.e_hat[1]) < 1e-9 and wi < 4]
    assert screen_wedges and not set(kept) & set(screen_wedges)


@pytest.mark.gpu
def test_edge_map_worker_determinism(cuda):
    # test_radiomap.py:517-527: bitwise-equal maps for 1 and 4 workers (with
    # exact_maps the cells accumulate in fixed point: deposit order is moot)
    from paper_2504_21719_b200 import compute_radio_map_diffraction
    from paper_2504_21719_b200.radiomap import exact_maps
    scene = _screen_scene()
    grid = MeasurementGrid((0.25, 2.25, 1.7), (1, 0, 0), (0, 1, 0), (0.5, 0.5), (1, 1))
    with exact_maps():
        runs = [compute_radio_map_diffraction(scene, SCREEN_TX, grid, [0, 1, 2, 3],
                                              RadioMapConfig(workers=w, wedge_samples=100_000,
                                                             seed=2))
                for w in (1, 4)]
    assert runs[0][1] == runs[1][1]
    assert np.array_equal(runs[0][0], runs[1][0])
    assert runs[0][0][0, 0] > 0.0


@pytest.mark.gpu
def test_bounce_map_worker_determinism(cuda):
    # test_radiomap.py:335-346
    from paper_2504_21719_b200.radiomap import exact_maps
    scene = _walled_room()
    grid = _small_grid(cell=0.5)
    with exact_maps():
        runs = [compute_radio_map_sbr(scene, TX_POS, grid,
                                      RadioMapConfig(workers=w, num_samples=40_000, max_depth=2,
                                                     enabled=RS, seed=5)) for w in (1, 3)]
    assert runs[0][1] == runs[1][1]
    assert np.array_equal(runs[0][0], runs[1][0])


@pytest.mark.gpu
def test_compute_radio_map_multi_source_with_diffraction(cuda):
    from paper_2504_21719_b200 import compute_radio_map
    scene = _screen_scene()
    grid = MeasurementGrid((0.0, 2.0, 1.0), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (2, 2))
    cfg = RadioMapConfig(num_samples=20_000, wedge_samples=20_000, max_depth=1, seed=0)
    sources = [np.array([0.0, -3.0, 2.5]), RadioDevice(position=(1.0, -2.0, 2.5))]
    res = compute_radio_map(scene, sources, grid, cfg)
    assert res.values.shape == (2, 2, 2)
    assert np.allclose(res.total(), res.values.sum(axis=0))
    assert len(res.diagnostics) == 2 and res.diagnostics[0]["wedges"] == 4
    plain = compute_radio_map(scene, sources[:1], grid,
                              RadioMapConfig(num_samples=20_000, max_depth=1, enabled=RS))
    assert "wedges" not in plain.diagnostics[0]
    with pytest.raises(ValueError, match="precoder"):
        compute_radio_map(scene, sources, grid, cfg, precoders=[[1.0]])


# ---------------------------------------------------------------------------
# DedupTable / PathBuffer semantics of the device selection (GPU;
# test_paths.py:175-202): crafted rows straight into sbr_cir_select
# ---------------------------------------------------------------------------

def _select(pairs, n_hash, n_buffer=16):
    """Chain rows (pair_r, pair_f) in this ordinal order at depth 1, one
    target whose line of sight is blocked -> (selected row indices, counters)."""
    import torch
    from paper_2504_21719_b200 import _abi
    from paper_2504_21719_b200.cir import _cir_params, _select_rows
    dev = torch.device("cuda", 0)
    n = len(pairs)
    cfg = PathConfig(num_samples=max(n, 1), max_depth=1, enabled=R_ONLY, q_diffraction=0.0,
                     hash_capacity=n_hash, buffer_capacity=n_buffer)
    tgt = torch.zeros((1, 3), dtype=torch.float64, device=dev)
    params = _cir_params(np.zeros(3), tgt, cfg)
    key = torch.tensor([(1 << 60) | (i << 20) for i in range(n)], dtype=torch.int64,
                       device=dev).view(torch.uint64)
    as_u64 = lambda v: torch.tensor(np.array(v, dtype=np.uint64).view(np.int64),  # noqa: E731
                                    device=dev).view(torch.uint64)
    pr, pf = as_u64([p[0] for p in pairs]), as_u64([p[1] for p in pairs])
    chain = torch.ones(n, dtype=torch.uint8, device=dev)
    los = torch.zeros(1, dtype=torch.uint8, device=dev)
    counters = torch.zeros(_abi.SBR_CC_COUNT, dtype=torch.int64, device=dev)
    rec_row, m = _select_rows(params, key, pr, pf, chain, n, los, cfg, counters, dev)
    c = counters.cpu().numpy()
    return rec_row[:m].cpu().tolist(), {k: int(c[i]) for k, i in _abi.CC.items()}


@pytest.mark.gpu
def test_dedup_registers_exactly_once(cuda):
    rows, c = _select([(11, 500), (11, 500)], n_hash=1024)
    assert rows == [0]
    assert c["hash_registered"] == 1 and c["duplicates"] == 1


@pytest.mark.gpu
def test_dedup_one_shared_slot_rejects(cuda):
    # capacity 100: (105, 207) lands on slots (5, 7), (5, 8) shares slot 5
    rows, c = _select([(5, 7), (105, 207), (5, 8)], n_hash=100)
    assert rows == [0] and c["hash_registered"] == 1


@pytest.mark.gpu
def test_dedup_rejection_leaves_no_trace(cuda):
    # slot 9 appears in a rejected pair; a later pair must still claim it
    rows, c = _select([(5, 7), (5, 9), (9, 9)], n_hash=100)
    assert rows == [0, 2] and c["hash_registered"] == 2


@pytest.mark.gpu
def test_buffer_drops_on_overflow_keeps_first(cuda):
    # the first two are kept, the third dropped; within one chunk the
    # reference trims rows to the buffer's room before appending
    # (_emit_records paths.py:954-960), so it counts as chunk_truncated
    rows, c = _select([(1, 2), (3, 4), (5, 6)], n_hash=1024, n_buffer=2)
    assert rows == [0, 1]
    assert c["chunk_truncated"] == 1 and c["buffer_overflow"] == 0


# ---------------------------------------------------------------------------
# plane / chain hashing (test_paths.py:106-172): the host helpers on CPU, the
# per-slot plane hashes the device derives in sbr_scene_create on the GPU
# ---------------------------------------------------------------------------

def test_host_plane_hash_properties():
    from paper_2504_21719_b200.paths import hash_plane, pair_with_target
    rng = np.random.default_rng(122)
    for _ in range(20):
        n, p = rng.normal(size=3), rng.normal(size=3) * 10.0
        assert hash_plane(n, p) == hash_plane(-n, p)  # winding
    z = np.array([0.0, 0.0, 1.0])
    assert hash_plane(z, np.array([0.3, -0.7, 1.25])) == hash_plane(z, np.array([-5.0, 2.0, 1.25]))
    # noise at a quantizer boundary flips at most one of the two hashes
    r_lo, f_lo = hash_plane(z, np.array([0.0, 0.0, 1.5e-4 - 1e-9]))
    r_hi, f_hi = hash_plane(z, np.array([0.0, 0.0, 1.5e-4 + 1e-9]))
    assert r_lo != r_hi and f_lo == f_hi
    r_lo, f_lo = hash_plane(z, np.array([0.0, 0.0, 2.0e-4 - 1e-9]))
    r_hi, f_hi = hash_plane(z, np.array([0.0, 0.0, 2.0e-4 + 1e-9]))
    assert f_lo != f_hi and r_lo == r_hi
    assert len({pair_with_target(0x1234ABCD5678, k) for k in range(64)}) == 64


def _horizontal_tri(z, x0=0.0, y0=0.0, flip=False, object_id=0):
    v = np.array([[x0, y0, z], [x0 + 1.0, y0, z], [x0, y0 + 1.0, z]])
    t = np.array([[0, 2, 1]] if flip else [[0, 1, 2]])
    return Mesh(v, t, object_id=object_id)


def _device_plane_hashes(meshes):
    acc = build_scene_accel(meshes)
    _, hr, hf = acc._device_tables()
    return {int(acc.tri_object_id[s]): (int(hr[s]), int(hf[s])) for s in range(acc.num_triangles)}


@pytest.mark.gpu
def test_device_plane_hashes_ignore_winding_and_anchor(cuda):
    h = _device_plane_hashes([_horizontal_tri(1.25, object_id=0),
                              _horizontal_tri(1.25, flip=True, object_id=1),
                              _horizontal_tri(1.25, x0=-5.0, y0=2.0, object_id=2),
                              _horizontal_tri(1.30, object_id=3)])
    assert h[0] == h[1] == h[2]
    assert h[3][0] != h[0][0] and h[3][1] != h[0][1]


@pytest.mark.gpu
def test_device_plane_hashes_boundary_straddle(cuda):
    eps = 1e-9
    h = _device_plane_hashes([_horizontal_tri(1.5e-4 - eps, object_id=0),
                              _horizontal_tri(1.5e-4 + eps, object_id=1),
                              _horizontal_tri(2.0e-4 - eps, object_id=2),
                              _horizontal_tri(2.0e-4 + eps, object_id=3)])
    assert h[0][0] != h[1][0] and h[0][1] == h[1][1]  # half-cell: round flips
    assert h[2][1] != h[3][1] and h[2][0] == h[3][0]  # cell: floor flips


@pytest.mark.gpu
def test_map_bitwise_reproducible_across_runs_and_wave_streams(cuda):
    # a multi-pass map (3 wavefront passes) deposits from 1 or 2 streams in a
    # different order every run; with exact_maps the result is bitwise
    # identical anyway, and equals the float64-atomics map to 1e-12
    from paper_2504_21719_b200 import _native
    from paper_2504_21719_b200.radiomap import exact_maps
    scene = _walled_room()
    grid = MeasurementGrid((0.0, 0.0, 1.0), (1, 0, 0), (0, 1, 0), (0.5, 0.5), (10, 14))
    cfg = RadioMapConfig(num_samples=3 * (1 << 24) - 777, max_depth=2, enabled=RS, seed=9)
    plain, dplain = compute_radio_map_sbr(scene, TX_POS, grid, cfg)
    with exact_maps():
        ref, dref = compute_radio_map_sbr(scene, TX_POS, grid, cfg)
        again, dagain = compute_radio_map_sbr(scene, TX_POS, grid, cfg)
        try:
            _native.check(_native.lib().sbr_set_wave_streams(1))
            one, done_ = compute_radio_map_sbr(scene, TX_POS, grid, cfg)
        finally:
            _native.check(_native.lib().sbr_set_wave_streams(2))
    assert dplain == dref == dagain == done_
    assert np.array_equal(ref, again) and np.array_equal(ref, one)
    assert np.all(ref > 0)
    np.testing.assert_allclose(ref, plain, rtol=1e-12, atol=0.0)
