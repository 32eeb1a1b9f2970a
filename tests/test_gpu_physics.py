"""Physical / analytic behaviour of the public API on the GPU path.

Checks stated in closed form rather than against fixtures: free-space
delay and Friis gain, Doppler of moving devices and walls, the specular
law at refined bounce points, the CFR as an explicit per-path sum,
multi-source maps and the depth limit (the reference states the same
properties in its test-suite: test_paths.py / test_radiomap.py).
"""

import math

import numpy as np
import pytest

from paper_2504_21719_b200 import (MeasurementGrid, PathConfig, RadioDevice, RadioMapConfig,
                                   SceneModel, compute_paths, compute_radio_map,
                                   compute_radio_map_sbr, frequency_response, scenes)
from paper_2504_21719_b200.em import planar_array
from paper_2504_21719_b200.materials import RadioMaterial
from paper_2504_21719_b200.sampling import Interaction

pytestmark = pytest.mark.gpu

C0 = 299792458.0
LO, HI = np.array([-3.0, -4.0, 0.0]), np.array([3.0, 4.0, 3.0])
CONC = RadioMaterial("concrete", eps_r=5.24, sigma=0.1, thickness=0.3)
R = frozenset({Interaction.REFLECTION})


def _room(velocity=None):
    mesh = scenes.box_mesh(LO, HI, object_id=0, inward=True)
    return SceneModel([mesh], {0: CONC}, velocities=velocity)


def test_line_of_sight_delay_gain_and_directions(cuda):
    tx, rx = np.array([-1.0, -2.0, 1.5]), np.array([1.5, 2.0, 1.2])
    cfg = PathConfig(num_samples=1000, max_depth=0, enabled=R, q_diffraction=0.0)
    ps = compute_paths(_room(), [RadioDevice(position=tx)], [RadioDevice(position=rx)], cfg)
    (p,) = ps.paths
    d = float(np.linalg.norm(rx - tx))
    assert p.delay == pytest.approx(d / C0, rel=1e-12)
    assert abs(p.gain) == pytest.approx(cfg.wavelength / (4 * np.pi * d), rel=1e-9)
    k = (rx - tx) / d
    np.testing.assert_allclose(p.departure, k, atol=1e-12)
    np.testing.assert_allclose(p.arrival, k, atol=1e-12)
    assert p.doppler == 0.0


def test_doppler_of_moving_transmitter_and_wall(cuda):
    cfg0 = PathConfig(num_samples=1000, max_depth=0, enabled=R, q_diffraction=0.0)
    v = 10.0
    tx = RadioDevice(position=[-2.0, 0.0, 1.0], velocity=[v, 0.0, 0.0])
    (p,) = compute_paths(_room(), [tx], [RadioDevice(position=[2.0, 0.0, 1.0])], cfg0).paths
    assert p.doppler == pytest.approx(v / cfg0.wavelength, rel=1e-12)

    w = 5.0
    cfg1 = PathConfig(num_samples=60_000, max_depth=1, enabled=R, q_diffraction=0.0)
    ps = compute_paths(_room({0: [-w, 0.0, 0.0]}), [RadioDevice(position=[0.0, -1.0, 1.5])],
                       [RadioDevice(position=[0.0, 1.0, 1.5])], cfg1)
    hit = [q for q in ps.paths if q.depth == 1 and abs(q.vertices[1][0] - HI[0]) < 1e-9]
    assert hit
    k1 = np.array([3.0, 1.0, 0.0]) / math.sqrt(10.0)   # towards the +x wall at (3, 0, 1.5)
    k2 = np.array([-3.0, 1.0, 0.0]) / math.sqrt(10.0)
    want = float(np.array([-w, 0.0, 0.0]) @ (k2 - k1)) / cfg1.wavelength
    assert hit[0].doppler == pytest.approx(want, rel=1e-12)


def test_refined_bounces_obey_specular_law_and_depth_limit(cuda):
    cfg = PathConfig(num_samples=20_000, max_depth=2, enabled=R, q_diffraction=0.0)
    ps = compute_paths(_room(), [RadioDevice(position=[-1.0, -2.0, 1.5])],
                       [RadioDevice(position=[1.5, 2.0, 1.5])], cfg)
    assert ps.paths and max(p.depth for p in ps.paths) <= 2
    assert {p.depth for p in ps.paths} == {0, 1, 2}
    for p in ps.paths:
        v = np.asarray(p.vertices)
        for j, st in enumerate(p.steps):
            n = np.asarray(st.normal, dtype=np.float64)
            a = v[j + 1] - v[j]
            b = v[j + 2] - v[j + 1]
            a, b = a / np.linalg.norm(a), b / np.linalg.norm(b)
            np.testing.assert_allclose(b, a - 2 * (a @ n) * n, atol=1e-9)  # mirror law
        # delay = unfolded length / c
        length = np.linalg.norm(np.diff(v, axis=0), axis=1).sum()
        assert p.delay == pytest.approx(length / C0, rel=1e-12)


def test_more_samples_find_a_superset_of_specular_chains(cuda):
    tx, rx = [RadioDevice(position=[-1.0, -2.0, 1.5])], [RadioDevice(position=[1.5, 2.0, 1.5])]
    chains = []
    for n in (300, 20_000):
        cfg = PathConfig(num_samples=n, max_depth=3, enabled=R, q_diffraction=0.0)
        chains.append({p.chain_hash for p in compute_paths(_room(), tx, rx, cfg).paths})
    assert chains[0] <= chains[1] and len(chains[1]) > len(chains[0])


def test_frequency_response_is_the_per_path_sum(cuda):
    lam = C0 / 3.5e9
    tx = RadioDevice(position=np.array([-1.0, -2.0, 1.5]), array=planar_array(2, 2, lam / 2, lam / 2))
    rx = RadioDevice(position=np.array([1.5, 2.0, 1.5]), array=planar_array(1, 3, lam / 2, lam / 2))
    cfg = PathConfig(num_samples=10_000, max_depth=2, enabled=R, q_diffraction=0.0)
    ps = compute_paths(_room(), [tx], [rx], cfg)
    f = 3.5e9 + np.arange(-8, 8) * 1e6
    H = frequency_response(ps, f)
    want = np.zeros((3, 4, len(f)), complex)
    kw = 2 * np.pi / cfg.wavelength
    for p in ps.paths:
        u_t = np.exp(1j * kw * (tx.array.offsets @ p.departure))
        u_r = np.exp(1j * kw * (rx.array.offsets @ -p.arrival))
        want += p.gain * u_r[:, None, None] * u_t[None, :, None] * \
            np.exp(-2j * np.pi * f * p.delay)[None, None, :]
    assert np.abs(H - want).max() <= 1e-12 * np.abs(want).max()


def test_multi_source_map_layers_and_precoder_check(cuda):
    scene = _room()
    grid = MeasurementGrid((0.0, 0.0, 1.0), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (4, 6))
    cfg = RadioMapConfig(num_samples=50_000, max_depth=2, enabled=R, seed=3)
    srcs = [np.array([-1.0, -2.0, 2.0]), RadioDevice(position=(1.0, 2.5, 2.2))]
    res = compute_radio_map(scene, srcs, grid, cfg)
    assert res.values.shape == (2, 6, 4) and len(res.diagnostics) == 2
    np.testing.assert_array_equal(res.total(), res.values.sum(axis=0))
    for k, s in enumerate(srcs):
        pos = s.position if isinstance(s, RadioDevice) else s
        single, _ = compute_radio_map_sbr(scene, pos, grid, cfg)
        # same rays and deposits; fp64 atomics only reorder the cell sums
        np.testing.assert_allclose(res.values[k], single, rtol=1e-13, atol=0)
    with pytest.raises(ValueError, match="precoder"):
        compute_radio_map(scene, srcs, grid, cfg, precoders=[[1.0]])


def test_precoded_broadside_array_gain(cuda):
    """Direct-term map of an M-element broadside panel with the default 1/sqrt(M)
    precoder: |sum_m e^{j0}/sqrt(M)|^2 = M times the single-element gain."""
    floor = scenes.quad_mesh(half=5.0, z=-60.0, object_id=1)   # never reached at depth 0
    scene = SceneModel([floor], {1: CONC})
    lam = C0 / 3.5e9
    grid = MeasurementGrid((40.0, 0.0, 3.0), (0, 1, 0), (0, 0, 1), (0.5, 0.5), (1, 1))
    cfg = RadioMapConfig(num_samples=1000, max_depth=0, enabled=R)
    one, _ = compute_radio_map_sbr(scene, np.array([0.0, 0.0, 3.0]), grid, cfg)
    arr = planar_array(1, 4, lam / 2, lam / 2)    # elements along y, broadside = +x
    many, _ = compute_radio_map_sbr(scene, np.array([0.0, 0.0, 3.0]), grid, cfg, array=arr)
    assert many[0, 0] == pytest.approx(4.0 * one[0, 0], rel=1e-3)
