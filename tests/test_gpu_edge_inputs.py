"""Empty, ragged and boundary inputs through the public API (GPU path).

The reference handles these without special cases (empty batches return
empty arrays, sample ranges need not align to chunks, a receiver with no
path yields an all-zero response); the drop-in must do the same.
"""

import numpy as np
import pytest

from paper_2504_21719_b200 import (MeasurementGrid, PathConfig, RadioDevice, RadioMapConfig,
                                   SceneModel, build_scene_accel, compute_paths,
                                   compute_radio_map_sbr, frequency_response, scenes)
from paper_2504_21719_b200.errors import EmptyScene
from paper_2504_21719_b200.materials import RadioMaterial
from paper_2504_21719_b200.sampling import Interaction

pytestmark = pytest.mark.gpu
CONC = RadioMaterial("concrete", eps_r=5.24, sigma=0.1, thickness=0.3)
R = frozenset({Interaction.REFLECTION})


def _room():
    return SceneModel([scenes.box_mesh((-3, -4, 0), (3, 4, 3), object_id=0, inward=True)],
                      {0: CONC})


def test_empty_scene_and_empty_batches(cuda):
    with pytest.raises(EmptyScene):
        build_scene_accel([])
    acc = _room().accel
    t, tri, u, v = acc.trace_batch(np.zeros((0, 3)), np.zeros((0, 3)))
    assert t.shape == (0,) and tri.shape == (0,) and u.shape == (0,) and v.shape == (0,)
    assert acc.occluded_batch(np.zeros((0, 3)), np.zeros((0, 3))).shape == (0,)


def test_single_ray_batch_and_t_max_cap(cuda):
    acc = _room().accel
    o, d = np.array([[0.0, 0.0, 1.0]]), np.array([[0.0, 0.0, -1.0]])
    t, tri, _, _ = acc.trace_batch(o, d)
    assert tri[0] >= 0 and t[0] == pytest.approx(1.0, abs=1e-12)
    t, tri, _, _ = acc.trace_batch(o, d, t_max=0.5)      # hit beyond t_max: a miss
    assert tri[0] == -1 and np.isinf(t[0])
    # zero-length segment (len <= 2 eps) is never occluded
    assert not acc.occluded_batch(np.array([[0.0, 0.0, 1.0]]), np.array([[0.0, 0.0, 1.0]]))[0]


@pytest.mark.parametrize("rng_", [(0, 1), (0, 7), (3, 2 ** 19 + 5), (2 ** 19 - 1, 2 ** 19 + 1)])
def test_ragged_sample_ranges_add_up(cuda, rng_):
    """Any split of [0, N) into ranges (chunk-straddling, single samples)
    reproduces the full map: the RNG is keyed by global sample id."""
    scene = _room()
    grid = MeasurementGrid((0.0, 0.0, 1.0), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (6, 8))
    n = 2 ** 19 + 9
    cfg = RadioMapConfig(num_samples=n, max_depth=3, enabled=R, seed=1)
    lo, hi = rng_
    parts = [(0, lo), (lo, hi), (hi, n)]
    total, _ = compute_radio_map_sbr(scene, (0.5, -1.0, 2.0), grid, cfg, include_direct=False)
    acc = np.zeros_like(total)
    for a, b in parts:
        if b > a:
            v, _ = compute_radio_map_sbr(scene, (0.5, -1.0, 2.0), grid, cfg,
                                         sample_range=(a, b), include_direct=False)
            acc += v
    np.testing.assert_allclose(acc, total, rtol=1e-12, atol=0)


def test_one_sample_map_and_one_cell_grid(cuda):
    scene = _room()
    grid = MeasurementGrid((0.0, 0.0, 1.0), (1, 0, 0), (0, 1, 0), (0.25, 0.25), (1, 1))
    vals, diag = compute_radio_map_sbr(scene, (0.0, 0.0, 2.0), grid,
                                       RadioMapConfig(num_samples=1, max_depth=2, enabled=R))
    assert vals.shape == (1, 1) and vals[0, 0] > 0.0     # direct term of the one cell
    assert diag["ray_bounces"] >= 1


def test_receiver_without_paths_gives_zero_response(cuda):
    """A receiver outside the closed room: no path reaches it, H is all zero."""
    cfg = PathConfig(num_samples=2000, max_depth=2, enabled=R, q_diffraction=0.0)
    ps = compute_paths(_room(), [RadioDevice(position=[0.0, 0.0, 1.5])],
                       [RadioDevice(position=[50.0, 0.0, 1.5])], cfg)
    assert len(ps.paths) == 0
    H = frequency_response(ps, [3.5e9, 3.6e9])
    assert H.shape == (1, 1, 2) and not H.any()


def test_cyclic_shards_with_fewer_chunks_than_ranks(cuda):
    """Ranks that own no chunk contribute nothing (maps and CIR rows)."""
    import torch
    from paper_2504_21719_b200 import cir
    scene = _room()
    grid = MeasurementGrid((0.0, 0.0, 1.0), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (4, 4))
    cfg = RadioMapConfig(num_samples=1000, max_depth=2, enabled=R, seed=1)
    full, cf = compute_radio_map_sbr(scene, (0.5, -1.0, 2.0), grid, cfg, include_direct=False,
                                     return_tensors=True)
    parts = [compute_radio_map_sbr(scene, (0.5, -1.0, 2.0), grid, cfg, shard=(r, 3),
                                   include_direct=False, return_tensors=True) for r in range(3)]
    assert torch.equal(parts[0][1], cf) and not parts[1][1].any() and not parts[2][1].any()
    np.testing.assert_allclose(parts[0][0].cpu().numpy(), full.cpu().numpy(), rtol=1e-13,
                               atol=0)  # fp64 atomics reorder the cell sums
    pcfg = PathConfig(num_samples=5000, max_depth=2, enabled=R, q_diffraction=0.0)
    _, targets, *_ = cir._device_plan([RadioDevice(position=[0.0, 0.0, 1.5])],
                                      [RadioDevice(position=[1.0, 2.0, 1.0])], pcfg)
    scene.bind_frequency(pcfg.frequency)
    rows = [cir._sweep_rows(scene, np.array([0.0, 0.0, 1.5]), targets, pcfg, 0, 0, shard=(r, 3))
            for r in range(3)]
    assert rows[0].n > 0 and rows[1].n > 0 and rows[2].n == 0   # 2 chunks of 4096 ids
    kept = cir._local_rows(rows[2])
    assert kept[1].numel() == 0 and kept[2] == 0


def test_non_finite_vertex_rejected_without_leak(cuda):
    """A non-finite corner is rejected by sbr_scene_create (ValueError) instead
    of spinning the PLOC build; the failed build leaks nothing and
    leaves the caller's current device unchanged."""
    import torch

    from paper_2504_21719_b200 import _native
    from paper_2504_21719_b200.geometry import Mesh
    good = scenes.box_mesh((-3, -4, 0), (3, 4, 3), object_id=0)
    for bad_value in (np.inf, -np.inf, np.nan):
        v = good.vertices.copy()
        v[2, 1] = bad_value
        with pytest.raises(ValueError, match="non-finite"):
            build_scene_accel([Mesh(v, good.triangles, object_id=0)])
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(20):
        v = good.vertices.copy()
        v[0, 0] = np.inf
        with pytest.raises(ValueError):
            build_scene_accel([Mesh(v, good.triangles, object_id=0)])
    torch.cuda.synchronize()
    _native.release_scratch(cuda)
    assert torch.cuda.mem_get_info()[0] >= free0 - (8 << 20)
    assert torch.cuda.current_device() == 0
    # the library still works afterwards
    acc = build_scene_accel([good])
    t, tri, _, _ = acc.trace_batch(np.array([[0.0, 0.0, 1.0]]), np.array([[0.0, 0.0, -1.0]]))
    assert tri[0] >= 0 and t[0] == pytest.approx(1.0)


def test_release_scratch_returns_memory(cuda):
    """sbr_release_scratch trims the library's private pool: a radio map's ray
    queues are returned to the driver (and the next map still runs)."""
    import torch

    from paper_2504_21719_b200 import _native
    sc = _room()
    grid = MeasurementGrid((0.0, 0.0, 1.5), (1, 0, 0), (0, 1, 0), (0.5, 0.5), (8, 8))
    cfg = RadioMapConfig(num_samples=4_000_000, max_depth=2, enabled=R)
    v1, d1 = compute_radio_map_sbr(sc, (0.5, 0.5, 1.0), grid, cfg)
    torch.cuda.synchronize()
    held = torch.cuda.mem_get_info()[0]
    _native.release_scratch(cuda)
    freed = torch.cuda.mem_get_info()[0]
    assert freed - held > (1 << 30)  # ~2 GB of queues for 4e6 samples
    v2, d2 = compute_radio_map_sbr(sc, (0.5, 0.5, 1.0), grid, cfg)
    assert d1 == d2
    np.testing.assert_allclose(v2, v1, rtol=1e-12)  # float64 atomics: summation order only


def _deep_chain_meshes(n=110):
    """Unit squares perpendicular to x at x = 2^k (k < n): every Morton code of
    the cubic grid is equal except the last few, and each clustering step can
    merge only the two nearest clusters, so the tree degenerates into a chain
    of depth ~n (> the 64 entries round 1's traversal stack held)."""
    from paper_2504_21719_b200.geometry import Mesh
    verts, tris = [], []
    for k in range(n):
        x = float(2.0 ** k)
        b = len(verts)
        verts += [(x, -1.0, -1.0), (x, 1.0, -1.0), (x, 1.0, 1.0), (x, -1.0, 1.0)]
        tris += [(b, b + 1, b + 2), (b, b + 2, b + 3)]
    return [Mesh(np.array(verts), np.array(tris), object_id=0)]


def test_degenerate_deep_tree_traverses_like_the_reference(cuda):
    """A pathological scene whose (PLOC-only) BVH is a chain ~110 deep: closest hits (far
    to near and near to far along the chain) and occlusion queries match the
    oracle, whose SAH tree needs a deep stack too -- no stack overflow below the
    reference's 256-entry limit (_core.pyx:15)."""
    import oracle
    from paper_2504_21719_b200 import _native
    meshes = _deep_chain_meshes()
    L = _native.lib()
    L.sbr_set_bvh_builder(2)  # PLOC only: the SAH top would build this chain 27 deep
    try:
        acc = build_scene_accel(meshes)
    finally:
        L.sbr_set_bvh_builder(1)
    nodes = np.zeros((int(_native.lib().sbr_scene_num_nodes(acc.handle)), 16), np.int32)
    _native.check(_native.lib().sbr_scene_copy_nodes(acc.handle, nodes.ctypes.data))
    depth, todo = {0: 1}, [0]
    while todo:
        i = todo.pop()
        for c in nodes[i, 12:14]:   # int4 child codes: >= 0 inner node, < 0 leaf
            if c >= 0:
                depth[int(c)] = depth[i] + 1
                todo.append(int(c))
    assert max(depth.values()) > 64
    osc = oracle.OracleScene(meshes)
    rng = np.random.default_rng(3)
    m = 2000
    o = np.column_stack([np.full(m, -10.0), rng.uniform(-0.9, 0.9, m), rng.uniform(-0.9, 0.9, m)])
    d = np.tile([1.0, 0.0, 0.0], (m, 1))
    o2 = o.copy()
    o2[:, 0] = 2.0 ** 112
    for orig, dirs in ((o, d), (o2, -d)):
        t, tri, u, v = acc.trace_batch(orig, dirs)
        want = osc.trace_batch(orig, dirs)
        assert np.array_equal(t, want[0])
        assert np.array_equal(acc.tri_object_id[tri], osc.tri_object_id[want[1]])
        assert np.array_equal(acc.tri_primitive_id[tri], osc.tri_primitive_id[want[1]])
    # segments between consecutive squares: exactly the ones spanning a square are occluded
    a = np.column_stack([2.0 ** rng.integers(0, 100, m) * 1.5, rng.uniform(-0.9, 0.9, m),
                         rng.uniform(-0.9, 0.9, m)])
    b = a.copy()
    b[:, 0] *= rng.choice([0.9, 1.2, 4.0], m)
    occ = acc.occluded_batch(a, b)
    assert np.array_equal(occ, osc.occluded_batch(a, b))
    assert occ.any() and not occ.all()


@pytest.mark.gpu
@pytest.mark.parametrize("streams", [1, 3, 4])
def test_wave_streams_same_map(cuda, streams):
    """A multi-pass map (3 wavefront passes of 2^24 samples) is the same map
    whether its passes run on 1, 2 (default), 3 or 4 streams: identical
    counters, values equal up to float64 atomic summation order (bitwise
    with exact_maps: tests/test_reference_suite.py)."""
    from paper_2504_21719_b200 import _native
    sc = _room()
    grid = MeasurementGrid((0.0, 0.0, 1.5), (1, 0, 0), (0, 1, 0), (0.5, 0.5), (8, 8))
    cfg = RadioMapConfig(num_samples=3 * (1 << 24) - 12345, max_depth=1, enabled=R)
    v2, d2 = compute_radio_map_sbr(sc, (0.5, 0.5, 1.0), grid, cfg)
    try:
        _native.check(_native.lib().sbr_set_wave_streams(streams))
        v, d = compute_radio_map_sbr(sc, (0.5, 0.5, 1.0), grid, cfg)
    finally:
        _native.check(_native.lib().sbr_set_wave_streams(2))
    assert d == d2
    np.testing.assert_allclose(v, v2, rtol=1e-12)



def test_deep_tree_radio_map_matches_oracle(cuda):
    """A radio map over the degenerate chain tree (PLOC only, depth ~110): the
    map trace's warp-uniform loop with unchecked pushes (tree shallower than
    the 256-entry stack) gives the oracle's map (whose SAH tree is shallow)
    with identical counters.  The chain spans 1 .. 2^109: with the box test's
    old pad floor (2^-26 x the scene size) boxes were padded by
    ~1e25 and the float64 triangle test ran on triangles ~1e16 away, where its
    cancellation reported hits the reference's own box test culls."""
    import oracle
    from paper_2504_21719_b200 import _native
    meshes = _deep_chain_meshes(110)
    L = _native.lib()
    L.sbr_set_bvh_builder(2)
    try:
        sc = SceneModel(meshes, {0: CONC})
        acc = sc.accel  # build with the PLOC-only builder
    finally:
        L.sbr_set_bvh_builder(1)
    nodes = np.zeros((int(L.sbr_scene_num_nodes(acc.handle)), 16), np.int32)
    _native.check(L.sbr_scene_copy_nodes(acc.handle, nodes.ctypes.data))
    depth, todo = {0: 1}, [0]
    while todo:
        i = todo.pop()
        for c in nodes[i, 12:14]:
            if c >= 0:
                depth[int(c)] = depth[i] + 1
                todo.append(int(c))
    assert 100 < max(depth.values()) < 256
    grid = MeasurementGrid((2.0, 0.0, 0.05), (1, 0, 0), (0, 1, 0), (0.25, 0.25), (32, 8))
    cfg = RadioMapConfig(num_samples=200_000, max_depth=4, enabled=R, seed=5)
    src = (1.5, 0.3, 0.2)  # between the squares at x = 1 and x = 2
    vals, diag = compute_radio_map_sbr(sc, src, grid, cfg, include_direct=False)
    want, wdiag = oracle.OracleScene(meshes, {0: CONC}).radiomap(np.array(src), grid, cfg,
                                                                 include_direct=False)
    for key in ("deposits", "escaped", "ray_bounces", "terminated"):
        assert diag.get(key, 0) == wdiag.get(key, 0), key
    assert diag["deposits"] > 1000
    np.testing.assert_allclose(vals, want, rtol=1e-12, atol=0.0)
