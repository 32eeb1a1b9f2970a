"""Small workloads that exercise every libsbr kernel family, for compute-sanitizer.

    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize_cases.py CASE

CASE: map   -- box room radio map ({R,S,T}, roulette, threshold, direct term):
               k_map_trace / k_map_shade / k_map_scatter / k_direct
      cir   -- box_collide (40 targets, N_H = 997: heavy slot collisions) and a
               64-receiver canyon CIR (occluder tables, emission-time duplicate
               drop): sweep, vertex order, visibility, select, refine, fields, CFR
      build -- PLOC and LBVH builds of the canyon and a degenerate deep chain,
               ray queries and occlusion through both trees
      edge  -- diffraction: wedge tables, D rows in CIR, the edge map estimator
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from paper_2504_21719_b200 import (MeasurementGrid, PathConfig, RadioDevice,  # noqa: E402
                                   RadioMapConfig, SceneModel, compute_paths,
                                   compute_radio_map_sbr, frequency_response, scenes)
from paper_2504_21719_b200.sampling import Interaction  # noqa: E402

ALL = frozenset(Interaction)
case = sys.argv[1]
if os.environ.get("SBR_REQUIRE_CHECKED") == "1":
    from paper_2504_21719_b200 import _native
    assert _native.lib().sbr_build_flags() & 1, "SBR_LIB_PATH is not the checked build"
    print("checked build:", _native.LIB_PATH)
if case == "map":
    meshes = scenes.box_room_walls()
    mats = scenes.uniform_materials(meshes, scenes.concrete(scattering=0.3))
    sc = SceneModel(meshes, mats)
    grid = MeasurementGrid((0.5, 1.0, 1.2), (1, 0, 0), (0, 1, 0), (0.5, 0.5), (6, 6))
    for cfg in (RadioMapConfig(num_samples=20_000, max_depth=3, seed=1,
                               enabled=frozenset({Interaction.REFLECTION,
                                                  Interaction.SCATTERING,
                                                  Interaction.TRANSMISSION})),
                RadioMapConfig(num_samples=(1 << 19) + 999, max_depth=4, seed=2, rr_depth=1,
                               gain_threshold=1e-9,
                               enabled=frozenset({Interaction.REFLECTION,
                                                  Interaction.SCATTERING}))):
        v, d = compute_radio_map_sbr(sc, (-1.0, -2.0, 1.5), grid, cfg)
        v2, _ = compute_radio_map_sbr(sc, (-1.0, -2.0, 1.5), grid, cfg, shard=(1, 3))
    print("map ok", d["ray_bounces"])
elif case == "cir":
    from test_gpu_cir import build
    for name in ("box_collide", "box_rst"):
        scene, _, cfg, txs, rxs = build(name)
        ps = compute_paths(scene, txs, rxs, cfg)
        print(name, ps.diagnostics["paths"], ps.diagnostics["candidates"])
    from cir_cases import _canyon_targets
    meshes = scenes.street_canyon()
    sc = SceneModel(meshes, scenes.uniform_materials(meshes, scenes.concrete(scattering=0.2)))
    rx = [RadioDevice(position=np.array(d["pos"])) for d in _canyon_targets(64, seed=9)]
    tx = RadioDevice(position=np.array([0.0, 5.0, 20.0]))
    cfg = PathConfig(num_samples=20_000, max_depth=4, q_diffraction=0.0, seed=3,
                     enabled=frozenset({Interaction.REFLECTION, Interaction.SCATTERING}))
    ps = compute_paths(sc, [tx], rx, cfg)
    H = frequency_response(ps, 3.5e9 + np.arange(64) * 30e3, receiver=3)
    print("canyon cir ok", ps.diagnostics["paths"], H.shape)
elif case == "build":
    from paper_2504_21719_b200 import _native
    from test_gpu_edge_inputs import _deep_chain_meshes
    L = _native.lib()
    rng = np.random.default_rng(0)
    for builder in (1, 2, 0):
        L.sbr_set_bvh_builder(builder)
        for meshes in (scenes.street_canyon(), _deep_chain_meshes()):
            sc = SceneModel(meshes, {m.object_id: scenes.concrete() for m in meshes})
            lo, hi = sc.accel.bounds
            o = rng.uniform(lo, hi, (4096, 3))
            d = rng.normal(size=(4096, 3))
            d /= np.linalg.norm(d, axis=1, keepdims=True)
            t, tri, u, v = sc.accel.trace_batch(o, d)
            occ = sc.accel.occluded_batch(o, o + 50.0 * d)
    L.sbr_set_bvh_builder(1)
    print("build ok")
elif case == "edge":
    from test_gpu_cir import build
    for name in ("screen_d", "canyon_rd", "blocks_rtd"):
        scene, _, cfg, txs, rxs = build(name)
        ps = compute_paths(scene, txs, rxs, cfg)
        print(name, ps.diagnostics["paths"])
    from paper_2504_21719_b200 import compute_radio_map
    from test_oracle_edge import edge_case
    meshes, pm, grid, cfg, src, kw = edge_case("blocks_edge")
    scene = SceneModel(meshes, pm)
    pre = kw.pop("precoder", None)
    res = compute_radio_map(scene, [RadioDevice(position=src, **kw)], grid, cfg,
                            precoders=None if pre is None else [pre])
    print("edge ok", res.diagnostics[0].get("deposits"))
torch.cuda.synchronize()
