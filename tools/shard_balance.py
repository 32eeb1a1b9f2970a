"""Ray-bounces per rank for contiguous vs chunk-cyclic shards (canyon, N x 1e7 lattice)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_21719_b200 import SceneModel, _abi, scenes
from paper_2504_21719_b200.radiomap import MeasurementGrid, RadioMapConfig, compute_radio_map_sbr
from paper_2504_21719_b200.sampling import Interaction
from paper_2504_21719_b200.sharding import shard_range
RB = _abi.MAP_COUNTERS.index("ray_bounces")
meshes = scenes.street_canyon()
scene = SceneModel(meshes, scenes.uniform_materials(meshes, scenes.concrete(scattering=0.3)))
grid = MeasurementGrid((0, 0, 1.5), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (200, 200))
for world in (2, 4, 8):
    cfg = RadioMapConfig(num_samples=world * 10_000_000, max_depth=5, seed=0,
                         enabled=frozenset({Interaction.REFLECTION, Interaction.SCATTERING}))
    out = {}
    for mode in ("contiguous", "cyclic"):
        rb = []
        for r in range(world):
            kw = {"shard": (r, world)} if mode == "cyclic" else {
                "sample_range": shard_range(cfg.num_samples, r, world)}
            _, c = compute_radio_map_sbr(scene, (0.0, 5.0, 20.0), grid, cfg, include_direct=False,
                                         return_tensors=True, **kw)
            rb.append(int(c[RB].item()))
        out[mode] = rb
        print(f"world {world} {mode:10s} rb/rank {[f'{x/1e6:.1f}M' for x in rb]} "
              f"max/mean {max(rb) / (sum(rb) / world):.3f}", flush=True)
