"""Visibility work per rank for contiguous CIR sample shards (config 3)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_21719_b200 import PathConfig, RadioDevice, SceneModel, scenes, cir, _abi
from paper_2504_21719_b200.sampling import Interaction
from paper_2504_21719_b200.sharding import shard_range
meshes = scenes.city()
scene = SceneModel(meshes, scenes.uniform_materials(meshes, scenes.concrete()))
rxs = [RadioDevice(position=p) for p in scenes.city_receivers(1024)]
cfg = PathConfig(num_samples=1_000_000, max_depth=5, q_diffraction=0.0,
                 enabled=frozenset({Interaction.REFLECTION}), buffer_capacity=2 ** 24)
_, targets, *_ = cir._device_plan([RadioDevice(position=(0.0, 0.0, 30.0))], rxs, cfg)
scene.bind_frequency(cfg.frequency)
VIS = _abi.CIR_COUNTERS.index("visibility_rays")
for world in (8,):
    for mode in ("contiguous", "cyclic"):
        vis = []
        for r in range(world):
            lo, hi = shard_range(cfg.num_samples, r, world)
            R = cir._sweep_rows(scene, np.array([0.0, 0.0, 30.0]), targets, cfg, lo, hi,
                                shard=(r, world) if mode == "cyclic" else None)
            vis.append(int(R.counters[VIS].item()))
        print(world, mode, [f"{v/1e6:.0f}M" for v in vis],
              "max/mean %.3f" % (max(vis) / (sum(vis) / world)), flush=True)
