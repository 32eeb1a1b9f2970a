"""Rows a shard would all-gather with and without the local pre-selection (config 3)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_21719_b200 import PathConfig, RadioDevice, SceneModel, scenes, cir
from paper_2504_21719_b200.sampling import Interaction
from paper_2504_21719_b200.sharding import shard_range
meshes = scenes.city()
scene = SceneModel(meshes, scenes.uniform_materials(meshes, scenes.concrete()))
rxs = [RadioDevice(position=p) for p in scenes.city_receivers(1024)]
cfg = PathConfig(num_samples=1_000_000, max_depth=5, q_diffraction=0.0,
                 enabled=frozenset({Interaction.REFLECTION}), buffer_capacity=2 ** 24)
_, targets, *_ = cir._device_plan([RadioDevice(position=(0.0, 0.0, 30.0))], rxs, cfg)
scene.bind_frequency(cfg.frequency)
for world in (1, 8):
    lo, hi = shard_range(cfg.num_samples, 0, world)
    R = cir._sweep_rows(scene, np.array([0.0, 0.0, 30.0]), targets, cfg, lo, hi)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rows, kept, nd = cir._local_rows(R)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"world {world}: shard rows {R.n}, kept {kept.numel()}, dropped {nd}, "
          f"local dedup {1e3 * (t1 - t0):.1f} ms")
