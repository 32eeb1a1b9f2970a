"""Host-side profile of one warm config-3 compute_paths (cProfile, top cumulative)."""
import cProfile, os, pstats, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_21719_b200 import PathConfig, RadioDevice, SceneModel, compute_paths, scenes
from paper_2504_21719_b200.sampling import Interaction

meshes = scenes.city()
scene = SceneModel(meshes, scenes.uniform_materials(meshes, scenes.concrete()), device="cuda:0")
rxs = [RadioDevice(position=p) for p in scenes.city_receivers(1024)]
tx = RadioDevice(position=np.array([0.0, 0.0, 30.0]))
cfg = PathConfig(num_samples=1_000_000, max_depth=5, q_diffraction=0.0,
                 enabled=frozenset({Interaction.REFLECTION}), buffer_capacity=2 ** 24)
for _ in range(2):
    compute_paths(scene, [tx], rxs, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    compute_paths(scene, [tx], rxs, cfg)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
