import sys, time, cProfile, pstats
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2504_21719_b200 import SceneModel, scenes
from paper_2504_21719_b200.radiomap import MeasurementGrid, RadioMapConfig, compute_radio_map_sbr
from paper_2504_21719_b200.sampling import Interaction
m = scenes.street_canyon(); sc = SceneModel(m, scenes.uniform_materials(m, scenes.concrete(scattering=0.3)))
g = MeasurementGrid((0, 0, 1.5), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (200, 200))
cfg = RadioMapConfig(num_samples=10_000_000, max_depth=5, seed=0, enabled=frozenset({Interaction.REFLECTION, Interaction.SCATTERING}))
for _ in range(3): compute_radio_map_sbr(sc, np.array((0.0, 5.0, 20.0)), g, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
t0 = time.perf_counter()
for _ in range(5): compute_radio_map_sbr(sc, np.array((0.0, 5.0, 20.0)), g, cfg)
torch.cuda.synchronize(); t1 = time.perf_counter()
pr.disable()
print("per call ms", (t1 - t0) / 5 * 1e3)
pstats.Stats(pr).sort_stats('tottime').print_stats(12)
