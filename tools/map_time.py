"""Device time of one canyon config-2 bounce call (CUDA events), for A/B of library variants."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2504_21719_b200 import SceneModel, scenes, _abi
from paper_2504_21719_b200.radiomap import MeasurementGrid, RadioMapConfig, compute_radio_map_sbr
from paper_2504_21719_b200.sampling import Interaction
m = scenes.street_canyon(); sc = SceneModel(m, scenes.uniform_materials(m, scenes.concrete(scattering=0.3)))
g = MeasurementGrid((0, 0, 1.5), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (200, 200))
cfg = RadioMapConfig(num_samples=10_000_000, max_depth=5, seed=0,
                     enabled=frozenset({Interaction.REFLECTION, Interaction.SCATTERING}))
ts = []
for k in range(8):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    v, c = compute_radio_map_sbr(sc, np.array((0.0, 5.0, 20.0)), g, cfg, include_direct=False,
                                 return_tensors=True)
    b.record(); torch.cuda.synchronize()
    if k >= 3:
        ts.append(a.elapsed_time(b))
rb = int(c[_abi.MAP_COUNTERS.index("ray_bounces")].item())
print(os.path.basename(os.environ.get("SBR_LIB_PATH", "default")), "ms %.2f" % np.mean(ts),
      "rb/s %.3e" % (rb / (np.mean(ts) / 1e3)), "sum %.6e" % float(v.sum().item()))
