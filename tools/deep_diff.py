"""Find the samples whose radio-map diagnostics differ between the GPU and the
oracle on the degenerate chain scene (diagnostics)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from test_gpu_edge_inputs import CONC, R, _deep_chain_meshes  # noqa: E402
from paper_2504_21719_b200 import (MeasurementGrid, RadioMapConfig, SceneModel,  # noqa: E402
                                   compute_radio_map_sbr)

meshes = _deep_chain_meshes(110)
grid = MeasurementGrid((2.0, 0.0, 0.05), (1, 0, 0), (0, 1, 0), (0.25, 0.25), (32, 8))
cfg = RadioMapConfig(num_samples=200_000, max_depth=4, enabled=R, seed=5)
src = np.array([1.5, 0.3, 0.2])
sc = SceneModel(meshes, {0: CONC})
osc = oracle.OracleScene(meshes, {0: CONC})
keys = ("escaped", "ray_bounces", "deposits")


def both(a, b):
    _, d = compute_radio_map_sbr(sc, tuple(src), grid, cfg, sample_range=(a, b), include_direct=False)
    _, w = osc.radiomap(src, grid, cfg, sample_range=(a, b), include_direct=False)
    return tuple(d.get(k, 0) for k in keys), tuple(w.get(k, 0) for k in keys)


bad = []
step = 2000
for a in range(0, cfg.num_samples, step):
    g, w = both(a, a + step)
    if g != w:
        bad.append(a)
print("chunks", bad)
ids = []
for a in bad[:6]:
    for s in range(a, a + step):
        g, w = both(s, s + 1)
        if g != w:
            ids.append(s)
            print("sample", s, "gpu", g, "oracle", w, flush=True)
            if len(ids) > 12:
                break
