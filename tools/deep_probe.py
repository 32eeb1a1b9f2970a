"""Radio map over the degenerate chain scene with the PLOC-only and default
builders, against the oracle (diagnostics for tests/test_gpu_edge_inputs.py)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from test_gpu_edge_inputs import CONC, R, _deep_chain_meshes  # noqa: E402
from paper_2504_21719_b200 import (MeasurementGrid, RadioMapConfig, SceneModel,  # noqa: E402
                                   _native, compute_radio_map_sbr)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 110
meshes = _deep_chain_meshes(n)
grid = MeasurementGrid((2.0, 0.0, 0.05), (1, 0, 0), (0, 1, 0), (0.25, 0.25), (32, 8))
cfg = RadioMapConfig(num_samples=200_000, max_depth=int(os.environ.get("DEPTH", 4)), enabled=R, seed=5)
src = (1.5, 0.3, 0.2)
want, wdiag = oracle.OracleScene(meshes, {0: CONC}).radiomap(np.array(src), grid, cfg,
                                                             include_direct=False)
print("oracle", {k: wdiag[k] for k in ("deposits", "escaped", "ray_bounces")})
for b in (2, 1, 0):
    L = _native.lib()
    L.sbr_set_bvh_builder(b)
    sc = SceneModel(meshes, {0: CONC})
    sc.accel
    L.sbr_set_bvh_builder(1)
    vals, diag = compute_radio_map_sbr(sc, src, grid, cfg, include_direct=False)
    print("builder", b, {k: diag.get(k, 0) for k in ("deposits", "escaped", "ray_bounces", "stack_overflow")},
          "maxrel", float(np.max(np.abs(vals - want)) / max(np.max(np.abs(want)), 1e-300)))
