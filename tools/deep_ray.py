"""Trace the second segment of sample 34048 of the chain scene on the GPU
(diagnostics for the deep-chain parity test)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from test_gpu_edge_inputs import CONC, _deep_chain_meshes  # noqa: E402
from paper_2504_21719_b200 import SceneModel  # noqa: E402

meshes = _deep_chain_meshes(110)
sc = SceneModel(meshes, {0: CONC})
o = np.array([[1.5, 0.3, 0.2], [0.9999999999999999, 0.5652435295164298, -0.2965992795855905]])
d = np.array([[-0.6640364043121106, 0.3522627192142863, -0.65952],
              [0.6640364043121106, 0.3522627192142863, -0.65952]])
t, tri, u, v = sc.accel.trace_batch(o, d)
print("gpu", t, tri, sc.accel.tri_primitive_id[tri] if (tri >= 0).all() else tri)
osc = oracle.OracleScene(meshes, {0: CONC})
print("oracle", osc.trace_batch(o, d)[:2])
# the map's own segment-1 origin: o + t*d as the shade forms it
p = o[0] + t[0] * d[0]
print("p", p.tolist(), "t0", repr(t[0]))
