"""Nodes visited / triangles tested per ray-bounce with the SBR_COUNT_VISITS variant."""
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
os.environ["SBR_LIB_PATH"] = os.path.join(os.getcwd(), "paper_2504_21719_b200/_lib/variants/libsbr_%s.so" % os.environ.get("SBR_VISITS_LIB", "visits"))
import torch
from paper_2504_21719_b200 import SceneModel, scenes, _abi
from paper_2504_21719_b200.radiomap import compute_radio_map_sbr, MeasurementGrid, RadioMapConfig
from paper_2504_21719_b200.sampling import Interaction
for name in ("canyon", "city"):
    meshes = scenes.street_canyon() if name == "canyon" else scenes.city()
    sc = SceneModel(meshes, scenes.uniform_materials(meshes, scenes.concrete(scattering=0.3)))
    grid = MeasurementGrid((0, 0, 1.5), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (200, 200))
    cfg = RadioMapConfig(num_samples=1_000_000, max_depth=5, seed=0,
                         enabled=frozenset({Interaction.REFLECTION, Interaction.SCATTERING}))
    tx = (0.0, 5.0, 20.0) if name == "canyon" else (0.0, 0.0, 30.0)
    _, c = compute_radio_map_sbr(sc, tx, grid, cfg, include_direct=False, return_tensors=True)
    c = c.cpu().numpy()
    rb = c[_abi.MAP_COUNTERS.index("ray_bounces")]
    print(name, "tris", sc.accel.num_triangles, "nodes", sc.accel.num_nodes, "rb", rb,
          "nodes/rb %.2f" % (c[_abi.MAP_COUNTERS.index("direct_visible")] / rb),
          "tris/rb %.2f" % (c[_abi.MAP_COUNTERS.index("threshold_killed")] / rb))
