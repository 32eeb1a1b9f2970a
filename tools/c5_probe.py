import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
import torch
from paper_2504_21719_b200 import PathConfig, RadioDevice, SceneModel, make_pattern, scenes, compute_paths
from paper_2504_21719_b200.cir import frequency_response
from paper_2504_21719_b200.em import planar_array
from paper_2504_21719_b200.sampling import Interaction
meshes = scenes.city()
scene = SceneModel(meshes, scenes.uniform_materials(meshes, scenes.concrete()))
lam = 299792458.0 / 3.5e9
tx = RadioDevice(position=np.array([0.0, 0.0, 30.0]), pattern=make_pattern("tr38901"), array=planar_array(8, 8, lam / 2, lam / 2))
rx = RadioDevice(position=np.array([2.0, 60.0, 1.5]), array=planar_array(4, 4, lam / 2, lam / 2))
cfg = PathConfig(num_samples=1_000_000, max_depth=6, q_diffraction=0.0, enabled=frozenset({Interaction.REFLECTION}))
freqs = 3.5e9 + (np.arange(1024) - 512) * 30e3
for i in range(3):
    t0 = time.perf_counter(); ps = compute_paths(scene, [tx], [rx], cfg); torch.cuda.synchronize(); t1 = time.perf_counter()
    H = frequency_response(ps, freqs); t2 = time.perf_counter()
    print("paths %.1f ms cfr %.1f ms" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3))
