"""One wavefront pass of the config-4 city map (the bench headline) for ncu.

    python tools/c4_probe.py [--samples N] [--begin B] [--full]

Traces global sample ids [B, B + N) of the 1e9-ray configuration (default: one
2^24-sample pass from the middle of the lattice, so its 6 segment launches of
k_map_trace / k_map_shade look like the full map's), or the whole map.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--samples", type=int, default=1 << 24)
ap.add_argument("--begin", type=int, default=500_000_000)
ap.add_argument("--full", action="store_true")
ap.add_argument("--repeat", type=int, default=1)
a = ap.parse_args()

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2504_21719_b200 import SceneModel, compute_radio_map_sbr  # noqa: E402

meshes, mats, grid, cfg = bench.c4_workload()
scene = SceneModel(meshes, mats)
for _ in range(a.repeat):
    if a.full:
        v, d = compute_radio_map_sbr(scene, np.array(bench.C4_TX), grid, cfg)
    else:
        v, d = compute_radio_map_sbr(scene, np.array(bench.C4_TX), grid, cfg,
                                     sample_range=(a.begin, a.begin + a.samples),
                                     include_direct=False)
torch.cuda.synchronize()
print("c4 probe:", d["ray_bounces"], "ray-bounces")
