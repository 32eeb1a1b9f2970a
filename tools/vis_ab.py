"""A/B of k_cir_visibility variants on config 3 (city, 1 Tx x 1024 Rx, N_S=1e6):
per-kernel ms + a digest of the path set (must be identical across variants).

    SBR_LIB_PATH=.../libsbr_X.so python tools/vis_ab.py [--samples N]
"""
import argparse, hashlib, json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--samples", type=int, default=1_000_000)
ap.add_argument("--repeat", type=int, default=3)
args = ap.parse_args()
import torch
from paper_2504_21719_b200 import PathConfig, RadioDevice, SceneModel, compute_paths, scenes, _native
from paper_2504_21719_b200.sampling import Interaction

meshes = scenes.city()
scene = SceneModel(meshes, scenes.uniform_materials(meshes, scenes.concrete()), device="cuda:0")
rxs = [RadioDevice(position=p) for p in scenes.city_receivers(1024)]
tx = RadioDevice(position=np.array([0.0, 0.0, 30.0]))
cfg = PathConfig(num_samples=args.samples, max_depth=5, q_diffraction=0.0,
                 enabled=frozenset({Interaction.REFLECTION}), buffer_capacity=2 ** 24)
ps = compute_paths(scene, [tx], rxs, cfg)   # warm-up
torch.cuda.synchronize()
_native.profile_enable(True)
t0 = time.perf_counter()
for _ in range(args.repeat):
    ps = compute_paths(scene, [tx], rxs, cfg)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / args.repeat
ms = {k: _native.profile_kernel_ms(k)[0] / args.repeat for k in ("k_cir_sweep", "k_cir_visibility")}
_native.profile_enable(False)
T = ps.tensors
h = hashlib.sha256()
for a in (T.rx, T.depth, T.chain_hash, T.sample, T.kind, T.obj, T.prim):
    h.update(np.ascontiguousarray(a).tobytes())
d = {k: v for k, v in ps.diagnostics.items() if not isinstance(v, dict)}
print(json.dumps({"lib": os.path.basename(os.environ.get("SBR_LIB_PATH", "default")),
                  "wall_ms": wall * 1e3, "kernel_ms": ms, "paths": len(T),
                  "digest": h.hexdigest()[:16], "gain_sum": complex(T.gain.sum()).__repr__(),
                  "diag": d}, default=float))
