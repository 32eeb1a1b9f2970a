"""Where a config-3 compute_paths goes: every device kernel / memcpy of one warm solve
(torch.profiler / CUPTI), summed by name, against the wall time of the call.

    python tools/cir_breakdown.py [--samples N] [--rx 1024]
"""
import argparse, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--samples", type=int, default=1_000_000)
ap.add_argument("--rx", type=int, default=1024)
args = ap.parse_args()
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2504_21719_b200 import PathConfig, RadioDevice, SceneModel, compute_paths, scenes
from paper_2504_21719_b200.sampling import Interaction

meshes = scenes.city()
scene = SceneModel(meshes, scenes.uniform_materials(meshes, scenes.concrete()), device="cuda:0")
rxs = [RadioDevice(position=p) for p in scenes.city_receivers(args.rx)]
tx = RadioDevice(position=np.array([0.0, 0.0, 30.0]))
cfg = PathConfig(num_samples=args.samples, max_depth=5, q_diffraction=0.0,
                 enabled=frozenset({Interaction.REFLECTION}), buffer_capacity=2 ** 24)
for _ in range(2):
    compute_paths(scene, [tx], rxs, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
compute_paths(scene, [tx], rxs, cfg)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    compute_paths(scene, [tx], rxs, cfg)
    torch.cuda.synchronize()
tot = {}
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        k = ev.name[:90]
        ms, n = tot.get(k, (0.0, 0))
        tot[k] = (ms + ev.device_time / 1e3, n + 1)
dev = sum(v[0] for v in tot.values())
print(f"wall {wall:.2f} ms (unprofiled), device kernels+copies {dev:.2f} ms")
for k, (ms, n) in sorted(tot.items(), key=lambda t: -t[1][0])[:30]:
    print(f"{ms:9.3f} ms {n:5d}x  {k}")
cpu = prof.key_averages()
print(cpu.table(sort_by="cpu_time_total", row_limit=15))
