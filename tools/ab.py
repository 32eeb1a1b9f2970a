"""A/B of libsbr variants on the bench workloads (run under gpurun, one GPU):

    python tools/ab.py [variant ...]     (variants: paper_2504_21719_b200/_lib/variants/libsbr_<v>.so)

For the default library and each variant, in a fresh process: device ms of a
config-4 city map (1e9 rays) with its k_map_trace / k_map_shade / k_map_scatter
split, a config-2 canyon map, and the config-3 CIR visibility kernel; plus the
ray-bounce / path counts so a variant that changes results is visible.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, ROOT)
import bench
from paper_2504_21719_b200 import SceneModel, _native, _abi, scenes, PathConfig, RadioDevice, compute_paths
from paper_2504_21719_b200.sampling import Interaction
out = {}
import os
if os.environ.get("AB_BUILDER"):
    _native.check(_native.lib().sbr_set_bvh_builder(int(os.environ["AB_BUILDER"])))
def maps(workload, tx, n, what):
    meshes, mats, grid, cfg = workload
    sc = SceneModel(meshes, mats)
    run = bench.MapRunner(sc, grid, cfg, tx, torch.device("cuda", 0), 0, 1)
    run.step(); torch.cuda.synchronize()
    _native.profile_enable(True)
    ev = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); run.step(); b.record(); ev.append((a, b))
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in ev]
    split = {k: round(_native.profile_kernel_ms(k)[0] / n, 2) for k in ("k_map_trace", "k_map_shade", "k_map_scatter")}
    _native.profile_enable(False)
    out[what] = {"ms": round(float(np.median(ms)), 2), "split": split,
                 "rb": int(run.counters[run.rb_idx].item())}
if "c4" in WHAT:
    maps(bench.c4_workload(), bench.C4_TX, 3, "c4")
if "c2" in WHAT:
    maps(bench.c2_workload(bench.C2_SAMPLES_PER_GPU), bench.C2_TX, 5, "c2")
if "c3" in WHAT:
    meshes = scenes.city()
    sc = SceneModel(meshes, scenes.uniform_materials(meshes, scenes.concrete()))
    rxs = [RadioDevice(position=p) for p in scenes.city_receivers(1024)]
    tx = RadioDevice(position=np.array([0.0, 0.0, 30.0]))
    cfg = PathConfig(num_samples=1_000_000, max_depth=5, q_diffraction=0.0,
                     enabled=frozenset({Interaction.REFLECTION}), buffer_capacity=2 ** 24)
    compute_paths(sc, [tx], rxs, cfg)
    _native.profile_enable(True)
    ev = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); ps = compute_paths(sc, [tx], rxs, cfg); b.record(); ev.append((a, b))
    torch.cuda.synchronize()
    out["c3"] = {"ms": round(float(np.median([a.elapsed_time(b) for a, b in ev])), 2),
                 "vis": round(_native.profile_kernel_ms("k_cir_visibility")[0] / 3, 2),
                 "sweep": round(_native.profile_kernel_ms("k_cir_sweep")[0] / 3, 2),
                 "paths": ps.diagnostics["paths"], "cand": ps.diagnostics["candidates"],
                 "dup": ps.diagnostics["duplicates"]}
    _native.profile_enable(False)
print("AB " + json.dumps(out))
'''


def main():
    what = os.environ.get("AB_WHAT", "c4,c2,c3")
    variants = ["default"] + sys.argv[1:]
    for rnd in range(int(os.environ.get("AB_ROUNDS", "1"))):
        for v in variants:
            env = dict(os.environ)
            if v != "default":
                env["SBR_LIB_PATH"] = os.path.join(ROOT, "paper_2504_21719_b200", "_lib",
                                                   "variants", f"libsbr_{v}.so")
            code = CHILD.replace("ROOT", repr(ROOT)).replace("WHAT", repr(what))
            r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                               text=True)
            line = [ln for ln in r.stdout.splitlines() if ln.startswith("AB ")]
            print(v, line[-1][3:] if line else "FAILED " + r.stderr[-800:], flush=True)


if __name__ == "__main__":
    main()
