"""Config 3 / 5 timing probe: procedural city CIR on one B200, stage by stage.

    python tools/cir_city.py [--samples 1000000] [--rx 1024] [--depth 5]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=1_000_000)
    ap.add_argument("--rx", type=int, default=1024)
    ap.add_argument("--depth", type=int, default=5)
    ap.add_argument("--repeat", type=int, default=2)
    args = ap.parse_args()
    import torch
    from paper_2504_21719_b200 import PathConfig, RadioDevice, SceneModel, compute_paths, scenes
    from paper_2504_21719_b200 import cir
    from paper_2504_21719_b200.sampling import Interaction

    t0 = time.perf_counter()
    meshes = scenes.city()
    mats = scenes.uniform_materials(meshes, scenes.concrete())
    t1 = time.perf_counter()
    scene = SceneModel(meshes, mats, device="cuda:0")
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    rxs = [RadioDevice(position=p) for p in scenes.city_receivers(args.rx)]
    tx = RadioDevice(position=np.array([0.0, 0.0, 30.0]))
    cfg = PathConfig(num_samples=args.samples, max_depth=args.depth, q_diffraction=0.0,
                     enabled=frozenset({Interaction.REFLECTION}), buffer_capacity=2 ** 24)
    out = {"triangles": scene.accel.num_triangles, "nodes": scene.accel.num_nodes,
           "mesh_gen_s": t1 - t0, "scene_build_s": t2 - t1}
    for rep in range(args.repeat):
        torch.cuda.synchronize()
        s0 = time.perf_counter()
        cand, c, gdiag = cir._generate_device(scene, tx.position,
                                              np.array([r.position for r in rxs]), cfg)
        torch.cuda.synchronize()
        s1 = time.perf_counter()
        pv, status, rc = cir._refine_device(scene, cand)
        torch.cuda.synchronize()
        s2 = time.perf_counter()
        cir._fields_device(scene, cand, pv, status, tx, rxs, cfg)
        torch.cuda.synchronize()
        s3 = time.perf_counter()
        ps = compute_paths(scene, [tx], rxs, cfg)
        torch.cuda.synchronize()
        s4 = time.perf_counter()
        out[f"rep{rep}"] = {"generate_s": s1 - s0, "refine_s": s2 - s1, "fields_s": s3 - s2,
                            "compute_paths_s": s4 - s3, "paths": len(ps.tensors),
                            "counters": c, "diag": ps.diagnostics}
    print(json.dumps(out, default=float))


if __name__ == "__main__":
    main()
