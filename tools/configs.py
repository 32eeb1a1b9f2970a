"""Timing of BASELINE configs 1, 4 and 5 on one B200 (config 2 and 3 are in bench.py).

    python tools/configs.py [--c4-samples 1000000000]
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
    ap.add_argument("--c4-samples", type=int, default=1_000_000_000)
    ap.add_argument("--repeat", type=int, default=2)
    args = ap.parse_args()
    import torch
    from paper_2504_21719_b200 import (PathConfig, RadioDevice, SceneModel, _native, compute_paths,
                                       frequency_response, make_pattern, scenes)
    from paper_2504_21719_b200.em import planar_array
    from paper_2504_21719_b200.radiomap import MeasurementGrid, RadioMapConfig, compute_radio_map_sbr
    from paper_2504_21719_b200.sampling import Interaction
    R, S = Interaction.REFLECTION, Interaction.SCATTERING
    out = {}

    def timed(fn):
        ts, res = [], None
        for _ in range(args.repeat + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return min(ts[1:]), res

    # config 1: ground + box wall CIR, 1e5 rays, depth 3, {R}
    m1 = scenes.config1_scene()
    s1 = SceneModel(m1, scenes.uniform_materials(m1, scenes.concrete()))
    cfg1 = PathConfig(num_samples=100_000, max_depth=3, q_diffraction=0.0,
                      enabled=frozenset({R}))
    t, ps = timed(lambda: compute_paths(s1, [RadioDevice(position=np.array([0.0, 0.0, 10.0]))],
                                        [RadioDevice(position=np.array([5.0, 8.0, 1.5]))], cfg1))
    out["config1"] = {"ms": t * 1e3, "paths": len(ps.tensors), "kinds":
                      sorted(p.kinds for p in ps.paths), "reference_cpu_ms": 196.0}

    # city scene for 4 and 5
    mc = scenes.city()
    sc = SceneModel(mc, scenes.uniform_materials(mc, scenes.concrete(scattering=0.3)))
    grid = MeasurementGrid((0.0, 0.0, 1.5), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (1000, 1000))
    cfg4 = RadioMapConfig(num_samples=args.c4_samples, max_depth=5, enabled=frozenset({R, S}),
                          seed=0)
    _native.profile_enable(True)
    t, (vals, diag) = timed(lambda: compute_radio_map_sbr(sc, (0.0, 0.0, 30.0), grid, cfg4))
    ks = {k: _native.profile_kernel_ms(k)[0] / (args.repeat + 1)
          for k in ("k_map_trace", "k_map_shade", "k_map_scatter")}
    _native.profile_enable(False)
    out["config4_1gpu"] = {"samples": args.c4_samples, "s": t, "ray_bounces": diag["ray_bounces"],
                           "rb_per_s": diag["ray_bounces"] / t, "kernel_ms": ks,
                           "deposits": diag.get("deposits", 0),
                           "nonzero_cells": int(np.count_nonzero(vals))}

    # config 5: arrays + CFR, depth 6
    sc5 = SceneModel(mc, scenes.uniform_materials(mc, scenes.concrete()))
    lam = 299792458.0 / 3.5e9
    tx = RadioDevice(position=np.array([0.0, 0.0, 30.0]), pattern=make_pattern("tr38901"),
                     array=planar_array(8, 8, lam / 2, lam / 2))
    rx = RadioDevice(position=np.array([2.0, 60.0, 1.5]), array=planar_array(4, 4, lam / 2,
                                                                             lam / 2))
    cfg5 = PathConfig(num_samples=1_000_000, max_depth=6, q_diffraction=0.0,
                      enabled=frozenset({R}))
    freqs = 3.5e9 + (np.arange(1024) - 512) * 30e3

    def c5():
        p = compute_paths(sc5, [tx], [rx], cfg5)
        return p, frequency_response(p, freqs)
    t, (ps5, H) = timed(c5)
    out["config5"] = {"ms": t * 1e3, "paths": len(ps5.tensors), "H_shape": list(H.shape),
                      "samples": 1_000_000, "depth": 6}
    print(json.dumps(out, default=float))


if __name__ == "__main__":
    main()
