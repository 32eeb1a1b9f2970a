"""One rank of the multi-rank GPU test (tests/test_gpu_multirank.py).

Launched by torchrun with N ranks on ONE GPU over gloo (the ranks share
cuda:0; the driver's GPU box has one device): every rank runs the product's
distributed entry points -- compute_paths_sharded (chunk-cyclic sample
shards, shard-local pre-selection, all-gathered rows, replicated selection,
owned-record refinement, gathered paths) and compute_radio_map_sbr_distributed
(chunk-cyclic shards, all-reduced grid) -- with the real kernels, and writes
its results to OUT/r<rank>.npz for the test to compare with one process.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/multirank_worker.py OUT CASE
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def setup(case):
    from paper_2504_21719_b200 import PathConfig, RadioDevice, SceneModel, scenes
    from paper_2504_21719_b200.radiomap import MeasurementGrid, RadioMapConfig
    from paper_2504_21719_b200.sampling import Interaction
    RS = frozenset({Interaction.REFLECTION, Interaction.SCATTERING})
    if case == "canyon":
        meshes = scenes.street_canyon()
        scene = SceneModel(meshes, scenes.uniform_materials(meshes,
                                                            scenes.concrete(scattering=0.3)))
        rxs = [RadioDevice(position=p) for p in ([10.0, 0.5, 1.5], [-30.0, 10.0, 1.5],
                                                  [0.5, 50.0, 1.5])]
        tx = [RadioDevice(position=(0.0, 5.0, 20.0))]
        pcfg = PathConfig(num_samples=3 * 4096 * 7 + 5, max_depth=3, q_diffraction=0.0,
                          enabled=RS)
        grid = MeasurementGrid((0, 0, 1.5), (1, 0, 0), (0, 1, 0), (2.0, 2.0), (100, 100))
        mcfg = RadioMapConfig(num_samples=5 * (1 << 19) + 3, max_depth=3, seed=2, enabled=RS)
        src = (0.0, 5.0, 20.0)
    else:  # "city": config 3 receivers / config 4 grid at reduced sample counts
        meshes = scenes.city()
        scene = SceneModel(meshes, scenes.uniform_materials(meshes,
                                                            scenes.concrete(scattering=0.3)))
        rxs = [RadioDevice(position=p) for p in scenes.city_receivers(1024)]
        tx = [RadioDevice(position=(0.0, 0.0, 30.0))]
        pcfg = PathConfig(num_samples=50_000, max_depth=5, q_diffraction=0.0,
                          enabled=frozenset({Interaction.REFLECTION}), buffer_capacity=2 ** 24)
        grid = MeasurementGrid((0.0, 0.0, 1.5), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (1000, 1000))
        mcfg = RadioMapConfig(num_samples=7 * (1 << 19) + 12345, max_depth=5, seed=0,
                              enabled=RS)
        src = (0.0, 0.0, 30.0)
    return scene, tx, rxs, pcfg, grid, mcfg, src


def main():
    import torch
    import torch.distributed as dist
    out, case = sys.argv[1], sys.argv[2]
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    try:
        from paper_2504_21719_b200.cir import compute_paths_sharded
        from paper_2504_21719_b200.sharding import compute_radio_map_sbr_distributed
        scene, tx, rxs, pcfg, grid, mcfg, src = setup(case)
        ps = compute_paths_sharded(scene, tx, rxs, pcfg)
        vals, diag = compute_radio_map_sbr_distributed(scene, src, grid, mcfg)
        T = ps.tensors
        np.savez(os.path.join(out, f"r{rank}.npz"), chain=T.chain_hash, gain=T.gain,
                 delay=T.delay, rx=T.rx, sample=T.sample, depth=T.depth, vals=vals,
                 dup=ps.diagnostics["duplicates"], cand=ps.diagnostics["candidates"],
                 paths=ps.diagnostics["paths"], rb=diag["ray_bounces"],
                 deposits=diag.get("deposits", 0), escaped=diag["escaped"],
                 direct=diag["direct_visible"])
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
