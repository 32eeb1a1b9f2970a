"""Correctness check of the multi-rank host paths with real kernels: two gloo ranks
sharing cuda:0 run compute_paths_sharded / compute_radio_map_sbr_distributed and
must reproduce the single-process results (no timing: one GPU, two processes).

    python tools/two_rank_check.py
"""
import os, socket, sys
import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def setup():
    from paper_2504_21719_b200 import (PathConfig, RadioDevice, RadioMapConfig, SceneModel, scenes)
    from paper_2504_21719_b200.radiomap import MeasurementGrid
    from paper_2504_21719_b200.sampling import Interaction
    meshes = scenes.street_canyon()
    scene = SceneModel(meshes, scenes.uniform_materials(meshes, scenes.concrete(scattering=0.3)))
    rxs = [RadioDevice(position=p) for p in ([10.0, 0.5, 1.5], [-30.0, 10.0, 1.5],
                                              [0.5, 50.0, 1.5])]
    tx = [RadioDevice(position=(0.0, 5.0, 20.0))]
    pcfg = PathConfig(num_samples=3 * 4096 * 7 + 5, max_depth=3, q_diffraction=0.0,
                      enabled=frozenset({Interaction.REFLECTION, Interaction.SCATTERING}))
    grid = MeasurementGrid((0, 0, 1.5), (1, 0, 0), (0, 1, 0), (2.0, 2.0), (100, 100))
    mcfg = RadioMapConfig(num_samples=5 * (1 << 19) + 3, max_depth=3, seed=2,
                          enabled=frozenset({Interaction.REFLECTION, Interaction.SCATTERING}))
    return scene, tx, rxs, pcfg, grid, mcfg


def worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_21719_b200.cir import compute_paths_sharded
        from paper_2504_21719_b200.sharding import compute_radio_map_sbr_distributed
        scene, tx, rxs, pcfg, grid, mcfg = setup()
        ps = compute_paths_sharded(scene, tx, rxs, pcfg)
        vals, diag = compute_radio_map_sbr_distributed(scene, (0.0, 5.0, 20.0), grid, mcfg)
        np.savez(os.path.join(out, f"r{rank}.npz"), chain=ps.tensors.chain_hash,
                 gain=ps.tensors.gain, delay=ps.tensors.delay, vals=vals,
                 dup=ps.diagnostics["duplicates"], cand=ps.diagnostics["candidates"],
                 rb=diag["ray_bounces"])
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    import tempfile
    from paper_2504_21719_b200 import compute_paths
    from paper_2504_21719_b200.radiomap import compute_radio_map_sbr
    with tempfile.TemporaryDirectory() as td:
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        mp.start_processes(worker, args=(2, port, td), nprocs=2, join=True, start_method="spawn")
        scene, tx, rxs, pcfg, grid, mcfg = setup()
        ref = compute_paths(scene, tx, rxs, pcfg)
        rv, rd = compute_radio_map_sbr(scene, (0.0, 5.0, 20.0), grid, mcfg)
        for r in range(2):
            g = np.load(os.path.join(td, f"r{r}.npz"))
            assert np.array_equal(g["chain"], ref.tensors.chain_hash), "chains"
            assert np.allclose(g["gain"], ref.tensors.gain, rtol=1e-12, atol=0), "gains"
            assert int(g["dup"]) == ref.diagnostics["duplicates"], "duplicates"
            assert int(g["cand"]) == ref.diagnostics["candidates"], "candidates"
            np.testing.assert_allclose(g["vals"], rv, rtol=1e-12, atol=0)
            assert int(g["rb"]) == rd["ray_bounces"]
        print(f"two-rank check ok: {len(ref.tensors)} paths, duplicates "
              f"{ref.diagnostics['duplicates']}, map rb {rd['ray_bounces']}")
