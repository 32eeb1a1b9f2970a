"""Multi-rank host logic on CPU: world_size-2 gloo runs of the sharded radio map.

The per-rank compute is the CPU oracle (the checker) standing in for the GPU
kernel; what is under test is the product's sharding + all-reduce path
(paper_2504_21719_b200/sharding.py), which bench.py drives over NCCL on the
GPU box.  The reference asserts bitwise-identical maps for any worker count
(pkg/tests/test_radiomap.py:335-346); across ranks the sum order of the
float64 grid changes, so the map must agree to 1e-12 and counters exactly.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_21719_b200 import _abi
from paper_2504_21719_b200.sharding import cyclic_chunks, shard_of_chunks, shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_range_partitions_exactly():
    for n in (1, 7, 1000, 10_000_001):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def test_chunk_aligned_shards():
    n = 5 * (1 << 19) + 123
    spans = [shard_of_chunks(n, r, 2) for r in range(2)]
    assert spans == [(0, 3 << 19), (3 << 19, n)]


def test_cyclic_chunks_partition_and_balance():
    C = 1 << 19
    for n in (1, C, 5 * C + 123, 80_000_000):
        for world in (1, 2, 3, 8):
            spans = [cyclic_chunks(n, r, world) for r in range(world)]
            ids = sorted(x for sp in spans for x in sp)
            assert ids[0][0] == 0 and ids[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ids, ids[1:]))   # exact partition
            sizes = [sum(hi - lo for lo, hi in sp) for sp in spans]
            assert max(sizes) - min(sizes) <= C                        # within one chunk
            # every rank's ids cover the whole pole-to-pole range when it can
            if n >= 2 * world * C:
                assert all(sp[0][0] < n // 2 < sp[-1][1] for sp in spans)


def _cyclic_case():
    import dataclasses
    from cases import build_case
    meshes, mats, src, grid, cfg, kw = build_case("box_rst_rr")
    cfg = dataclasses.replace(cfg, num_samples=3 * (1 << 19) + 11, max_depth=2)
    return meshes, mats, src, grid, cfg, kw


def _cyclic_worker(rank, world, port, out_dir):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2504_21719_b200.sharding import allreduce_map
        meshes, mats, src, grid, cfg, kw = _cyclic_case()
        osc = oracle.OracleScene(meshes, mats)
        vals = np.zeros((grid.shape[1], grid.shape[0]))
        cnt = np.zeros(len(_abi.MAP_COUNTERS), np.int64)
        first = True
        for lo, hi in cyclic_chunks(cfg.num_samples, rank, world):
            v, d = osc.radiomap(src, grid, cfg, sample_range=(lo, hi),
                                include_direct=(rank == 0 and first), **kw)
            first = False
            vals += v
            cnt += np.array([d[k] for k in _abi.MAP_COUNTERS], np.int64)
        v, c = allreduce_map(torch.from_numpy(vals), torch.from_numpy(cnt))
        np.save(os.path.join(out_dir, f"cvals_{rank}.npy"), v.numpy())
        np.save(os.path.join(out_dir, f"ccnt_{rank}.npy"), c.numpy())
    finally:
        dist.destroy_process_group()


def test_three_rank_gloo_cyclic_shards_equal_full_map(tmp_path):
    """The chunk-cyclic partition bench.py / compute_radio_map_sbr_distributed use
    (sbr_radiomap_bounce_sharded on the GPU) reproduces the unsharded map."""
    import oracle
    world = 3
    mp.start_processes(_cyclic_worker, args=(world, _free_port(), str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    meshes, mats, src, grid, cfg, kw = _cyclic_case()
    full, d = oracle.OracleScene(meshes, mats).radiomap(src, grid, cfg, **kw)
    fcnt = np.array([d[k] for k in _abi.MAP_COUNTERS], np.int64)
    for r in range(world):
        np.testing.assert_allclose(np.load(tmp_path / f"cvals_{r}.npy"), full, rtol=1e-12, atol=0)
        assert np.array_equal(np.load(tmp_path / f"ccnt_{r}.npy"), fcnt)


def _oracle_run_shard(case, lo, hi, include_direct):
    import oracle
    from cases import build_case
    meshes, mats, src, grid, cfg, kw = build_case(case)
    vals, diag = oracle.OracleScene(meshes, mats).radiomap(
        src, grid, cfg, sample_range=(lo, hi), include_direct=include_direct, **kw)
    counters = torch.tensor([diag[k] for k in _abi.MAP_COUNTERS], dtype=torch.int64)
    return torch.from_numpy(vals), counters


def _worker(rank, world, port, case, out_dir):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from cases import build_case
        from paper_2504_21719_b200.sharding import sharded_radio_map
        cfg = build_case(case)[4]
        vals, counters = sharded_radio_map(
            lambda lo, hi, d: _oracle_run_shard(case, lo, hi, d), cfg.num_samples)
        np.save(os.path.join(out_dir, f"vals_{rank}.npy"), vals.numpy())
        np.save(os.path.join(out_dir, f"cnt_{rank}.npy"), counters.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["box_rst_rr", "box_directive_array"])
def test_two_rank_gloo_map_equals_single_rank(tmp_path, case):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), case, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    cfg = __import__("cases").build_case(case)[4]
    full, fcnt = _oracle_run_shard(case, 0, cfg.num_samples, True)
    for r in range(world):
        v = np.load(tmp_path / f"vals_{r}.npy")
        c = np.load(tmp_path / f"cnt_{r}.npy")
        np.testing.assert_allclose(v, full.numpy(), rtol=1e-12, atol=0)
        assert np.array_equal(c, fcnt.numpy())


# ---------------------------------------------------------------------------
# CIR: sample shards -> all-gathered candidate rows -> one global selection

def _cir_case():
    from test_oracle_cir import oracle_case
    sc, cfg, txs, rxs = oracle_case("box_trunc")
    targets = np.array([r.position for r in rxs])
    return sc, cfg, txs[0].position, targets


def _cir_worker(rank, world, port, out_dir):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_21719_b200.sharding import gather_rows, owned_records
        sc, cfg, src, targets = _cir_case()
        lo, hi = shard_range(cfg.num_samples, rank, world)
        rows, _ = sc.cir_rows(src, targets, cfg, lo, hi)
        local = {k: torch.from_numpy(v) for k, v in rows.items()}
        g, offsets = gather_rows(local)
        gathered = {k: v.numpy() for k, v in g.items()}
        rec_row, counters = sc.cir_select(src, targets, cfg, gathered)
        pos, loc = owned_records(rec_row, offsets, rank)
        # this rank's records, identified by (ordinal key or LoS code)
        keys = np.where(loc >= 0, rows["key"][np.maximum(loc, 0)] if len(rows["key"]) else 0,
                        loc.astype(np.int64).view(np.uint64))
        np.save(os.path.join(out_dir, f"keys_{rank}.npy"), keys.astype(np.uint64))
        np.save(os.path.join(out_dir, f"pos_{rank}.npy"), pos)
        np.save(os.path.join(out_dir, f"cnt_{rank}.npy"), counters)
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_cir_selection_equals_single_rank(tmp_path):
    """Global dedup over all-gathered rows == the reference's single-chunk selection."""
    world = 2
    mp.start_processes(_cir_worker, args=(world, _free_port(), str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    sc, cfg, src, targets = _cir_case()
    rows, _ = sc.cir_rows(src, targets, cfg, 0, cfg.num_samples)
    rec_row, counters = sc.cir_select(src, targets, cfg, rows)
    want = np.where(rec_row >= 0, rows["key"][np.maximum(rec_row, 0)],
                    rec_row.astype(np.int64).view(np.uint64))
    got = np.zeros(len(want), np.uint64)
    seen = np.zeros(len(want), bool)
    for r in range(world):
        pos = np.load(tmp_path / f"pos_{r}.npy")
        got[pos] = np.load(tmp_path / f"keys_{r}.npy")
        assert not seen[pos].any()
        seen[pos] = True
        # every rank computes identical selection counters (dedup, truncation, overflow)
        assert np.array_equal(np.load(tmp_path / f"cnt_{r}.npy")[5:], counters[5:])
    assert seen.all()
    assert np.array_equal(got, want)
    # and the oracle's row/select split equals its one-shot generation
    rec, diag = sc.generate_candidates(src, targets, cfg)
    assert len(rec["sample"]) == len(want)
    assert diag["chunk_truncated"] > 0 and diag["buffer_overflow"] > 0


def test_owned_records_device_matches_host_form():
    """owned_records_device (the no-host-copy form compute_paths_sharded uses)
    selects the same records as owned_records, with the kept-row mapping."""
    import torch

    from paper_2504_21719_b200.sharding import owned_records, owned_records_device
    rng = np.random.default_rng(5)
    offsets = [0, 40, 75, 120]
    rec_row = np.concatenate([~np.arange(6), rng.permutation(120)[:90]]).astype(np.int64)
    for rank in range(3):
        kept = torch.from_numpy(rng.permutation(500)[:offsets[rank + 1] - offsets[rank]]
                                .astype(np.int64))
        _, loc = owned_records(rec_row, offsets, rank)
        loc = np.array(loc, dtype=np.int64)
        m = loc >= 0
        loc[m] = kept.numpy()[loc[m]]
        got, n = owned_records_device(torch.from_numpy(rec_row), offsets, rank, kept)
        assert n == len(loc)
        assert np.array_equal(got.numpy(), loc)
