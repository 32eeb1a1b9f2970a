"""Multi-GPU sharding of the SBR sample lattice (one process per GPU).

The reference parallelises only over host threads (a ThreadPool over
sample chunks, radiomap.py:605-628, paths.py:1057-1075) and guarantees the
result is identical for any worker count.  Here the same contract holds
across GPUs: the RNG is keyed by global sample id, so
a contiguous shard of ids traced on any rank makes exactly the decisions
the single-GPU run makes for those ids.

Radio map: each rank traces its shard into a private float64 grid, rank 0
adds the analytic direct term, then ONE all-reduce (sum) of the grid and
one of the diagnostics counters (NCCL over NVLink on the GPU box; gloo in
the CPU tests).  There is no other data-path collective.
"""


def shard_range(num_samples, rank, world):
    """Contiguous [lo, hi) of the global sample ids owned by `rank`.

    Balanced to within one sample; shard sizes differ by at most 1 so the
    max-over-ranks time is the per-rank time.
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    n = int(num_samples)
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def allreduce_map(values, counters, group=None):
    """Sum the per-rank float64 grid and int64 counters in place (one collective each)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(values, group=group)
        dist.all_reduce(counters, group=group)
    return values, counters


def sharded_radio_map(run_shard, num_samples, group=None):
    """Generic multi-rank radio map.

    run_shard(lo, hi, include_direct) -> (values tensor (ny,nx) f64,
    counters tensor int64) computes this rank's contribution (on the GPU in
    the product: `compute_radio_map_sbr(..., return_tensors=True)`).
    Returns the all-reduced (values, counters) tensors, identical on every
    rank.
    """
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        rank, world = dist.get_rank(group), dist.get_world_size(group)
    else:
        rank, world = 0, 1
    lo, hi = shard_range(num_samples, rank, world)
    values, counters = run_shard(lo, hi, rank == 0)
    return allreduce_map(values, counters, group)


def compute_radio_map_sbr_distributed(scene, source, grid, cfg, group=None, **kw):
    """compute_radio_map_sbr over all ranks of `group` (torch.distributed).

    Each rank traces its shard of the N_S sample ids on its own GPU; the
    returned (values (ny,nx) numpy f64, diagnostics dict) equals the
    single-GPU result up to float64 summation order.
    """
    import torch.distributed as dist

    from . import _abi
    from .radiomap import CHUNK_SAMPLES, compute_radio_map_sbr
    if dist.is_available() and dist.is_initialized():
        rank, world = dist.get_rank(group), dist.get_world_size(group)
    else:
        rank, world = 0, 1
    # chunk-cyclic shards (cyclic_chunks): every rank sees the whole sphere
    values, counters = compute_radio_map_sbr(scene, source, grid, cfg, shard=(rank, world),
                                             include_direct=(rank == 0), return_tensors=True,
                                             **kw)
    values, counters = allreduce_map(values, counters, group)
    counts = counters.cpu().numpy()
    diag = {name: int(counts[i]) for i, name in enumerate(_abi.MAP_COUNTERS)
            if name != "stack_overflow" and (counts[i] or name in ("escaped", "ray_bounces"))}
    if counts[_abi.MAP_COUNTERS.index("stack_overflow")]:
        raise RuntimeError("BVH traversal stack overflow")
    diag["samples"] = cfg.num_samples
    diag["chunks"] = -(-cfg.num_samples // CHUNK_SAMPLES)
    diag["direct_visible"] = int(counts[_abi.MAP_COUNTERS.index("direct_visible")])
    return values.cpu().numpy(), diag


def cyclic_chunks(num_samples, rank, world, chunk=None):
    """Global sample-id ranges of a chunk-cyclic shard (sbr_radiomap_bounce_sharded):
    RNG chunks rank, rank + world, ... of 2^19 ids each, as [(lo, hi), ...].

    The Fibonacci ids run pole to pole, so contiguous shards hand one GPU the
    upward rays (which escape at once) and another the grazing ones; dealing
    the chunks round-robin gives every shard the whole sphere.
    """
    from .radiomap import CHUNK_SAMPLES
    chunk = CHUNK_SAMPLES if chunk is None else int(chunk)
    nchunks = -(-int(num_samples) // chunk)
    return [(c * chunk, min((c + 1) * chunk, int(num_samples)))
            for c in range(int(rank), nchunks, int(world))]


def shard_of_chunks(num_samples, rank, world, chunk=None):
    """Shard boundaries rounded to the RNG chunk size (2^19), as SURVEY §8e suggests.

    Not required for correctness (the RNG is keyed per sample) but keeps every
    reference chunk on one rank, which makes per-chunk debugging comparable.
    """
    from .radiomap import CHUNK_SAMPLES
    chunk = CHUNK_SAMPLES if chunk is None else int(chunk)
    nchunks = -(-int(num_samples) // chunk)
    clo, chi = shard_range(nchunks, rank, world)
    return min(clo * chunk, num_samples), min(chi * chunk, num_samples)



def gather_rows(tensors, group=None):
    """All-gather variable-length per-rank row arrays (CIR candidate exchange).

    tensors: dict name -> 1-D tensor of this rank's rows (same length for
    every entry; integer dtypes of <= 8 bytes).  Returns (gathered dict,
    offsets) where rank r's rows occupy [offsets[r], offsets[r+1]).  Two
    collectives in all: one all_gather of the row counts (read back with a
    single host copy) and one all_gather of the rows packed as an (n, k)
    int64 matrix -- for the CIR rows (key, pair_r, pair_f, chain) 32 B per
    row -- padded to the largest rank.  NCCL over NVLink on the GPU box, gloo
    in the CPU tests; uint64 payloads travel bit-identically as int64.
    """
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        n = next(iter(tensors.values())).shape[0]
        return dict(tensors), [0, n]
    world = dist.get_world_size(group)
    names = list(tensors)
    first = tensors[names[0]]
    dev = first.device
    n = int(first.shape[0])
    n_local = torch.tensor([n], dtype=torch.int64, device=dev)
    sizes_l = [torch.empty_like(n_local) for _ in range(world)]
    dist.all_gather(sizes_l, n_local, group=group)
    sizes = [int(x) for x in torch.cat(sizes_l).cpu().tolist()]   # one host copy
    m = max(max(sizes), 1)
    offsets = [0]
    for s_ in sizes:
        offsets.append(offsets[-1] + s_)

    def as_i64(t):
        if t.dtype == torch.uint64:
            return t.view(torch.int64)
        if t.dtype == torch.int64:
            return t
        return t.to(torch.int64)

    packed = torch.zeros((m, len(names)), dtype=torch.int64, device=dev)
    for j, name in enumerate(names):
        packed[:n, j] = as_i64(tensors[name].reshape(-1))
    parts = [torch.empty_like(packed) for _ in range(world)]
    dist.all_gather(parts, packed, group=group)
    cat = torch.cat([p[:s_] for p, s_ in zip(parts, sizes)])
    out = {}
    for j, name in enumerate(names):
        col = cat[:, j].contiguous()
        dt = tensors[name].dtype
        out[name] = col.view(torch.uint64) if dt == torch.uint64 else col.to(dt)
    return out, offsets


def owned_records_device(rec_row, offsets, rank, kept=None):
    """Device form of owned_records: (local row indices / LoS codes tensor,
    count) for the selected entries this rank materialises, with `kept`
    (positions of the gathered rows in the shard's own row list) applied.
    No host copy of the selection."""
    import torch
    lo, hi = offsets[rank], offsets[rank + 1]
    mine = (rec_row >= lo) & (rec_row < hi)
    if rank == 0:
        mine |= rec_row < 0
    sel = rec_row[mine]
    local = torch.where(sel >= 0, sel - lo, sel)
    if kept is not None:
        pos = local >= 0
        local = torch.where(pos, kept.index_select(0, torch.clamp(local, min=0)), local)
    return local.contiguous(), int(local.numel())


def owned_records(rec_row, offsets, rank):
    """Records this rank materialises: rows it produced, plus LoS records on rank 0.

    rec_row: selected entries (index into the gathered rows, or ~target < 0).
    Returns (positions in rec_row, local row indices / LoS codes).
    """
    import numpy as np
    rr = np.asarray(rec_row)
    lo, hi = offsets[rank], offsets[rank + 1]
    mine = (rr >= lo) & (rr < hi)
    if rank == 0:
        mine |= rr < 0
    pos = np.nonzero(mine)[0]
    local = np.where(rr[pos] >= 0, rr[pos] - lo, rr[pos])
    return pos, local
