"""Multi-GPU sharding of a pool job.

Pools are fully independent ("distinct instances with distinct seeds may run
in parallel", generator.hpp:96-97), so a job of P pools shards into
contiguous pool ranges, one per rank, with no data-path collective.  The only
exchange is the fused consumer's final reduction (4 fp64 sums + 258 counts,
~2 KB), done by all-gathering the per-rank partials and folding them in rank
order on every rank, so the result is deterministic and identical everywhere.
"""
from __future__ import annotations

import numpy as np


def shard_range(n_pools: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, start+count) of pool ids for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_pools, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def shard_seeds(n_pools: int, rank: int, world: int, seed_base: int = 1) -> np.ndarray:
    """Seeds of this rank's pools: pool p of the whole job has seed seed_base + p."""
    start, count = shard_range(n_pools, rank, world)
    return np.arange(seed_base + start, seed_base + start + count, dtype=np.uint64)


def reduce_consumer(sums: np.ndarray, hist: np.ndarray, group=None):
    """Deterministic all-reduce of consumer partials (rank-order fold)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return np.asarray(sums, dtype=np.float64).copy(), np.asarray(hist, dtype=np.uint64).copy()
    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    s = torch.tensor(np.asarray(sums, dtype=np.float64), device=dev)
    h = torch.tensor(np.asarray(hist, dtype=np.uint64).astype(np.int64), device=dev)
    gs = [torch.empty_like(s) for _ in range(world)]
    gh = [torch.empty_like(h) for _ in range(world)]
    dist.all_gather(gs, s, group=group)
    dist.all_gather(gh, h, group=group)
    out_s = np.zeros(4, dtype=np.float64)
    out_h = np.zeros(hist.shape, dtype=np.uint64)
    for r in range(world):  # fixed order
        out_s = out_s + gs[r].cpu().numpy()
        out_h = out_h + gh[r].cpu().numpy().astype(np.uint64)
    return out_s, out_h
