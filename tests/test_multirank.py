"""N>1 host logic on CPU with gloo, world_size 2: pool sharding covers the
job exactly once, and the consumer reduction over ranks equals the
single-process result (histogram exactly, sums to fold-order rounding) and
is identical on every rank."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1005_2314_b200.shard import shard_range, shard_seeds


def test_shard_ranges_partition():
    for n in (1, 7, 16384, 65536):
        for world in (1, 2, 3, 8):
            covered = []
            for r in range(world):
                s, c = shard_range(n, r, world)
                covered.extend(range(s, s + c))
            assert covered == list(range(n))
    assert shard_seeds(10, 1, 2).tolist() == [6, 7, 8, 9, 10]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist

    from oracle.oracle import Cfg, consume_pools
    from paper_1005_2314_b200.shard import reduce_consumer, shard_seeds
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seeds = shard_seeds(16, rank, world)
    sums, hist = consume_pools(Cfg(pool_size=1024), "f32", seeds, 4096, threads=1)
    rs, rh = reduce_consumer(sums, hist)
    out[rank] = (rs.tolist(), rh.tolist())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.usefixtures("oracle_built")
def test_two_rank_consumer_reduction():
    from oracle.oracle import Cfg, consume_pools
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    s0, h0 = out[0]
    s1, h1 = out[1]
    assert s0 == s1 and h0 == h1  # identical on every rank
    ws, wh = consume_pools(Cfg(pool_size=1024), "f32", np.arange(1, 17, dtype=np.uint64), 4096)
    assert np.array_equal(np.array(h0, dtype=np.uint64), wh)
    np.testing.assert_allclose(np.array(s0), ws, rtol=1e-12, atol=1e-9)


def _gpu_worker(rank, world, port, n_pools, count, out):
    """One rank of a sharded config-5 style job on cuda:0: the device
    consumer over this rank's pools, then the deterministic gloo reduction
    (the kernels of the two processes never wait on each other)."""
    import torch
    import torch.distributed as dist

    import paper_1005_2314_b200 as pb
    from paper_1005_2314_b200.shard import reduce_consumer, shard_seeds
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seeds = shard_seeds(n_pools, rank, world)
    b = pb.PoolBatch(pb.GeneratorConfig(pool_size=1024, discard_every=1), n_pools=len(seeds), seeds=seeds)
    sums, hist = b.consume(count)
    b.close()
    rs, rh = reduce_consumer(sums, hist)
    out[rank] = (rs.tolist(), [int(x) for x in rh])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_gpu_consume_equals_single_process(cuda):
    """two processes, each running PoolBatch.consume on its
    shard_seeds range on the GPU, reduced with shard.reduce_consumer, give
    the single-process GPU consume of the whole job: histogram exactly, sums
    to fold-order rounding, identical on both ranks."""
    import paper_1005_2314_b200 as pb
    n_pools, count = 600, 3 * 1023 + 17
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.start_processes(_gpu_worker, args=(world, port, n_pools, count, out), nprocs=world, join=True,
                       start_method="spawn")
    s0, h0 = out[0]
    s1, h1 = out[1]
    assert s0 == s1 and h0 == h1
    b = pb.PoolBatch(pb.GeneratorConfig(pool_size=1024, discard_every=1), n_pools=n_pools,
                     seeds=np.arange(1, n_pools + 1, dtype=np.uint64))
    ws, wh = b.consume(count)
    assert np.array_equal(np.array(h0, dtype=np.uint64), wh)
    np.testing.assert_allclose(np.array(s0), ws, rtol=1e-12, atol=1e-9)
