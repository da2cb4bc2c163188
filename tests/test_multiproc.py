"""Multi-process host logic of the message-sharded path,
on CPU with the gloo backend at world size 2: the shard arithmetic, the
broadcast of pk + caches as int64 views of uint64 words, the max-over-ranks
timing reduction, and that sharded encryption with msg_base = global offset is
bit-identical to the unsharded batch (the oracle stands in for each rank's
device, since there is no GPU here)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2408_07304_b200.dist import broadcast_words, max_over_ranks, shard_range


@pytest.mark.parametrize("total", [0, 1, 7, 8, 16384, 65537])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_range_partitions(total, world):
    ranges = [shard_range(r, world, total) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == total
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c                                  # contiguous, disjoint
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1                # balanced


def test_shard_range_rejects_bad_arguments():
    with pytest.raises(ValueError):
        shard_range(2, 2, 10)
    with pytest.raises(ValueError):
        shard_range(0, 0, 10)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle as O
        from workloads import CONFIGS, int_plaintexts
        cfg = CONFIGS["C1"]
        P = O.Params.make(cfg.log_n, cfg.bits, cfg.log_scale)
        _, _, pk_np = O.keygen(P, cfg.key_seed)
        cache_np = O.precompute_cache(P, pk_np, cfg.cache_seed, O.COEFF)
        # rank 0 owns the keys; the others start from garbage and receive them
        if rank == 0:
            pk = torch.from_numpy(pk_np.copy())
            cache = torch.from_numpy(cache_np.copy())
        else:
            pk = torch.full(pk_np.shape, 7, dtype=torch.uint64)
            cache = torch.full(cache_np.shape, 9, dtype=torch.uint64)
        broadcast_words([pk, cache], src=0)
        bcast_ok = np.array_equal(pk.numpy(), pk_np) and np.array_equal(cache.numpy(), cache_np)
        # each rank encrypts its shard of a 5-message batch with msg_base = begin
        total = 5
        m = int_plaintexts(cfg.log_n, total, seed=3)
        b0, b1 = shard_range(rank, world, total)
        mine = [O.zinc_encrypt(P, cache.numpy(), O.COEFF, m[b], cfg.enc_seed, b) for b in range(b0, b1)]
        gathered = [None] * world
        dist.all_gather_object(gathered, (b0, b1, mine))
        shard_ok = True
        if rank == 0:
            full = [O.zinc_encrypt(P, cache_np, O.COEFF, m[b], cfg.enc_seed, b) for b in range(total)]
            got = [c for _, _, cs in sorted(gathered, key=lambda g: g[0]) for c in cs]
            shard_ok = len(got) == total and all(np.array_equal(a, b) for a, b in zip(got, full))
        mx = max_over_ranks([1.0 + rank, 5.0 - rank])
        q.put((rank, bcast_ok, shard_ok, mx))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface the failure in the parent
        q.put((rank, repr(e), None, None))


def test_gloo_world2_broadcast_shard_and_max():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, bcast_ok, shard_ok, mx in res:
        assert bcast_ok is True, (rank, bcast_ok)
        assert shard_ok is True, rank
        assert mx == [2.0, 5.0], mx
