"""Multi-GPU plumbing for the message-sharded path.

Messages are independent (Algorithm 1, touches one message at
a time), so P ranks split a batch by message index with no data-path
collective.  The only collectives are a one-off broadcast of the public key and
the Zinc caches from rank 0 and a max-reduction of per-rank elapsed times.
Everything here is backend-agnostic torch.distributed (NCCL on B200s, gloo in
the CPU tests), and takes no part in the arithmetic.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(rank: int, world: int, total: int) -> tuple[int, int]:
    """Global message range [begin, end) of `rank` when `total` messages are
    split over `world` ranks as evenly as possible (the first total % world ranks
    take one extra).  msg_base = begin keeps the Philox streams global."""
    if world < 1 or not 0 <= rank < world or total < 0:
        raise ValueError(f"bad shard request rank={rank} world={world} total={total}")
    q, r = divmod(total, world)
    begin = rank * q + min(rank, r)
    return begin, begin + q + (1 if rank < r else 0)


def broadcast_words(tensors, src: int = 0) -> None:
    """Broadcast uint64 key / cache tensors from `src` in place.  Collectives do
    not take uint64, so the same bytes travel as an int64 view."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return
    for t in tensors:
        if not t.is_contiguous():
            raise ValueError("broadcast_words needs contiguous tensors")
        dist.broadcast(t.view(torch.int64) if t.dtype == torch.uint64 else t, src=src)


def max_over_ranks(values, device=None) -> list[float]:
    """Element-wise max over ranks of a list of floats (per-rank elapsed times)."""
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]
