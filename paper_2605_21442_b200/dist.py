"""Host-side plumbing of the vocab-parallel path (P:169, P:180 loss parallel).

torch.distributed is used only to move the 128-byte NCCL id and to take the
max-over-ranks step time; all data-path collectives run inside liblce.so.
"""

from __future__ import annotations


def shard_range(vocab: int, world: int, rank: int):
    """Contiguous vocab shard of `rank` (R17): V_l = ceil(V / P),
    the last rank shorter.  Returns (vocab_start, vocab_local)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    vl = -(-vocab // world)
    start = min(vocab, rank * vl)
    return start, min(vocab, start + vl) - start


def broadcast_bytes(payload, group=None, src: int = 0) -> bytes:
    """Rank `src` supplies `payload` (bytes); every rank returns it."""
    import torch.distributed as dist

    obj = [payload if dist.get_rank(group) == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


def max_over_ranks(value: float, group=None, device=None) -> float:
    """Max of a per-rank scalar (the bench's step time is the slowest rank's)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
