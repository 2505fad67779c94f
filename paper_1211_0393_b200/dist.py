"""Multi-GPU plumbing for the batched config (C3): one process per GPU, images
sharded by contiguous ranges, NO per-iteration collective (every image's
Landweber loop is independent).  torch.distributed is only used for
the start/stop barriers, the max-over-ranks timing and the optional end-of-run
gather of per-image histories."""
from __future__ import annotations

from typing import List, Tuple


def shard(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Balanced contiguous shard (first, count) of `total` images for `rank`."""
    if world < 1 or not 0 <= rank < world or total < 0:
        raise ValueError("shard: bad arguments")
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def weak_shard(per_rank: int, rank: int) -> Tuple[int, int]:
    """Weak scaling: every rank restores its own `per_rank` images."""
    return rank * per_rank, per_rank


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_histories(best_iters: List[int], rre_last: List[float], device=None):
    """All-gathers (image-count, best iteration, last RRE) per rank; returns the
    concatenation in rank order on every rank."""
    import torch
    import torch.distributed as dist
    mine = torch.tensor([[float(b), float(r)] for b, r in zip(best_iters, rre_last)],
                        dtype=torch.float64, device=device).reshape(-1, 2)
    if not (dist.is_available() and dist.is_initialized()):
        return mine.cpu().numpy()
    n = torch.tensor([mine.shape[0]], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(dist.get_world_size())]
    dist.all_gather(sizes, n)
    mx = int(max(int(s.item()) for s in sizes))
    pad = torch.zeros((mx, 2), dtype=torch.float64, device=device)
    pad[: mine.shape[0]] = mine
    out = [torch.zeros_like(pad) for _ in sizes]
    dist.all_gather(out, pad)
    import numpy as np
    return np.concatenate([o[: int(s.item())].cpu().numpy() for o, s in zip(out, sizes)])
