"""Host-side sharding plans and collective helpers (backend-agnostic: NCCL on
GPUs, gloo in the CPU tests).  No arithmetic of the method lives here: the
exact statistic reductions and the log-sum-exp merge run in the CUDA library
(magicpig_reduce_stats, magicpig_merge_partials)."""
from __future__ import annotations

from typing import List, Tuple

import torch


def sequence_shard(n_global: int, world: int, rank: int, align: int = 1024) -> Tuple[int, int]:
    """Contiguous key range [offset, offset + n_local) of `rank` (sequence
    parallelism).  Boundaries are multiples of `align` (code chunks stay whole)
    except the last; every key belongs to exactly one rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    blocks = -(-n_global // align)
    b0 = rank * blocks // world
    b1 = (rank + 1) * blocks // world
    lo = min(b0 * align, n_global)
    hi = min(b1 * align, n_global)
    return lo, hi - lo


def head_shard(Hkv: int, world: int, rank: int) -> Tuple[int, int]:
    """kv heads [h0, h1) owned by `rank` (head parallelism; GQA query heads
    h*G .. h*G+G-1 follow their kv head).  No collective on the data path."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return rank * Hkv // world, (rank + 1) * Hkv // world


def all_gather_stacked(t: torch.Tensor, group=None) -> torch.Tensor:
    """[P, *t.shape] tensor of every rank's `t`, in rank order."""
    import torch.distributed as dist
    P = dist.get_world_size(group)
    t = t.contiguous()
    out = torch.empty((P,) + tuple(t.shape), dtype=t.dtype, device=t.device)
    try:
        dist.all_gather_into_tensor(out, t, group=group)
    except (RuntimeError, NotImplementedError, AttributeError):
        parts: List[torch.Tensor] = [torch.empty_like(t) for _ in range(P)]
        dist.all_gather(parts, t, group=group)
        out = torch.stack(parts)
    return out
