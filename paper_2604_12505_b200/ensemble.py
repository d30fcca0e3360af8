"""Ensemble sharding across ranks: rollouts are independent units, so each rank owns
a contiguous block of GLOBAL rollout ids and seeds its inputs by global id; the only collective
is one gather of the trajectory dataset after the run (NCCL all_gather on GPUs; any
torch.distributed backend works, the tests use gloo on CPU)."""
from __future__ import annotations


def shard(n_total: int, world: int, rank: int) -> range:
    """Global rollout ids owned by `rank` (contiguous blocks; the first n_total % world ranks
    get one extra)."""
    if not (0 <= rank < world) or n_total < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def gather_trajectories(y_local, group=None):
    """Gather per-rank trajectory tensors [B_local, K, C] into [sum B, K, C] in global-id order on
    every rank.  Equal B_local uses all_gather_into_tensor (one NCCL call); unequal falls back to
    padded all_gather."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n = torch.tensor([y_local.shape[0]], device=y_local.device, dtype=torch.int64)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    if len(set(sizes)) == 1:
        out = torch.empty((world * sizes[0],) + tuple(y_local.shape[1:]), dtype=y_local.dtype,
                          device=y_local.device)
        if y_local.device.type == "cuda":
            dist.all_gather_into_tensor(out, y_local.contiguous(), group=group)
        else:
            parts = list(out.chunk(world))
            dist.all_gather(parts, y_local.contiguous(), group=group)
            out = torch.cat(parts)
        return out
    m = max(sizes)
    pad = torch.zeros((m,) + tuple(y_local.shape[1:]), dtype=y_local.dtype, device=y_local.device)
    pad[:y_local.shape[0]] = y_local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)])
