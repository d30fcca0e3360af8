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
    if y_local.is_cuda and dist.get_backend(group) == "gloo":   # gloo gathers host tensors
        return gather_trajectories(y_local.cpu(), group).to(y_local.device)
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


def ensemble_inputs_for(ids, K: int, kind: str, n_total: int):
    """(u [B, K, 3] float32, theta_ref [B, K] float32 or None) of the given GLOBAL rollout ids:
    "excitation" = the C3 open-loop identification train (seed 1000 + id),
    "profiles" = C5: ids < n_total / 2 fly manoeuvre profile 1, the others profile 2
    (P:376-379), amplitudes / timings randomised by id (seed 2000 + id), under the PD law."""
    import numpy as np
    import sph_inputs as si
    ids = list(ids)
    if not ids:
        return np.zeros((0, K, 3), np.float32), (np.zeros((0, K), np.float32) if kind == "profiles" else None)
    if kind == "excitation":
        return si.ensemble_inputs(ids, K)[0], None
    if kind == "profiles":
        return si.profile_inputs(ids, n_total, K)
    raise ValueError(kind)


def gather_dataset(y, u_applied, status, group=None):
    """One collective step after the run: the trajectory dataset D_N = {(u_k, y_k)}
    (Eq. dataset) of every rank plus the per-rollout status, in global-id order."""
    import torch
    yu = torch.cat([y, u_applied], dim=2)                        # [B, K, 9]: one gather
    out = gather_trajectories(yu, group)
    st = gather_trajectories(status.to(torch.float32).reshape(-1, 1, 1), group).reshape(-1)
    return out[..., :6], out[..., 6:], st.to(torch.int32)


def run_ensemble(sp, fluid_pv, ghost_b, n_total: int, K: int, kind: str = "excitation",
                 rank: int = 0, world: int = 1, device: int = 0, group=None, **ctx_kw):
    """Shard n_total rollouts over `world` ranks by global id, run K slow ticks of this rank's
    shard on `device` through the C ABI (sph_rollout_batch, device pointers), gather the
    dataset.  Returns (y [n_total, K, 6], u_applied [n_total, K, 3], status [n_total]) on every
    rank (torch tensors on the device) -- bitwise independent of world and of the batch
    position (each rollout's inputs and arithmetic depend only on its global id)."""
    import torch
    from .binding import SphContext
    ids = list(shard(n_total, world, rank))
    u, th = ensemble_inputs_for(ids, K, kind, n_total)
    dev = torch.device("cuda", device)
    ctx = SphContext(sp, fluid_pv, ghost_b, n_rollouts=max(len(ids), 1), device=device, **ctx_kw)
    try:
        ud = torch.from_numpy(u).to(dev)
        if len(ids) == 0:
            raise ValueError("empty shard")
        thd = torch.from_numpy(th).to(dev) if th is not None else None
        y, ua = ctx.rollout(ud, theta_ref=thd, Kp=sp.Kp if thd is not None else 0.0,
                            Kd=sp.Kd if thd is not None else 0.0)
        st = torch.from_numpy(ctx.get_status()[0]).to(dev)
    finally:
        ctx.close()
    if world == 1:
        return y, ua, st
    return gather_dataset(y, ua, st, group)
